// Probe for the tcgen05 weight-streaming engine (gemv_umma.cuh): exactness
// against a CPU reference on integer-valued bf16 data (fp32 sums are exact)
// and HBM bandwidth of a 470 MB dense stream.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -Iinclude \
//        -Ipaper_2506_20675_b200/csrc -o scripts/umma_probe scripts/umma_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gemv_umma.cuh"

using namespace cascade;

__host__ __device__ inline uint32_t hmix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return (uint32_t)x;
}
__host__ __device__ inline float wval(long long row, int col) { return (float)((int)(hmix(row * 100003ull + col) % 7) - 3) * 0.125f; }
__host__ __device__ inline float xval(int tok, int col) { return (float)((int)(hmix(0x9999ull + tok * 7777ull + col) % 5) - 2) * 0.25f; }

__global__ void fill_w(uint16_t* W, long long rows, int K) {
    const int n_ks = K / 16;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < rows * K; i += (long long)gridDim.x * blockDim.x) {
        const long long row = i / K;
        const int col = (int)(i % K);
        W[umma_a_index(row, col, n_ks)] = bf16_bits(wval(row, col));
    }
}
__global__ void fill_x(uint16_t* B, int K) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 16 * K; i += gridDim.x * blockDim.x) {
        const int tok = i / K, col = i % K;
        B[umma_b_index(tok, col)] = bf16_bits(xval(tok, col));
    }
}

// PDL primary: triggers its dependents at once, then stays busy for `ns`
__global__ void spin_kernel(unsigned long long ns, unsigned long long* dbg) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const unsigned long long t0 = globaltimer_raw();
    while (globaltimer_raw() - t0 < ns) {
    }
    if (threadIdx.x == 0) atomicMax(dbg + 11, globaltimer_raw());
}

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);     \
            return 1;                                                                           \
        }                                                                                       \
    } while (0)

static int run(long long rows, int K, int T, int reps, int grid) {
    uint16_t *W, *B;
    float *out, *partial;
    int* counters;
    const int n_st = (int)(rows / kURows), n_ks = K / 16;
    CK(cudaMalloc(&W, rows * K * 2));
    CK(cudaMalloc(&B, 16 * K * 2));
    CK(cudaMalloc(&out, 16 * rows * 4));
    CK(cudaMalloc(&partial, (size_t)grid * 2 * kUPartialFloats * 4));
    CK(cudaMalloc(&counters, n_st * 4));
    CK(cudaMemset(counters, 0, n_st * 4));
    fill_w<<<1024, 256>>>(W, rows, K);
    fill_x<<<64, 256>>>(B, K);
    CK(cudaDeviceSynchronize());
    UGemvParams p{};
    p.W = W;
    p.B = B;
    p.n_blocks = 1;
    p.n_st = n_st;
    p.n_ks = n_ks;
    p.T = T;
    p.partial = partial;
    p.counters = counters;
    p.out = out;
    p.ld = (int)rows;
    const int smem = gemv_umma_smem_bytes();
    CK(cudaFuncSetAttribute(stream_gemv_umma_kernel<UEPI_STORE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaMemset(out, 0, 16 * rows * 4));
    stream_gemv_umma_kernel<UEPI_STORE><<<grid, kUThreads, smem>>>(p);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<float> h(16 * rows);
    CK(cudaMemcpy(h.data(), out, h.size() * 4, cudaMemcpyDeviceToHost));
    long long bad = 0, checked = 0;
    for (long long row = 0; row < rows; row += (rows > 4096 ? 97 : 1)) {
        for (int t = 0; t < T; ++t) {
            double ref = 0;
            for (int c = 0; c < K; ++c) ref += (double)wval(row, c) * xval(t, c);
            ++checked;
            if ((float)ref != h[(size_t)t * rows + row]) {
                if (bad < 5) printf("  mismatch row %lld tok %d: gpu %g ref %g\n", row, t, h[(size_t)t * rows + row], ref);
                ++bad;
            }
        }
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double bytes = (double)rows * K * 2;
    printf("rows=%lld K=%d T=%d grid=%d: %lld/%lld mismatches\n", rows, K, T, grid, bad, checked);
    CK(cudaFuncSetAttribute(stream_gemv_umma_kernel<UEPI_STORE, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(stream_gemv_umma_kernel<UEPI_STORE, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int mode = 0; mode < 4; ++mode) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = kUThreads;
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = mode == 3 ? 1 : 0;
        auto k = mode == 1 ? stream_gemv_umma_kernel<UEPI_STORE, 1>
               : mode == 2 ? stream_gemv_umma_kernel<UEPI_STORE, 2> : stream_gemv_umma_kernel<UEPI_STORE, 0>;
        CK(cudaLaunchKernelEx(&cfg, k, p));
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        for (int r = 0; r < reps; ++r) cudaLaunchKernelEx(&cfg, k, p);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("   %-22s %8.2f us/launch, %7.1f GB/s\n",
               mode == 0 ? "full" : mode == 1 ? "no-mma" : mode == 2 ? "no-B" : "full+PDL back-to-back",
               ms * 1e3 / reps, bytes / (ms / reps) / 1e6);
    }
    // phase timeline behind a 10 us PDL primary (the in-graph situation)
    {
        unsigned long long* dbg;
        CK(cudaMalloc(&dbg, 16 * 8));
        for (int rep = 0; rep < 3; ++rep) {
            std::vector<unsigned long long> h0(16, 0);
            h0[10] = ~0ull;
            CK(cudaMemcpy(dbg, h0.data(), 16 * 8, cudaMemcpyHostToDevice));
            UGemvParams q = p;
            q.dbg = dbg;
            spin_kernel<<<grid, 32>>>(10000, dbg);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = grid;
            cfg.blockDim = kUThreads;
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            CK(cudaLaunchKernelEx(&cfg, stream_gemv_umma_kernel<UEPI_STORE, 0>, q));
            CK(cudaDeviceSynchronize());
            std::vector<unsigned long long> h(16);
            CK(cudaMemcpy(h.data(), dbg, 16 * 8, cudaMemcpyDeviceToHost));
            const double z = (double)h[11];
            auto rel = [&](int i) { return ((double)h[i] - z) / 1e3; };
            if (rep == 2)
                printf("   PDL timeline (us rel. to primary end): first CTA entry %.2f | CTA0 entry %.2f prod-wait %.2f "
                       "prod-done %.2f mma-start %.2f mma-done %.2f epi-wait %.2f epi-first %.2f epi-end %.2f | last CTA end %.2f\n",
                       rel(10), rel(0), rel(1), rel(2), rel(3), rel(4), rel(5), rel(6), rel(7), rel(9));
        }
        cudaFree(dbg);
    }
    cudaFree(W);
    cudaFree(B);
    cudaFree(out);
    cudaFree(partial);
    cudaFree(counters);
    return bad != 0;
}

int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int rc = 0;
    rc |= run(128, 64, 16, 3, 1);        // one unit, one CTA
    rc |= run(384, 256, 9, 3, 4);        // tiny QKV shape, split units
    rc |= run(6144, 4096, 9, 20, sms);   // Mixtral QKV
    rc |= run(4096, 4096, 1, 20, sms);   // Mixtral O
    rc |= run(57344, 4096, 16, 10, sms); // two Mixtral gate/up experts (470 MB)
    rc |= run(4096, 4096, 9, 20, sms);   // Mixtral O at T=9
    rc |= run(32000, 4096, 3, 10, sms);  // LM head
    printf("rc=%d\n", rc);
    return rc;
}
