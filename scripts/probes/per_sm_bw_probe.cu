// Probe: streaming read bandwidth PER SM as a function of how many SMs
// stream (one CTA per SM), for a TMA bulk ring (the dense tcgen05 GEMV's
// producer pattern) and for LDG.128 (the expert GEMV's pattern).  Answers:
// is a kernel that streams from N < 148 SMs capped by a per-SM rate?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/probes/per_sm_bw_probe scripts/probes/per_sm_bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGE, int NST>
__global__ void __launch_bounds__(160) tma_ring(const char* __restrict__ src, long long per_cta, unsigned* sink) {
    extern __shared__ __align__(128) unsigned char ring[];
    __shared__ __align__(8) uint64_t full[NST], empty[NST];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&full[i])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&empty[i])), "r"(4));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const char* base = src + per_cta * blockIdx.x;
    const int nstage = (int)(per_cta / STAGE);
    if (warp == 4) {
        if (lane == 0) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            for (int i = 0; i < nstage; ++i) {
                const int s = i % NST;
                if (i >= NST)
                    asm volatile("{.reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W%=;}" ::"r"(su(&empty[s])), "r"(((i / NST) - 1) & 1) : "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(STAGE) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(su(ring + (size_t)s * STAGE)), "l"(base + (long long)i * STAGE), "r"(STAGE), "r"(su(&full[s])), "l"(pol) : "memory");
            }
        }
        return;
    }
    unsigned acc = 0;
    for (int i = 0; i < nstage; ++i) {
        const int s = i % NST;
        asm volatile("{.reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W%=;}" ::"r"(su(&full[s])), "r"((i / NST) & 1) : "memory");
        const uint4* r = reinterpret_cast<const uint4*>(ring + (size_t)s * STAGE);
        acc += r[threadIdx.x].x;
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
    }
    if (acc == 0x12345678u) *sink = acc;
}

template <int U>
__global__ void __launch_bounds__(1024) ldg_stream(const uint4* __restrict__ src, long long per_cta16, unsigned* sink) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const long long per_warp = per_cta16 / nw / 32 * 32;
    const uint4* p = src + per_cta16 * blockIdx.x + per_warp * warp + lane;
    unsigned acc = 0;
    for (long long i = 0; i + U * 32 <= per_warp; i += U * 32) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + i + u * 32));
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x;
    }
    if (acc == 0x12345678u) *sink = acc;
}

template <typename F>
static float timeit(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        f();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    const long long per_cta = 8ll << 20;  // 8 MB per CTA: steady state dominates
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    char* src;
    unsigned* sink;
    cudaMalloc(&src, per_cta * sms);
    cudaMalloc(&sink, 4);
    cudaMemset(src, 1, per_cta * sms);
    cudaDeviceSynchronize();
    const int ns[] = {8, 16, 32, 48, 64, 96, 128, 148};
    cudaFuncSetAttribute(tma_ring<32768, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 32768);
    cudaFuncSetAttribute(tma_ring<32768, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    printf("SMs streaming | TMA 3x32KB GB/s/SM total | TMA 6x32KB GB/s/SM total | LDG.128 U=8 x1024thr GB/s/SM total\n");
    for (int n : ns) {
        if (n > sms) continue;
        const float t3 = timeit([&] { tma_ring<32768, 3><<<n, 160, 3 * 32768>>>(src, per_cta, sink); });
        const float t6 = timeit([&] { tma_ring<32768, 6><<<n, 160, 6 * 32768>>>(src, per_cta, sink); });
        const float tl = timeit([&] { ldg_stream<8><<<n, 1024>>>(reinterpret_cast<const uint4*>(src), per_cta / 16, sink); });
        const double b = (double)per_cta * n;
        printf("%4d | %7.1f %8.1f | %7.1f %8.1f | %7.1f %8.1f   (%s)\n", n, b / t3 / 1e6 / n, b / t3 / 1e6, b / t6 / 1e6 / n,
               b / t6 / 1e6, b / tl / 1e6 / n, b / tl / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
