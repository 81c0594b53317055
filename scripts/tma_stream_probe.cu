// Probe: HBM streaming bandwidth of a TMA-bulk ring (one producer lane,
// consumers touch one word per 16 B chunk) vs plain LDG.128, for several
// stage sizes / ring depths / CTAs per SM.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/tma_stream_probe scripts/tma_stream_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGE, int NST>
__global__ void __launch_bounds__(160) tma_ring(const uint4* __restrict__ src, long long n16, unsigned* sink) {
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
    const long long bytes = n16 * 16;
    const long long per = bytes / gridDim.x / STAGE * STAGE;
    const long long lo = per * blockIdx.x;
    const int nstage = (int)(per / STAGE);
    if (warp == 4) {
        if (lane == 0) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            for (int i = 0; i < nstage; ++i) {
                const int s = i % NST;
                if (i >= NST) {
                    asm volatile("{.reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W%=;}" ::"r"(su(&empty[s])), "r"(((i / NST) - 1) & 1) : "memory");
                }
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(STAGE) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(su(ring + (size_t)s * STAGE)), "l"((const char*)src + lo + (long long)i * STAGE), "r"(STAGE), "r"(su(&full[s])), "l"(pol) : "memory");
            }
        }
        return;
    }
    unsigned acc = 0;
    for (int i = 0; i < nstage; ++i) {
        const int s = i % NST;
        asm volatile("{.reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W%=;}" ::"r"(su(&full[s])), "r"((i / NST) & 1) : "memory");
        const uint4* r = reinterpret_cast<const uint4*>(ring + (size_t)s * STAGE);
        for (int j = threadIdx.x; j < STAGE / 16; j += 128) acc += r[j].x;
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[s])) : "memory");
    }
    if (acc == 0x12345678u) *sink = acc;
}

template <int U>
__global__ void __launch_bounds__(256) ldg_stream(const uint4* __restrict__ src, long long n16, unsigned* sink) {
    const long long nthr = (long long)gridDim.x * blockDim.x;
    const long long per = n16 / nthr / 32 * 32;
    const int lane = threadIdx.x & 31;
    const long long warp_id = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint4* p = src + warp_id * per * 32 + lane;
    unsigned acc = 0;
    for (long long i = 0; i + U <= per; i += U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p + (i + u) * 32));
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

template <int STAGE, int NST>
static void run_tma(const uint4* src, long long n16, unsigned* sink, int ctas_per_sm, int sms) {
    const int smem = STAGE * NST;
    cudaFuncSetAttribute(tma_ring<STAGE, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = sms * ctas_per_sm;
    float ms = timeit([&] { tma_ring<STAGE, NST><<<grid, 160, smem>>>(src, n16, sink); });
    long long moved = (long long)(n16 * 16 / grid / STAGE) * STAGE * grid;
    printf("tma stage=%6d nst=%2d ctas/sm=%d inflight/SM=%4d KB: %7.1f GB/s  (%s)\n", STAGE, NST, ctas_per_sm,
           STAGE * NST * ctas_per_sm / 1024, moved / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    printf("start\n");
    const long long bytes = 4ll << 30;
    uint4* src;
    unsigned* sink;
    cudaMalloc(&src, bytes);
    cudaMalloc(&sink, 4);
    printf("malloc %s\n", cudaGetErrorString(cudaGetLastError()));
    cudaMemset(src, 1, bytes);
    cudaDeviceSynchronize();
    printf("memset %s\n", cudaGetErrorString(cudaGetLastError()));
    const long long n16 = bytes / 16;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int c = 1; c <= 2; ++c) {
        run_tma<8192, 8>(src, n16, sink, c, sms);
        run_tma<8192, 12>(src, n16, sink, c, sms);
        run_tma<16384, 4>(src, n16, sink, c, sms);
        run_tma<16384, 5>(src, n16, sink, c, sms);
        run_tma<16384, 6>(src, n16, sink, c, sms);
        run_tma<32768, 3>(src, n16, sink, c, sms);
    }
    run_tma<16384, 8>(src, n16, sink, 1, sms);
    run_tma<16384, 12>(src, n16, sink, 1, sms);
    run_tma<32768, 6>(src, n16, sink, 1, sms);
    run_tma<4096, 24>(src, n16, sink, 1, sms);
    run_tma<4096, 24>(src, n16, sink, 2, sms);
    for (int cps = 1; cps <= 4; cps *= 2) {
        float ms = timeit([&] { ldg_stream<4><<<sms * cps, 256>>>(src, n16, sink); });
        printf("ldg U=4 ctas/sm=%d: %7.1f GB/s\n", cps, bytes / ms / 1e6);
        ms = timeit([&] { ldg_stream<8><<<sms * cps, 256>>>(src, n16, sink); });
        printf("ldg U=8 ctas/sm=%d: %7.1f GB/s\n", cps, bytes / ms / 1e6);
    }
    return 0;
}
