// Probe: does compute-sanitizer racecheck model mbarrier ordering?  A minimal,
// correct TMA ring (one producer lane, cp.async.bulk -> full barrier with
// complete_tx; 4 consumer warps read the slot with LDS after try_wait and
// release it on an empty barrier) plus an mbarrier-ordered warp -> warp
// shared-memory handoff.  Any hazard racecheck reports here is a false
// positive of the same kind as in ffn_ring.cuh.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/probes/racecheck_mbarrier_probe scripts/probes/racecheck_mbarrier_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
    asm volatile("{.reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W%=;}" ::"r"(su(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }

constexpr int STAGE = 4096, NST = 2, N = 8;
__global__ void __launch_bounds__(192) ring(const char* src, unsigned* out) {
    __shared__ __align__(128) unsigned char buf[NST * STAGE];
    __shared__ __align__(8) uint64_t full[NST], empty[NST], hand_full, hand_empty;
    __shared__ float hand[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&full[i])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&empty[i])), "r"(4));
        }
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&hand_full)), "r"(1));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&hand_empty)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 4) {
        if (lane == 0)
            for (int i = 0; i < N; ++i) {
                const int s = i % NST;
                if (i >= NST) wait(&empty[s], ((i / NST) - 1) & 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(STAGE) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(buf + s * STAGE)),
                             "l"(src + (long long)i * STAGE), "r"(STAGE), "r"(su(&full[s])) : "memory");
            }
        return;
    }
    if (warp == 5) {  // consumer of warp 0's handoff
        for (int r = 0; r < N; ++r) {
            wait(&hand_full, r & 1);
            const float v = hand[lane];
            __syncwarp();
            if (lane == 0) arrive(&hand_empty);
            if (v == -1.f) out[1] = 1;
        }
        return;
    }
    unsigned acc = 0;
    for (int i = 0; i < N; ++i) {
        const int s = i % NST;
        wait(&full[s], (i / NST) & 1);
        acc += reinterpret_cast<const unsigned*>(buf + s * STAGE)[warp * 32 + lane];
        __syncwarp();
        if (lane == 0) arrive(&empty[s]);
        if (warp == 0) {  // handoff to warp 5 through shared memory, ordered by mbarriers
            if (i > 0) wait(&hand_empty, (i - 1) & 1);
            hand[lane] = (float)acc;
            __syncwarp();
            if (lane == 0) arrive(&hand_full);
        }
    }
    atomicAdd(out, acc);
}

int main() {
    char* src;
    unsigned* out;
    cudaMalloc(&src, N * STAGE);
    cudaMemset(src, 1, N * STAGE);
    cudaMalloc(&out, 8);
    cudaMemset(out, 0, 8);
    ring<<<1, 192>>>(src, out);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned h[2];
    cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
    printf("%s sum %u (expect %u)\n", cudaGetErrorString(e), h[0], (unsigned)(N * 128 * 0x01010101u));
    return 0;
}
