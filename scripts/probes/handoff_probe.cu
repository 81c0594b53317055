// Probe: per-kernel cost of a dependent-kernel chain inside one CUDA graph,
// handing off with (a) griddepcontrol.wait (PDL), (b) a release/acquire
// counter per launch (the dependent's CTAs are resident early via PDL and
// spin on the predecessor's counter instead of waiting for grid
// completion), (c) plain stream order.  Each kernel reads the previous
// kernel's output and writes its own (latency-bound, like route/combine).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/probes/handoff_probe scripts/probes/handoff_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <int MODE>  // 0 PDL wait, 1 flags, 2 plain
__global__ void link(float* buf, int k, int n, int* cnt, int prev_ctas) {
    if (MODE == 1) {
        dep_launch();
        if (k > 0 && threadIdx.x == 0) {
            int v;
            do {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(cnt + k - 1) : "memory");
            } while (v < prev_ctas);
        }
        __syncthreads();
    } else if (MODE == 0) {
        dep_wait();
        dep_launch();
    }
    // read the predecessor's slice, write ours
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const float x = k > 0 ? buf[(size_t)(k - 1) * n + i] : 0.f;
    buf[(size_t)k * n + i] = x + 1.f;
    if (MODE == 1) {
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(cnt + k), "r"(1) : "memory");
    }
}

template <int MODE>
static float run(int ctas, int chain) {
    const int thr = 256, n = ctas * thr;
    float* buf;
    int* cnt;
    cudaMalloc(&buf, (size_t)chain * n * 4);
    cudaMalloc(&cnt, chain * 4);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    cudaMemsetAsync(cnt, 0, chain * 4, st);
    for (int k = 0; k < chain; ++k) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ctas);
        cfg.blockDim = dim3(thr);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = (MODE == 2 || k == 0) ? 0 : 1;
        cudaLaunchKernelEx(&cfg, link<MODE>, buf, k, n, cnt, ctas);
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(a, st);
        cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    float chk = 0;
    cudaMemcpy(&chk, buf + (size_t)(chain - 1) * n, 4, cudaMemcpyDeviceToHost);
    if (chk != (float)chain) printf("  !! wrong result %f\n", chk);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaFree(buf);
    cudaFree(cnt);
    return best * 1000.f / chain;
}

int main() {
    const int chain = 200;
    printf("per-kernel time in a %d-kernel dependent chain (us), 256 threads per CTA\n", chain);
    printf("CTAs | PDL wait | release/acquire counter | plain stream order  (%s)\n", cudaGetErrorString(cudaGetLastError()));
    for (int ctas : {1, 9, 96, 148, 296}) {
        const float a = run<0>(ctas, chain), b = run<1>(ctas, chain), c = run<2>(ctas, chain);
        printf("%4d | %8.2f | %8.2f | %8.2f  (%s)\n", ctas, a, b, c, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
