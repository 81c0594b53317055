// Probe: is a cooperative launch (grid-wide co-residency guarantee) allowed
// together with programmatic dependent launch inside stream capture?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o coop_pdl_probe coop_pdl_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void producer(int* x) {
    asm volatile("griddepcontrol.launch_dependents;");
    if (threadIdx.x == 0) atomicAdd(x, 1);
}
__global__ void spin_all(int* flag, int* out) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // every CTA arrives, then waits for all: deadlocks unless co-resident
    __shared__ int ok;
    if (threadIdx.x == 0) {
        atomicAdd(flag, 1);
        int v;
        long long spins = 0;
        do {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
            if (++spins > (1ll << 26)) { ok = 0; break; }
            ok = 1;
        } while (v < (int)gridDim.x);
    }
    __syncthreads();
    if (threadIdx.x == 0 && ok) atomicAdd(out, 1);
}

static const char* run(bool coop, bool pdl, bool capture, int grid) {
    static char buf[256];
    int *flag, *out, *x;
    cudaMalloc(&flag, 4); cudaMalloc(&out, 4); cudaMalloc(&x, 4);
    cudaMemset(flag, 0, 4); cudaMemset(out, 0, 4);
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaGraph_t g = nullptr; cudaGraphExec_t ge = nullptr;
    cudaError_t e = cudaSuccess;
    if (capture) e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    producer<<<1, 32, 0, st>>>(x);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid); cfg.blockDim = dim3(256); cfg.stream = st;
    cudaLaunchAttribute at[2]; int na = 0;
    if (coop) { at[na].id = cudaLaunchAttributeCooperative; at[na].val.cooperative = 1; ++na; }
    if (pdl) { at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[na].val.programmaticStreamSerializationAllowed = 1; ++na; }
    cfg.attrs = at; cfg.numAttrs = na;
    cudaError_t le = cudaLaunchKernelEx(&cfg, spin_all, flag, out);
    if (capture) {
        cudaError_t ce = cudaStreamEndCapture(st, &g);
        if (le == cudaSuccess && ce == cudaSuccess) {
            e = cudaGraphInstantiate(&ge, g, 0);
            if (e == cudaSuccess) e = cudaGraphLaunch(ge, st);
        } else e = le != cudaSuccess ? le : ce;
    } else e = le;
    cudaError_t se = cudaStreamSynchronize(st);
    int h = -1; cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
    snprintf(buf, sizeof buf, "launch=%s sync=%s ok_ctas=%d/%d", cudaGetErrorString(e), cudaGetErrorString(se), h, grid);
    cudaGetLastError();
    if (ge) cudaGraphExecDestroy(ge);
    if (g) cudaGraphDestroy(g);
    cudaFree(flag); cudaFree(out); cudaFree(x); cudaStreamDestroy(st);
    return buf;
}

int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spin_all, 256, 0);
    printf("sms=%d occ/SM=%d\n", sms, occ);
    const int grid = 2 * sms;
    printf("coop+pdl, captured : %s\n", run(true, true, true, grid));
    printf("coop, captured     : %s\n", run(true, false, true, grid));
    printf("coop+pdl, eager    : %s\n", run(true, true, false, grid));
    printf("coop too large     : %s\n", run(true, false, false, sms * occ + 1));
    return 0;
}
