// common.cuh — device helpers shared by every kernel of the verify step.
//
// Data layouts in HBM:
//  * A-frag (weights).  A [rows, K] matrix is cut into super-tiles of
//    kTPW*16 = 64 rows; each super-tile is stored k-step by k-step (16
//    columns), and inside a k-step the kTPW 16x16 tiles are stored as the 32
//    lanes' mma.m16n8k16 A-fragments: lane (g = lane/4, t = lane%4) owns the
//    16 bytes {W[g][2t..2t+1], W[g+8][2t..2t+1], W[g][2t+8..2t+9],
//    W[g+8][2t+8..2t+9]}.  One warp therefore streams a weight matrix with
//    one fully coalesced 512-byte LDG.128 per tile per k-step and the bytes
//    land directly in mma registers: no shared-memory transpose, no bank
//    conflicts, no per-element index math on the hot path.
//  * B-frag (activations, <= 16 tokens).  Element (tok, k) of a [16, K]
//    bf16 activation lives where lane (g = tok%8, t = (k%8)/2) of n-tile
//    tok/8 expects it for k-step k/16: one 8-byte LDG.64 per n-tile per
//    k-step.  Producers (norms, SiLU epilogue, attention) write this layout
//    directly.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "cascade_weights.h"

namespace cascade {

constexpr int kTPW = 4;                 // 16-row tiles per super-tile (per warp)
constexpr int kSTRows = 16 * kTPW;      // 64 rows per super-tile
constexpr int kMaxT = 16;               // tokens in flight (two n8 tiles)
constexpr int kReadyStride = 32;        // ints: one 128-byte line per fused-FFN slot readiness counter

__device__ __forceinline__ uint64_t globaltimer_raw() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Programmatic dependent launch: every kernel of the step waits for its
// predecessor's completion (and memory) before touching any data, so the
// chain stays transitively ordered while launch latency and CTA
// rasterisation overlap the predecessor's tail.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// A/B switch (CASCADE_LATE_TRIGGER=1 for all, or a mask of kLate*):
// latency-bound kernels let their dependents launch only at exit, so the
// next GEMV's weight prologue does not compete with their loads.
enum { kLateAttn = 1, kLateAttnCombine = 2, kLateRoute = 4, kLateCombine = 8, kLateEmbed = 16 };
__device__ int g_late_trigger = 0;
__device__ __forceinline__ void griddep_launch_early(int kind) {
    if (!(g_late_trigger & kind)) griddep_launch();
}

// Bulk L2 prefetch of an upcoming weight matrix, spread over every thread
// of the grid.  Issued from latency-bound kernels (attention, combine) so
// HBM keeps streaming the next dense GEMV's weights into the 126 MB L2
// while those kernels wait on latency.
__device__ __forceinline__ void prefetch_l2(const void* base, unsigned long long bytes) {
    if (base == nullptr || bytes == 0) return;
    constexpr unsigned long long kChunkB = 16384;
    const unsigned long long n = (bytes + kChunkB - 1) / kChunkB;
    const unsigned long long nthr = (unsigned long long)gridDim.x * gridDim.y * blockDim.x;
    const unsigned long long me =
        ((unsigned long long)blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
    for (unsigned long long c = me; c < n; c += nthr) {
        const unsigned long long off = c * kChunkB;
        unsigned long long sz = bytes - off < kChunkB ? bytes - off : kChunkB;
        sz &= ~15ull;
        if (sz == 0) continue;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((const char*)base + off), "r"((uint32_t)sz)
                     : "memory");
    }
}

// Per-CTA timeline (diagnostic, cascade_step_cta_trace): when g_cta_trace
// is set, every CTA records the globaltimer at its start (after
// griddepcontrol.wait) and at its exit, at [(slot * kCtaTraceCap + cta) * kCtaRec + {0, 1}];
// records 2..3 hold optional per-CTA phase stamps (cta_phase).
// Null in normal runs: one predicated global load per kernel.
constexpr int kCtaTraceCap = 512;
constexpr int kCtaRec = 4;  // u64 per CTA record: start, exit, phase a, phase b
constexpr int kPhaseBase = 496;  // CTA records >= this hold CTA 0's phase stamps
__device__ unsigned long long* g_cta_trace = nullptr;
__device__ unsigned long long* g_cta_trace_base = nullptr;  // the session's trace slot 0

__device__ __forceinline__ unsigned long long* cta_trace_slot(unsigned long long* slot) {
    unsigned long long* buf = g_cta_trace;
    if (buf == nullptr || slot == nullptr) return nullptr;
    const long long cta = (long long)blockIdx.y * gridDim.x + blockIdx.x;
    if (cta >= kPhaseBase) return nullptr;
    return buf + ((slot - g_cta_trace_base) * kCtaTraceCap + cta) * kCtaRec;
}

// per-kernel start stamp for in-graph tracing (block 0, thread 0)
__device__ __forceinline__ void trace_start(unsigned long long* slot) {
    if (slot != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *slot = globaltimer_raw();
    if (threadIdx.x == 0) {
        unsigned long long* c = cta_trace_slot(slot);
        if (c != nullptr) {
            uint32_t smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            c[0] = (globaltimer_raw() & ~0xFFull) | (smid & 0xFF);  // low byte: SM id (timer resolution >= 256 ns... ~32 ns)
        }
    }
}

// CTA exit stamp: the latest warp to leave wins (RAII: every return path).
struct CtaExitStamp {
    unsigned long long* c;
    __device__ explicit CtaExitStamp(unsigned long long* slot) : c(cta_trace_slot(slot)) {}
    __device__ ~CtaExitStamp() {
        if (c != nullptr && (threadIdx.x & 31) == 0) atomicMax(c + 1, globaltimer_raw());
    }
};
// Phase stamps of CTA 0 (diagnostic): stamp i of a launch goes to the
// unused CTA records 496.. of its slot (scripts/cta_timeline.py).
__device__ __forceinline__ void phase_stamp(unsigned long long* slot, int i) {
    unsigned long long* buf = g_cta_trace;
    if (buf == nullptr || slot == nullptr || blockIdx.x != 0 || blockIdx.y != 0 || threadIdx.x != 0) return;
    buf[(slot - g_cta_trace_base) * kCtaTraceCap * kCtaRec + kPhaseBase * kCtaRec + i] = globaltimer_raw();
}
// CTA-0 phase stamp from any single thread (phase_stamp is thread 0's)
__device__ __forceinline__ void phase_stamp_cta0(unsigned long long* slot, int i) {
    unsigned long long* buf = g_cta_trace;
    if (buf == nullptr || slot == nullptr || blockIdx.x != 0 || blockIdx.y != 0) return;
    buf[(slot - g_cta_trace_base) * kCtaTraceCap * kCtaRec + kPhaseBase * kCtaRec + i] = globaltimer_raw();
}
// Per-warp stamp (diagnostic) of CTAs 0 and 1: stamp 16 + cta*16 + warp*2 + which
// of the CTA-0 phase area (e.g. each warp's end of its gate/up and down ranges).
__device__ __forceinline__ void warp_stamp(unsigned long long* slot, int which) {
    unsigned long long* buf = g_cta_trace;
    const int warp = threadIdx.x >> 5;
    if (buf == nullptr || slot == nullptr || blockIdx.x > 1 || blockIdx.y != 0 || (threadIdx.x & 31) != 0 || warp > 7) return;
    buf[(slot - g_cta_trace_base) * kCtaTraceCap * kCtaRec + kPhaseBase * kCtaRec + 16 + blockIdx.x * 16 + warp * 2 + which] =
        globaltimer_raw();
}
// Per-CTA phase stamp (diagnostic): record `which` (2 or 3) of this CTA
// keeps the latest stamp of any warp that reports it.
__device__ __forceinline__ void cta_phase(unsigned long long* slot, int which) {
    unsigned long long* c = cta_trace_slot(slot);
    if (c != nullptr && (threadIdx.x & 31) == 0) atomicMax(c + which, globaltimer_raw());
}
#define CTA_TRACE(slot)   \
    trace_start(slot);    \
    CtaExitStamp cta_exit_stamp_(slot)

// gpu-scope release / acq_rel atomics (one lane publishes what its CTA
// ordered before it with a barrier: PTX fences and release ops are cumulative)
__device__ __forceinline__ void red_add_release(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atomic_add_acq_rel(int* p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Weights are read exactly once per step: bypass L1, keep them from
// displacing activations in L2 (evict_first).
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint4 ldg_stream(const uint4* p, uint64_t pol) {
    uint4 v;
    asm volatile(
        "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
        : "l"(p), "l"(pol));
    return v;
}

// Activations: small, re-read by every warp of the SM -> cache in L1.
__device__ __forceinline__ uint2 ldg_act(const uint2* p) {
    uint2 v;
    asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}

// Activations written earlier in the same launch (fused expert FFN): L2 only.
__device__ __forceinline__ uint2 ldcg_act(const uint2* p) {
    uint2 v;
    asm volatile("ld.global.cg.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}

__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint4& a, const uint2& b) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y));
}

// bf16 element index of activation (tok, k) inside a B-frag buffer.
__host__ __device__ __forceinline__ long long bfrag_index(int tok, int k) {
    const int s = k >> 4, kk = k & 15;
    const int hi = kk >> 3, kk2 = kk & 7;
    const int t = kk2 >> 1, w = kk2 & 1;
    const int nt = tok >> 3, g = tok & 7;
    const int lane = g * 4 + t;
    return ((((long long)s * 2 + nt) * 32 + lane) * 4) + hi * 2 + w;
}

// Logical (row, col) of bf16 element `e` (0..7) of lane `lane` in a 16x16 tile.
__host__ __device__ __forceinline__ void afrag_coords(int lane, int e, int& r, int& c) {
    const int g = lane >> 2, t = lane & 3;
    r = g + 8 * ((e >> 1) & 1);
    c = 2 * t + (e & 1) + 8 * (e >> 2);
}

__device__ __forceinline__ float bf16_round(float x) {
    return __bfloat162float(__float2bfloat16_rn(x));
}

__device__ __forceinline__ uint16_t bf16_bits(float x) {
    __nv_bfloat16 h = __float2bfloat16_rn(x);
    return *reinterpret_cast<uint16_t*>(&h);
}

__device__ __forceinline__ float bits_to_f32(uint16_t b) {
    return __uint_as_float(((uint32_t)b) << 16);
}

// Block-wide sum (blockDim.x multiple of 32, <= 1024). `red` holds 32 floats.
__device__ __forceinline__ float block_sum(float v, float* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    const int nw = blockDim.x >> 5;
    float s = 0.f;
    if (warp == 0) {
        s = lane < nw ? red[lane] : 0.f;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red[0] = s;
    }
    __syncthreads();
    s = red[0];
    __syncthreads();
    return s;
}

// Order-preserving float key for atomicMax argmax; low word breaks ties
// toward the lower index (reference tie rule, controller.hpp:124-125).
__device__ __forceinline__ unsigned long long argmax_key(float v, int idx) {
    uint32_t u = __float_as_uint(v);
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ((unsigned long long)u << 32) | (0xFFFFFFFFu - (uint32_t)idx);
}
__device__ __forceinline__ int argmax_key_index(unsigned long long k) {
    return (int)(0xFFFFFFFFu - (uint32_t)(k & 0xFFFFFFFFull));
}

}  // namespace cascade
