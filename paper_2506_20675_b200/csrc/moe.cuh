// moe.cuh — step entry (embedding), router, expert combine
// (SURVEY.md §8(a2) stage K1 and the epilogue of K3; the expert union, K2,
// is built by every expert-GEMV CTA: gemv.cuh build_union).
//
// moe_route_kernel (grid = T, one CTA per token):
//   1. RMSNorm of the residual row -> bf16 MoE input (B-frag layout for the
//      expert GEMVs), 16-byte stores.
//   2. Router logits: one warp per router row (E routed rows + the Qwen
//      shared-expert gate row), bf16 weights staged in shared memory before
//      the dependency wait when they fit, fp32 accumulate.
//   3. Softmax and top-k (larger logit first, lower expert index on ties),
//      gate weights (renormalised over the k for Mixtral): the real
//      counterpart of the reference's stand-in draw_expert_set
//      (expert_model.hpp:100-112).
// moe_combine_kernel (grid = T): residual += sum_r w[t][r] * Y[t][r]
//   (+ shared-gate * sum_b Y[t][k+b]) in fixed order, then the next RMSNorm
//   (next layer's attention input, or the final norm).
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "gemv_umma.cuh"

namespace cascade {

constexpr int kRouteThreads = 256;
constexpr int kRouteWarps = kRouteThreads / 32;
constexpr int kMaxExperts = 128;  // expert_model.hpp:96 (kMaxRoutedExperts)
constexpr int kMaxTopK = 16;

struct RouteParams {
    const float* x;              // residual [T][d]
    const uint16_t* norm_w;      // [d] bf16
    const uint16_t* router_w;    // [E + shared_gate][d] bf16
    uint16_t* xn_bfrag;          // out: MoE input, B-frag
    float* logits;               // out: [T][E+1]
    int* topk_id;                // out: [T][k]
    float* topk_w;               // out: [T][k]
    float* gsh;                  // out: [T] shared-expert gate (1 if no gate)
    float* ycontrib;             // [T][k+S][d], zeroed for non-local entries (EP)
    uint16_t* tap_xn;            // optional [T][d]
    int T, d, E, k, S, renorm, shared_gate;
    int e_lo, e_hi;              // local routed experts [e_lo, e_hi)
    int ep_rank, ep_size;        // shared block b lives on rank b % ep_size
    float eps;
    int zero_nonlocal;
    int stage_w;                 // router weights staged in smem before griddepcontrol.wait
    int C;                       // > 1: cluster of C CTAs per token, each staging 1/C of the router rows
    int* ffn_ready;              // fused expert FFN readiness counters: zeroed here, before this layer's FFN
    int n_ready;
    int par_topk;                // 1: top-k by parallel rank counting (default); 0: k serial warp selections
    unsigned long long* stamp;   // MoE-block start (CostBreakdown split)
    unsigned long long* trace;
};

#ifndef CASCADE_ROW_THREADS
#define CASCADE_ROW_THREADS 512
#endif
constexpr int kRowThreads = CASCADE_ROW_THREADS;  // route / combine: one CTA per token row
constexpr int kRowG = 8192 / (8 * kRowThreads);   // 8-column groups per thread (d <= 8192)
constexpr int kRowWarps = kRowThreads / 32;
constexpr int kRouteStageBytes = 96 * 1024; // router weights staged in smem up to this size

// Eight consecutive columns k0..k0+7 (k0 % 8 == 0) of token t, as packed
// bf16 pairs, into a B-operand buffer with wide stores: one 16-byte store
// in the UMMA B layout (the 8 columns are contiguous there), four 4-byte
// stores in the mma.sync B-frag layout (pair 2q goes to lane g*4+q).
// Narrow scattered 2-byte stores from a single CTA cost ~4 us per row.
__device__ __forceinline__ void store_b8(uint16_t* dst, bool umma, int t, int k0, const uint32_t (&w)[4]) {
    if (umma) {
        *reinterpret_cast<uint4*>(dst + umma_b_index(t, k0)) = make_uint4(w[0], w[1], w[2], w[3]);
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) *reinterpret_cast<uint32_t*>(dst + bfrag_index(t, k0 + 2 * q)) = w[q];
    }
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    return (uint32_t)bf16_bits(lo) | ((uint32_t)bf16_bits(hi) << 16);
}
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// grid = T independent CTAs, CTA t = token t:
//  * before griddepcontrol.wait (independent of the predecessor): the
//    router weights (when they fit, e.g. Mixtral's 72 KB) are staged in
//    shared memory and the norm weights loaded;
//  * then 1/rms of the token's residual row, the bf16 MoE input (B-frag
//    for the expert GEMVs, and fp32 in smem), router logits (warp per
//    expert row, fixed lane order), softmax and top-k (larger logit first,
//    lower expert index on ties), gate weights (renormalised over the k for
//    Mixtral).
// The expert union over the T tokens is built by each CTA of the expert
// GEMVs from topk_id (gemv.cuh build_union), so the router needs no
// cross-CTA synchronisation: a cluster barrier costs a GPU-scope memory
// fence (MEMBAR.ALL.GPU, ~1 us) per use.
__global__ void __launch_bounds__(kRowThreads, 1) moe_route_kernel(RouteParams p) {
    extern __shared__ __align__(16) unsigned char rsm[];
    float* xs = reinterpret_cast<float*>(rsm);                         // [d] MoE input (bf16 values)
    const uint16_t* wsm = reinterpret_cast<const uint16_t*>(rsm + (size_t)p.d * 4);  // staged router rows
    __shared__ float red[32];
    __shared__ float s_lg[kMaxExperts + 1];
    // Large routers (OLMoE 64 x 2048, Qwen 61 x 2048) are split over a
    // cluster of C CTAs per token: rank r stages rows [row_lo, row_hi) in
    // its shared memory before the dependency wait, computes their logits
    // into rank 0's shared memory (DSMEM), and rank 0 finishes the token
    // after one cluster barrier (no global stores are pending at the
    // barrier, so its release fence is cheap).
    const int C = p.C > 1 ? p.C : 1;
    const int t = blockIdx.x / C;
    const int crank = blockIdx.x - t * C;
    const int n_rows = p.E + (p.shared_gate ? 1 : 0);
    const int row_lo = n_rows * crank / C, row_hi = n_rows * (crank + 1) / C;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool staged = p.stage_w != 0 || C > 1;
    namespace cg = cooperative_groups;
    // Cluster: every rank must have started before another rank writes its
    // shared memory (DSMEM).  Arrive now, wait just before the first remote
    // write; the wait overlaps the weight staging and the norm.
    if (C > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    // ---- independent of the predecessor
    if (staged) {
        const uint4* src = reinterpret_cast<const uint4*>(p.router_w + (size_t)row_lo * p.d);
        uint4* dst = reinterpret_cast<uint4*>(rsm + (size_t)p.d * 4);
        for (int i = threadIdx.x; i < (row_hi - row_lo) * p.d / 8; i += kRowThreads) dst[i] = __ldg(src + i);
    }
    constexpr int kPreIt = 8;  // 256 columns per chunk
    uint4 pre0[kPreIt];
    if (!staged) {
        // first chunk of this warp's first row: a constant, requested now
        const uint4* w0 = reinterpret_cast<const uint4*>(p.router_w + (size_t)(warp < n_rows ? warp : 0) * p.d);
#pragma unroll
        for (int j = 0; j < kPreIt; ++j) {
            const int i = lane + 32 * j;
            pre0[j] = i < p.d / 8 ? __ldg(w0 + i) : make_uint4(0, 0, 0, 0);
        }
    }
    uint4 nw[kRowG];  // norm weights of this thread's 8-column groups
#pragma unroll
    for (int j = 0; j < kRowG; ++j) {
        const int c = threadIdx.x + j * kRowThreads;
        nw[j] = c < (p.d >> 3) ? __ldg(reinterpret_cast<const uint4*>(p.norm_w) + c) : make_uint4(0, 0, 0, 0);
    }
    griddep_wait();
    griddep_launch_early(kLateRoute);
    CTA_TRACE(p.trace);
    if (t == 0 && crank == 0 && threadIdx.x == 0 && p.stamp) *p.stamp = globaltimer();
    if (p.ffn_ready != nullptr && blockIdx.x == 0)
        for (int i = threadIdx.x; i < p.n_ready; i += blockDim.x) p.ffn_ready[(long long)i * kReadyStride] = 0;
    phase_stamp(p.trace, 0);
    // ---- norm: thread owns groups of 8 consecutive columns (wide loads/stores)
    const float4* x4 = reinterpret_cast<const float4*>(p.x + (long long)t * p.d);
    constexpr int kG = kRowG;
    const int n8 = p.d >> 3;
    float4 xv[kG][2];
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < kG; ++j) {
        const int c = threadIdx.x + j * kRowThreads;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            xv[j][h] = c < n8 ? x4[2 * c + h] : make_float4(0.f, 0.f, 0.f, 0.f);
            ss += xv[j][h].x * xv[j][h].x + xv[j][h].y * xv[j][h].y + xv[j][h].z * xv[j][h].z +
                  xv[j][h].w * xv[j][h].w;
        }
    }
    ss = block_sum(ss, red);
    const float rinv = 1.0f / sqrtf(ss / (float)p.d + p.eps);
#pragma unroll
    for (int j = 0; j < kG; ++j) {
        const int c = threadIdx.x + j * kRowThreads;
        if (c >= n8) continue;
        const float4 a = xv[j][0], b = xv[j][1];
        uint32_t w[4];
        w[0] = pack_bf16((a.x * rinv) * bf16_lo(nw[j].x), (a.y * rinv) * bf16_hi(nw[j].x));
        w[1] = pack_bf16((a.z * rinv) * bf16_lo(nw[j].y), (a.w * rinv) * bf16_hi(nw[j].y));
        w[2] = pack_bf16((b.x * rinv) * bf16_lo(nw[j].z), (b.y * rinv) * bf16_hi(nw[j].z));
        w[3] = pack_bf16((b.z * rinv) * bf16_lo(nw[j].w), (b.w * rinv) * bf16_hi(nw[j].w));
        if (C == 1) {
            store_b8(p.xn_bfrag, false, t, 8 * c, w);
            if (p.tap_xn) *reinterpret_cast<uint4*>(p.tap_xn + (long long)t * p.d + 8 * c) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        float4* xs4 = reinterpret_cast<float4*>(xs + 8 * c);
        xs4[0] = make_float4(bf16_lo(w[0]), bf16_hi(w[0]), bf16_lo(w[1]), bf16_hi(w[1]));
        xs4[1] = make_float4(bf16_lo(w[2]), bf16_hi(w[2]), bf16_lo(w[3]), bf16_hi(w[3]));
    }
    if (p.zero_nonlocal && C == 1) {
        // EP: every (token, rank) row is written by exactly one rank's down
        // GEMV; the others must contribute exact zeros to the all-reduce.
        float4* y = reinterpret_cast<float4*>(p.ycontrib + (long long)t * (p.k + p.S) * p.d);
        for (int i = threadIdx.x; i < (p.k + p.S) * p.d / 4; i += kRowThreads) y[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    phase_stamp(p.trace, 1);
    // ---- router logits: warp per expert row, lane-strided 8-element pieces
    //      (the same per-lane order for staged and global rows)
    auto dot8 = [&](const uint4& w, int i, float acc) {
        const float4 a = reinterpret_cast<const float4*>(xs)[2 * i];
        const float4 b = reinterpret_cast<const float4*>(xs)[2 * i + 1];
        acc = fmaf(a.x, __uint_as_float(w.x << 16), acc);
        acc = fmaf(a.y, __uint_as_float(w.x & 0xFFFF0000u), acc);
        acc = fmaf(a.z, __uint_as_float(w.y << 16), acc);
        acc = fmaf(a.w, __uint_as_float(w.y & 0xFFFF0000u), acc);
        acc = fmaf(b.x, __uint_as_float(w.z << 16), acc);
        acc = fmaf(b.y, __uint_as_float(w.z & 0xFFFF0000u), acc);
        acc = fmaf(b.z, __uint_as_float(w.w << 16), acc);
        acc = fmaf(b.w, __uint_as_float(w.w & 0xFFFF0000u), acc);
        return acc;
    };
    if (C > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    float* lg0 = C > 1 ? cg::this_cluster().map_shared_rank(s_lg, 0) : s_lg;  // rank 0's logits
    auto emit = [&](int e, float acc) {
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            lg0[e] = acc;
            if (C == 1) p.logits[t * (p.E + 1) + e] = acc;
        }
    };
    // n8 = d / 8 column groups (declared with the norm)
    if (staged) {
        for (int e = row_lo + warp; e < row_hi; e += kRowWarps) {
            const uint4* w4 = reinterpret_cast<const uint4*>(wsm + (size_t)(e - row_lo) * p.d);
            float acc = 0.f;
#pragma unroll 8
            for (int i = lane; i < n8; i += 32) acc = dot8(w4[i], i, acc);
            emit(e, acc);
        }
    } else {
        // rows from global, two per warp at a time with every load of a
        // 256-column chunk issued before any FMA; the first chunk of the
        // first row was requested before griddepcontrol.wait (pre0).
        bool first = true;
        for (int e0 = warp; e0 < n_rows; e0 += 2 * kRowWarps) {
            const int e1 = e0 + kRowWarps;
            const bool has1 = e1 < n_rows;
            const uint4* w0 = reinterpret_cast<const uint4*>(p.router_w + (size_t)e0 * p.d);
            const uint4* w1 = reinterpret_cast<const uint4*>(p.router_w + (size_t)(has1 ? e1 : e0) * p.d);
            float a0 = 0.f, a1 = 0.f;
            for (int c0 = 0; c0 < n8; c0 += 32 * kPreIt) {
                uint4 r0[kPreIt], r1[kPreIt];
                if (first) {
#pragma unroll
                    for (int j = 0; j < kPreIt; ++j) {
                        const int i = c0 + lane + 32 * j;
                        r0[j] = pre0[j];
                        r1[j] = i < n8 ? __ldg(w1 + i) : make_uint4(0, 0, 0, 0);
                    }
                    first = false;
                } else {
#pragma unroll
                    for (int j = 0; j < kPreIt; ++j) {
                        const int i = c0 + lane + 32 * j;
                        r0[j] = i < n8 ? __ldg(w0 + i) : make_uint4(0, 0, 0, 0);
                        r1[j] = i < n8 ? __ldg(w1 + i) : make_uint4(0, 0, 0, 0);
                    }
                }
#pragma unroll
                for (int j = 0; j < kPreIt; ++j) {
                    const int i = c0 + lane + 32 * j;
                    if (i < n8) {
                        a0 = dot8(r0[j], i, a0);
                        a1 = dot8(r1[j], i, a1);
                    }
                }
            }
            emit(e0, a0);
            if (has1) emit(e1, a1);
        }
    }
    if (C > 1) {
        cg::this_cluster().sync();  // every rank's logits are in rank 0's s_lg
        if (crank != 0) return;
        // rank 0: the deferred global writes (router logits, MoE input, EP zeros)
        for (int e = threadIdx.x; e < n_rows; e += kRowThreads) p.logits[t * (p.E + 1) + e] = s_lg[e];
#pragma unroll
        for (int j = 0; j < kG; ++j) {
            const int c = threadIdx.x + j * kRowThreads;
            if (c >= n8) continue;
            const float4* xs4 = reinterpret_cast<const float4*>(xs + 8 * c);
            const float4 a = xs4[0], b = xs4[1];
            uint32_t w[4] = {pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y), pack_bf16(b.z, b.w)};
            store_b8(p.xn_bfrag, false, t, 8 * c, w);
            if (p.tap_xn) *reinterpret_cast<uint4*>(p.tap_xn + (long long)t * p.d + 8 * c) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        if (p.zero_nonlocal) {
            float4* y = reinterpret_cast<float4*>(p.ycontrib + (long long)t * (p.k + p.S) * p.d);
            for (int i = threadIdx.x; i < (p.k + p.S) * p.d / 4; i += kRowThreads) y[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    __syncthreads();
    phase_stamp(p.trace, 2);
    if (p.par_topk) {
        // ---- top-k by rank: thread i counts the experts ordered before i
        //      (larger logit first, lower index on ties); the k first ranks
        //      are the selection in order.  The serial selection below costs
        //      k rounds of 10 dependent shuffles (~2 us for OLMoE's k = 8).
        __shared__ int s_sel[kMaxTopK];
        if ((int)threadIdx.x < p.E) {
            const int i = threadIdx.x;
            const float vi = s_lg[i];
            int rk = 0;
#pragma unroll 8
            for (int j = 0; j < p.E; ++j) {
                const float vj = s_lg[j];
                rk += (vj > vi || (vj == vi && j < i)) ? 1 : 0;
            }
            if (rk < p.k) s_sel[rk] = i;
        }
        __syncthreads();
        if (warp == 0) {
            float m = -INFINITY;
#pragma unroll
            for (int q = 0; q < kMaxExperts / 32; ++q) {
                const int ei = lane + 32 * q;
                m = fmaxf(m, ei < p.E ? s_lg[ei] : -INFINITY);
            }
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            float z = 0.f;
#pragma unroll
            for (int q = 0; q < kMaxExperts / 32; ++q)
                if (lane + 32 * q < p.E) z += __expf(s_lg[lane + 32 * q] - m);
            for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
            float zk = 0.f, my_e = 0.f;
            for (int r = 0; r < p.k; ++r) {  // same order as the serial selection: r = 0..k-1
                const float ex = __expf(s_lg[s_sel[r]] - m);
                zk += ex;
                if (lane == r) my_e = ex;
            }
            const float den = p.renorm ? zk : z;
            if (lane < p.k) {
                p.topk_id[t * p.k + lane] = s_sel[lane];
                p.topk_w[t * p.k + lane] = my_e / den;
            }
            if (lane == 0) p.gsh[t] = p.shared_gate ? 1.0f / (1.0f + __expf(-s_lg[p.E])) : 1.0f;
        }
        phase_stamp(p.trace, 3);
        return;
    }
    // ---- softmax + top-k of this token (warp 0)
    if (warp == 0) {
        const int tt = t;
        const float* lg = s_lg;
        float v[kMaxExperts / 32];
        float m = -INFINITY;
#pragma unroll
        for (int q = 0; q < kMaxExperts / 32; ++q) {
            const int ei = lane + 32 * q;
            v[q] = ei < p.E ? lg[ei] : -INFINITY;
            m = fmaxf(m, v[q]);
        }
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float z = 0.f;
#pragma unroll
        for (int q = 0; q < kMaxExperts / 32; ++q)
            if (lane + 32 * q < p.E) z += __expf(v[q] - m);
        for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
        float zk = 0.f;
        float my_e = 0.f;  // lane r keeps the r-th choice
        int my_i = 0;
        for (int r = 0; r < p.k; ++r) {
            float bv = -INFINITY;
            int bi = 0x7fffffff;
#pragma unroll
            for (int q = 0; q < kMaxExperts / 32; ++q) {
                const int ei = lane + 32 * q;
                if (ei < p.E && (v[q] > bv || (v[q] == bv && ei < bi))) {
                    bv = v[q];
                    bi = ei;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ov > bv || (ov == bv && oi < bi)) {
                    bv = ov;
                    bi = oi;
                }
            }
#pragma unroll
            for (int q = 0; q < kMaxExperts / 32; ++q)
                if (lane + 32 * q == bi) v[q] = -INFINITY;
            const float ex = __expf(bv - m);
            zk += ex;  // same order on every lane: r = 0..k-1
            if (lane == r) {
                my_e = ex;
                my_i = bi;
            }
        }
        const float den = p.renorm ? zk : z;
        if (lane < p.k) {
            p.topk_id[tt * p.k + lane] = my_i;
            p.topk_w[tt * p.k + lane] = my_e / den;
        }
        if (lane == 0) p.gsh[tt] = p.shared_gate ? 1.0f / (1.0f + __expf(-lg[p.E])) : 1.0f;
    }
    phase_stamp(p.trace, 3);
}

struct CombineParams {
    float* x;                    // residual [T][d] (updated in place)
    const float* ycontrib;       // [T][k+S][d]
    const float* topk_w;         // [T][k]
    const float* gsh;            // [T]
    const uint16_t* norm_w;      // next norm weights [d]
    uint16_t* xn_bfrag;          // out
    int umma;                    // xn_bfrag in the UMMA B layout (dense tcgen05 GEMVs) instead of B-frag
    float* tap_moe;              // optional [T][d] (the MoE contribution)
    uint16_t* tap_xn;            // optional [T][d] next-norm output
    float* tap_x;                // optional [T][d] residual after the add
    int T, d, k, S;
    float eps;
    const void* pf;              // next layer's QKV weights -> L2
    unsigned long long pf_bytes;
    unsigned long long* trace;
};

// grid = T CTAs of 512 threads, one token row each; thread owns groups of
// 8 consecutive columns (d <= 8192), every load issued up front:
// residual += sum_r w[t][r] * Y[t][r] (+ shared-gate * sum_b Y[t][k+b]) in
// fixed order, then the next RMSNorm (next layer's attention input, or the
// final norm) of the updated row, stored with 16-byte stores.
__global__ void __launch_bounds__(kRowThreads, 1) moe_combine_kernel(CombineParams p) {
    __shared__ float red[32];
    const int t = blockIdx.x;
    constexpr int kG = kRowG;  // 8-column groups per thread
    const int n8 = p.d >> 3;
    uint4 nw[kG];          // norm weights: constants, loaded before the dependency wait
#pragma unroll
    for (int j = 0; j < kG; ++j) {
        const int c = threadIdx.x + j * kRowThreads;
        nw[j] = c < n8 ? __ldg(reinterpret_cast<const uint4*>(p.norm_w) + c) : make_uint4(0, 0, 0, 0);
    }
    griddep_wait();
    griddep_launch_early(kLateCombine);
    CTA_TRACE(p.trace);
    prefetch_l2(p.pf, p.pf_bytes);
    phase_stamp(p.trace, 0);
    const float4* y4 = reinterpret_cast<const float4*>(p.ycontrib + (long long)t * (p.k + p.S) * p.d);
    float4* x4 = reinterpret_cast<float4*>(p.x + (long long)t * p.d);
    const int n4 = p.d >> 2;
    const int nr = p.k + p.S;
    const float g = p.gsh[t];
    float wk[8];  // the token's gate weights (rows 0..k-1 of its contribution list)
#pragma unroll
    for (int q = 0; q < 8; ++q) wk[q] = q < p.k ? p.topk_w[t * p.k + q] : 0.f;
    float4 nx[kG][2];
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < kG; ++j) {
        const int c = threadIdx.x + j * kRowThreads;
        if (c >= n8) continue;
        // every load of the group issued before any math: both halves of the
        // residual and of up to kMaxR contribution rows (sums in row order)
        constexpr int kMaxR = 8;
        float4 x0v[2], yb[kMaxR][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) x0v[h] = x4[2 * c + h];
#pragma unroll
        for (int q = 0; q < kMaxR; ++q)
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (q < nr) yb[q][h] = y4[(long long)q * n4 + 2 * c + h];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int i = 2 * c + h;
            const float4 x0 = x0v[h];
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f), sh = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int q = 0; q < kMaxR; ++q) {
                if (q >= nr) break;
                if (q < p.k) {
                    const float w = wk[q];
                    acc.x += w * yb[q][h].x;
                    acc.y += w * yb[q][h].y;
                    acc.z += w * yb[q][h].z;
                    acc.w += w * yb[q][h].w;
                } else {
                    sh.x += yb[q][h].x;
                    sh.y += yb[q][h].y;
                    sh.z += yb[q][h].z;
                    sh.w += yb[q][h].w;
                }
            }
            for (int r0 = kMaxR; r0 < nr; r0 += 4) {  // rows beyond kMaxR: batches of 4, row order
                float4 yr[4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (r0 + q < nr) yr[q] = y4[(long long)(r0 + q) * n4 + i];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int r = r0 + q;
                    if (r < p.k) {
                        const float w = p.topk_w[t * p.k + r];
                        acc.x += w * yr[q].x;
                        acc.y += w * yr[q].y;
                        acc.z += w * yr[q].z;
                        acc.w += w * yr[q].w;
                    } else if (r < nr) {
                        sh.x += yr[q].x;
                        sh.y += yr[q].y;
                        sh.z += yr[q].z;
                        sh.w += yr[q].w;
                    }
                }
            }
            if (p.S > 0) {
                acc.x += g * sh.x;
                acc.y += g * sh.y;
                acc.z += g * sh.z;
                acc.w += g * sh.w;
            }
            if (p.tap_moe) reinterpret_cast<float4*>(p.tap_moe + (long long)t * p.d)[i] = acc;
            const float4 v = make_float4(x0.x + acc.x, x0.y + acc.y, x0.z + acc.z, x0.w + acc.w);
            nx[j][h] = v;
            x4[i] = v;
            if (p.tap_x) reinterpret_cast<float4*>(p.tap_x + (long long)t * p.d)[i] = v;
            ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
        }
    }
    phase_stamp(p.trace, 1);
    ss = block_sum(ss, red);
    phase_stamp(p.trace, 2);
    const float rinv = 1.0f / sqrtf(ss / (float)p.d + p.eps);
#pragma unroll
    for (int j = 0; j < kG; ++j) {
        const int c = threadIdx.x + j * kRowThreads;
        if (c >= n8) continue;
        const float4 a = nx[j][0], b = nx[j][1];
        uint32_t w[4];
        w[0] = pack_bf16((a.x * rinv) * bf16_lo(nw[j].x), (a.y * rinv) * bf16_hi(nw[j].x));
        w[1] = pack_bf16((a.z * rinv) * bf16_lo(nw[j].y), (a.w * rinv) * bf16_hi(nw[j].y));
        w[2] = pack_bf16((b.x * rinv) * bf16_lo(nw[j].z), (b.y * rinv) * bf16_hi(nw[j].z));
        w[3] = pack_bf16((b.z * rinv) * bf16_lo(nw[j].w), (b.w * rinv) * bf16_hi(nw[j].w));
        store_b8(p.xn_bfrag, p.umma != 0, t, 8 * c, w);
        if (p.tap_xn) *reinterpret_cast<uint4*>(p.tap_xn + (long long)t * p.d + 8 * c) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    phase_stamp(p.trace, 3);
}

// Step entry: token embedding + first RMSNorm + the step's RoPE table;
// stamps the step start.
struct StepParams {            // H2D-copied at the head of every step graph
    int32_t mode;              // 0 verify (row 0 = pending token), 1 prefill (all given)
    int32_t commit;            // 1: advance the cache; 0: re-verify the same context
    int32_t T;
    int32_t pad;
    int32_t tokens[kMaxT];
    double t_base_ns;
    double draft_ns;
};

struct DevState {
    int32_t cache_len;
    int32_t pending;
    int32_t steps;
    int32_t pad;
};

struct EmbedParams {
    const StepParams* sp;
    const DevState* st;
    const uint16_t* embed;       // [V][d]
    const uint16_t* norm_w;      // layer-0 attention norm
    float* x;                    // out residual [T][d]
    uint16_t* xn_bfrag;          // out
    int* tokens_used;            // out [T]
    float2* rope;                // out [T][hd/2] (cos, sin) at position ctx + t
    unsigned long long* stamp;   // step start
    float* tap_x;                // optional
    uint16_t* tap_xn;            // optional
    int T, d, hd;
    double rope_theta;
    float eps;
    const void* pf;              // layer-0 QKV weights -> L2
    unsigned long long pf_bytes;
    unsigned long long* trace;
    int umma;                    // xn_bfrag in the UMMA B layout
};

__global__ void __launch_bounds__(kRouteThreads) embed_norm_kernel(EmbedParams p) {
    griddep_wait();
    griddep_launch_early(kLateEmbed);
    CTA_TRACE(p.trace);
    prefetch_l2(p.pf, p.pf_bytes);
    __shared__ float red[32];
    const int t = blockIdx.x;
    if (t == 0 && threadIdx.x == 0) *p.stamp = globaltimer();
    const int tok = (p.sp->mode == 0 && t == 0) ? p.st->pending : p.sp->tokens[t];
    if (threadIdx.x == 0) p.tokens_used[t] = tok;
    const int pos = p.st->cache_len + t;
    for (int i = threadIdx.x; i < p.hd / 2; i += blockDim.x) {
        // angle in fp64: exact to fp32 rounding at any context length
        const double inv = pow(p.rope_theta, -2.0 * (double)i / (double)p.hd);
        double sn, cs;
        sincos((double)pos * inv, &sn, &cs);
        p.rope[t * (p.hd / 2) + i] = make_float2((float)cs, (float)sn);
    }
    // thread owns groups of 8 consecutive columns: 16-byte embedding loads,
    // 32-byte residual stores, 16-byte B-layout stores (d <= 8192)
    constexpr int kEG = 4;
    const int n8 = p.d >> 3;
    const uint4* e8 = reinterpret_cast<const uint4*>(p.embed + (long long)tok * p.d);
    float4* x4 = reinterpret_cast<float4*>(p.x + (long long)t * p.d);
    uint4 ev[kEG], nw[kEG];
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < kEG; ++j) {
        const int c = threadIdx.x + j * kRouteThreads;
        ev[j] = c < n8 ? __ldg(e8 + c) : make_uint4(0, 0, 0, 0);
        nw[j] = c < n8 ? __ldg(reinterpret_cast<const uint4*>(p.norm_w) + c) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < kEG; ++j) {
        const int c = threadIdx.x + j * kRouteThreads;
        if (c >= n8) continue;
        const float4 a = make_float4(bf16_lo(ev[j].x), bf16_hi(ev[j].x), bf16_lo(ev[j].y), bf16_hi(ev[j].y));
        const float4 b = make_float4(bf16_lo(ev[j].z), bf16_hi(ev[j].z), bf16_lo(ev[j].w), bf16_hi(ev[j].w));
        x4[2 * c] = a;
        x4[2 * c + 1] = b;
        if (p.tap_x) {
            reinterpret_cast<float4*>(p.tap_x + (long long)t * p.d)[2 * c] = a;
            reinterpret_cast<float4*>(p.tap_x + (long long)t * p.d)[2 * c + 1] = b;
        }
        ss += a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w + b.x * b.x + b.y * b.y + b.z * b.z + b.w * b.w;
    }
    ss = block_sum(ss, red);
    const float rinv = 1.0f / sqrtf(ss / (float)p.d + p.eps);
#pragma unroll
    for (int j = 0; j < kEG; ++j) {
        const int c = threadIdx.x + j * kRouteThreads;
        if (c >= n8) continue;
        uint32_t w[4];
        const uint32_t ew[4] = {ev[j].x, ev[j].y, ev[j].z, ev[j].w};
        const uint32_t ww[4] = {nw[j].x, nw[j].y, nw[j].z, nw[j].w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
            w[q] = pack_bf16((bf16_lo(ew[q]) * rinv) * bf16_lo(ww[q]), (bf16_hi(ew[q]) * rinv) * bf16_hi(ww[q]));
        store_b8(p.xn_bfrag, p.umma != 0, t, 8 * c, w);
        if (p.tap_xn) *reinterpret_cast<uint4*>(p.tap_xn + (long long)t * p.d + 8 * c) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

}  // namespace cascade
