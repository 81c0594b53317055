// moe.cuh — step entry (embedding), router + expert union, expert combine
// (SURVEY.md §8(a2) stages K1/K2 and the epilogue of K3).
//
// moe_route_kernel (grid = T tokens x router-row groups):
//   1. RMSNorm of the residual row -> bf16 MoE input (B-frag layout for the
//      expert GEMVs; written by the row-group-0 CTA of each token).
//   2. Router logits: one warp per router row (E routed rows + the Qwen
//      shared-expert gate row), bf16 weights, fp32 accumulate, all of a
//      lane's 16-byte loads issued before any FMA.
//   3. The last CTA to finish (atomic ticket) routes every token: softmax,
//      top-k (larger logit first, lower expert index on ties), gate weights
//      (renormalised over the k for Mixtral), then the expert union: OR of
//      per-token 128-bit masks, ascending unique-expert list, per-expert
//      token ranks.  This is the real counterpart of the reference's
//      stand-ins draw_expert_set / sample_active_experts
//      (expert_model.hpp:100-139): union = distinct routed experts, shared
//      blocks always active on top.
// moe_combine_kernel (grid = T): residual += sum_r w[t][r] * Y[t][r]
//   (+ shared-gate * sum_b Y[t][k+b]) in fixed order, then the next RMSNorm
//   (next layer's attention input, or the final norm).
#pragma once

#include "common.cuh"
#include "gemv_umma.cuh"

namespace cascade {

constexpr int kRouteThreads = 256;
constexpr int kRouteWarps = kRouteThreads / 32;
constexpr int kMaxExperts = 128;  // expert_model.hpp:96 (kMaxRoutedExperts)
constexpr int kMaxTopK = 16;

// 1/rms of one fp32 row (d % 4 == 0), block-wide.
__device__ __forceinline__ float row_rinv(const float* x, int d, float eps, float* red) {
    float ss = 0.f;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const int n4 = d >> 2;
#pragma unroll 4
    for (int i = threadIdx.x; i < n4; i += blockDim.x) {
        const float4 v = x4[i];
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    ss = block_sum(ss, red);
    return 1.0f / sqrtf(ss / (float)d + eps);
}

struct RouteParams {
    const float* x;              // residual [T][d]
    const uint16_t* norm_w;      // [d] bf16
    const uint16_t* router_w;    // [E + shared_gate][d] bf16
    uint16_t* xn_bfrag;          // out: MoE input, B-frag
    float* logits;               // out: [T][E+1]
    float* logit_part;           // scratch: [T][n_slices][E+1] per-slice partial logits
    int* ticket;                 // zero between launches
    int* topk_id;                // out: [T][k]
    float* topk_w;               // out: [T][k]
    float* gsh;                  // out: [T] shared-expert gate (1 if no gate)
    int* list;                   // out: active local block ids [U + S_local]
    int* count;                  // out: number of active local blocks
    int* route_rank;             // out: [slot][16]
    int* union_size;             // out: unique routed experts this layer (global)
    float* ycontrib;             // [T][k+S][d], zeroed for non-local entries (EP)
    uint16_t* tap_xn;            // optional [T][d]
    int T, d, E, k, S, renorm, shared_gate;
    int e_lo, e_hi;              // local routed experts [e_lo, e_hi)
    int ep_rank, ep_size;        // shared block b lives on rank b % ep_size
    float eps;
    int zero_nonlocal;
    unsigned long long* stamp;   // MoE-block start (CostBreakdown split)
    unsigned long long* trace;
};

constexpr int kRouteSlice = kRouteThreads;  // d columns per CTA (one per thread)
constexpr int kMaxSlices = 32;              // d <= 8192

// grid = (d / kRouteSlice, T).  CTA (slice, t): the router weights of its
// column slice are staged in shared memory BEFORE griddepcontrol.wait (they
// do not depend on the predecessor); after it, 1/rms of token t's full
// residual row (L2), the bf16 MoE input of its slice (written once, B-frag)
// and the slice's partial router logits for every expert row.  The last
// CTA (atomic ticket) sums the partials in slice order and routes all
// tokens: softmax, top-k (larger logit first, lower expert index on ties),
// gate weights (renormalised over the k for Mixtral), then the expert
// union: OR of per-token 128-bit masks, ascending unique-expert list,
// per-expert token ranks.  This is the real counterpart of the
// reference's stand-ins draw_expert_set / sample_active_experts
// (expert_model.hpp:100-139): union = distinct routed experts, shared
// blocks always active on top.
__global__ void __launch_bounds__(kRouteThreads) moe_route_kernel(RouteParams p) {
    extern __shared__ uint16_t wsl[];  // [n_rows][kRouteSlice] router weights of this slice
    __shared__ float red[32];
    __shared__ float wred[kRouteWarps][kMaxExperts + 1];
    __shared__ int s_last;
    __shared__ float s_logits[kMaxT][kMaxExperts + 1];
    __shared__ unsigned long long masks[kMaxT][2];
    const int slice = blockIdx.x, t = blockIdx.y;
    const int n_slices = gridDim.x;
    const int n_rows = p.E + (p.shared_gate ? 1 : 0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = slice * kRouteSlice + threadIdx.x;
    // ---- independent of the predecessor: router + norm weights of the slice
    for (int e = 0; e < n_rows; ++e) wsl[e * kRouteSlice + threadIdx.x] = p.router_w[(long long)e * p.d + c];
    const float nw = bits_to_f32(p.norm_w[c]);
    griddep_wait();
    griddep_launch();
    trace_start(p.trace);
    if (slice == 0 && t == 0 && threadIdx.x == 0 && p.stamp) *p.stamp = globaltimer();
    // ---- 1/rms of the full row (every load issued before the reduction)
    const float* x = p.x + (long long)t * p.d;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    float ss = 0.f;
    for (int i = threadIdx.x; i < (p.d >> 2); i += kRouteThreads) {
        const float4 v = x4[i];
        ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    ss = block_sum(ss, red);
    const float rinv = 1.0f / sqrtf(ss / (float)p.d + p.eps);
    const uint16_t b = bf16_bits((x[c] * rinv) * nw);
    p.xn_bfrag[bfrag_index(t, c)] = b;
    if (p.tap_xn) p.tap_xn[(long long)t * p.d + c] = b;
    const float xv = bits_to_f32(b);
    // ---- partial router logits of the slice (fixed reduction order)
    for (int e = 0; e < n_rows; ++e) {
        float v = xv * bits_to_f32(wsl[e * kRouteSlice + threadIdx.x]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) wred[warp][e] = v;
    }
    if (p.zero_nonlocal) {
        // EP: every (token, rank) row is written by exactly one rank's down
        // GEMV; the others must contribute exact zeros to the all-reduce.
        float* y = p.ycontrib + (long long)t * (p.k + p.S) * p.d;
        for (int r = 0; r < p.k + p.S; ++r) y[(long long)r * p.d + c] = 0.f;
    }
    __syncthreads();
    if (threadIdx.x < n_rows) {
        float v = 0.f;
        for (int w = 0; w < kRouteWarps; ++w) v += wred[w][threadIdx.x];
        p.logit_part[((long long)t * n_slices + slice) * (p.E + 1) + threadIdx.x] = v;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(p.ticket, 1) == (int)(gridDim.x * gridDim.y) - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();

    // ---- routing of all tokens (last CTA)
    for (int q = threadIdx.x; q < p.T * n_rows; q += kRouteThreads) {
        const int tt = q / n_rows, e = q - tt * n_rows;
        float pv[kMaxSlices];
#pragma unroll
        for (int sl = 0; sl < kMaxSlices; ++sl)
            pv[sl] = sl < n_slices ? __ldcg(p.logit_part + ((long long)tt * n_slices + sl) * (p.E + 1) + e) : 0.f;
        float v = 0.f;
#pragma unroll
        for (int sl = 0; sl < kMaxSlices; ++sl)
            if (sl < n_slices) v += pv[sl];
        s_logits[tt][e] = v;
        p.logits[tt * (p.E + 1) + e] = v;
    }
    __syncthreads();
    __shared__ int s_topk[kMaxT * kMaxTopK];
    __shared__ int s_warp_on[kMaxExperts / 32];
    for (int tt = warp; tt < p.T; tt += kRouteWarps) {
        const float* lg = s_logits[tt];
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
        unsigned long long m0 = 0, m1 = 0;
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
            if (bi < 64) m0 |= 1ull << bi;
            else m1 |= 1ull << (bi - 64);
        }
        const float den = p.renorm ? zk : z;
        if (lane < p.k) {
            s_topk[tt * p.k + lane] = my_i;
            p.topk_id[tt * p.k + lane] = my_i;
            p.topk_w[tt * p.k + lane] = my_e / den;
        }
        if (lane == 0) {
            p.gsh[tt] = p.shared_gate ? 1.0f / (1.0f + __expf(-lg[p.E])) : 1.0f;
            masks[tt][0] = m0;
            masks[tt][1] = m1;
        }
    }
    __syncthreads();
    // expert union: thread e owns expert e; ballots give ascending slots
    unsigned long long u0 = 0, u1 = 0;
    for (int tt = 0; tt < p.T; ++tt) {
        u0 |= masks[tt][0];
        u1 |= masks[tt][1];
    }
    const int ue = threadIdx.x;
    const bool in_union = ue < p.E && (ue < 64 ? ((u0 >> ue) & 1ull) : ((u1 >> (ue - 64)) & 1ull));
    const bool local_on = in_union && ue >= p.e_lo && ue < p.e_hi;
    const unsigned ball = __ballot_sync(0xffffffffu, local_on);
    if (lane == 0 && warp < kMaxExperts / 32) s_warp_on[warp] = __popc(ball);
    __syncthreads();
    int base = 0;
    for (int w = 0; w < warp && w < kMaxExperts / 32; ++w) base += s_warp_on[w];
    int n_local = 0;
    for (int w = 0; w < kMaxExperts / 32; ++w) n_local += s_warp_on[w];
    if (local_on) {
        const int slot = base + __popc(ball & ((1u << lane) - 1u));
        p.list[slot] = ue - p.e_lo;
        for (int tt = 0; tt < kMaxT; ++tt) {
            int rank = -1;
            if (tt < p.T)
                for (int r = 0; r < p.k; ++r)
                    if (s_topk[tt * p.k + r] == ue) rank = r;
            p.route_rank[slot * kMaxT + tt] = rank;
        }
    }
    if (threadIdx.x == 0) {
        *p.union_size = __popcll(u0) + __popcll(u1);
        const int n_local_routed = p.e_hi - p.e_lo;
        int n = n_local, lb = 0;
        for (int b2 = 0; b2 < p.S; ++b2) {
            if (b2 % p.ep_size != p.ep_rank) continue;
            p.list[n] = n_local_routed + lb;
            for (int tt = 0; tt < kMaxT; ++tt) p.route_rank[n * kMaxT + tt] = tt < p.T ? p.k + b2 : -1;
            ++n;
            ++lb;
        }
        *p.count = n;
        *p.ticket = 0;
    }
}

struct CombineParams {
    float* x;                    // residual [T][d] (updated in place)
    const float* ycontrib;       // [T][k+S][d]
    const float* topk_w;         // [T][k]
    const float* gsh;            // [T]
    const uint16_t* norm_w;      // next norm weights [d]
    uint16_t* xn_bfrag;          // out
    float* ss_part;              // scratch [T][n_slices] partial sums of squares
    int umma;                    // xn_bfrag in the UMMA B layout (dense tcgen05 GEMVs) instead of B-frag
    int* tok_ticket;             // [T] arrival counters (zero between launches)
    float* tap_moe;              // optional [T][d] (the MoE contribution)
    uint16_t* tap_xn;            // optional [T][d] next-norm output
    float* tap_x;                // optional [T][d] residual after the add
    int T, d, k, S;
    float eps;
    const void* pf;              // next layer's QKV weights -> L2
    unsigned long long pf_bytes;
    unsigned long long* trace;
};

// grid = (d / kRouteSlice, T).  CTA (slice, t): residual += sum_r w[t][r] *
// Y[t][r] (+ shared-gate * sum_b Y[t][k+b]) for its columns in fixed order,
// one column per thread with every load independent; the slice's sum of
// squares goes to ss_part.  The last slice CTA of token t (per-token ticket)
// sums the partials in slice order and writes the next RMSNorm (next
// layer's attention input, or the final norm) for the whole row.
__global__ void __launch_bounds__(kRouteThreads) moe_combine_kernel(CombineParams p) {
    __shared__ float red[32];
    __shared__ int s_last;
    const int slice = blockIdx.x, t = blockIdx.y;
    const int n_slices = gridDim.x;
    const int c = slice * kRouteSlice + threadIdx.x;
    griddep_wait();
    griddep_launch();
    trace_start(p.trace);
    prefetch_l2(p.pf, p.pf_bytes);
    const float* y = p.ycontrib + (long long)t * (p.k + p.S) * p.d + c;
    float* xr = p.x + (long long)t * p.d;
    // all loads first (one round trip), then the fixed-order sums
    float yv[kMaxTopK], wr[kMaxTopK], ys[kMaxTopK];
#pragma unroll
    for (int r = 0; r < kMaxTopK; ++r) {
        if (r < p.k) {
            yv[r] = y[(long long)r * p.d];
            wr[r] = __ldg(p.topk_w + t * p.k + r);
        }
        if (r < p.S) ys[r] = y[(long long)(p.k + r) * p.d];
    }
    const float x0 = xr[c];
    float acc = 0.f;
#pragma unroll
    for (int r = 0; r < kMaxTopK; ++r)
        if (r < p.k) acc += wr[r] * yv[r];
    if (p.S > 0) {
        float sh = 0.f;
#pragma unroll
        for (int b = 0; b < kMaxTopK; ++b)
            if (b < p.S) sh += ys[b];
        acc += __ldg(p.gsh + t) * sh;
    }
    if (p.tap_moe) p.tap_moe[(long long)t * p.d + c] = acc;
    const float nx = x0 + acc;
    xr[c] = nx;
    if (p.tap_x) p.tap_x[(long long)t * p.d + c] = nx;
    const float ss = block_sum(nx * nx, red);
    if (threadIdx.x == 0) p.ss_part[t * n_slices + slice] = ss;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(p.tok_ticket + t, 1) == n_slices - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // every load of the tail issued before any use (one L2 round trip each)
    float xv[kMaxSlices], wv[kMaxSlices], sp[kMaxSlices];
#pragma unroll
    for (int j = 0; j < kMaxSlices; ++j) {
        if (j < n_slices) {
            xv[j] = __ldcg(xr + j * kRouteSlice + threadIdx.x);
            wv[j] = bits_to_f32(p.norm_w[j * kRouteSlice + threadIdx.x]);
            sp[j] = __ldcg(p.ss_part + t * n_slices + j);
        }
    }
    float tot = 0.f;
#pragma unroll
    for (int j = 0; j < kMaxSlices; ++j)
        if (j < n_slices) tot += sp[j];
    const float rinv = 1.0f / sqrtf(tot / (float)p.d + p.eps);
#pragma unroll
    for (int j = 0; j < kMaxSlices; ++j) {
        if (j < n_slices) {
            const int i = j * kRouteSlice + threadIdx.x;
            const uint16_t b = bf16_bits((xv[j] * rinv) * wv[j]);
            p.xn_bfrag[p.umma ? umma_b_index(t, i) : bfrag_index(t, i)] = b;
            if (p.tap_xn) p.tap_xn[(long long)t * p.d + i] = b;
        }
    }
    if (threadIdx.x == 0) p.tok_ticket[t] = 0;
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
    griddep_launch();
    trace_start(p.trace);
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
    const uint16_t* e = p.embed + (long long)tok * p.d;
    float* x = p.x + (long long)t * p.d;
    float ss = 0.f;
    for (int i = threadIdx.x; i < p.d; i += blockDim.x) {
        const float v = bits_to_f32(e[i]);
        x[i] = v;
        if (p.tap_x) p.tap_x[(long long)t * p.d + i] = v;
        ss += v * v;
    }
    ss = block_sum(ss, red);
    const float rinv = 1.0f / sqrtf(ss / (float)p.d + p.eps);
    for (int i = threadIdx.x; i < p.d; i += blockDim.x) {
        const uint16_t b = bf16_bits((x[i] * rinv) * bits_to_f32(p.norm_w[i]));
        p.xn_bfrag[p.umma ? umma_b_index(t, i) : bfrag_index(t, i)] = b;
        if (p.tap_xn) p.tap_xn[(long long)t * p.d + i] = b;
    }
}

}  // namespace cascade
