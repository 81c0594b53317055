// moe.cuh — router, expert union and expert combine (SURVEY.md §8(a2)
// stages K1/K2 and the epilogue of K3).
//
// moe_route_kernel (grid = T CTAs, one per in-flight token):
//   1. RMSNorm of the residual row -> bf16 MoE input, written in B-frag
//      layout for the expert GEMVs.
//   2. Router logits (E routed rows, plus the Qwen shared-expert gate row)
//      from the bf16 input and bf16 router weights, fp32 accumulate.
//   3. The last CTA to finish (atomic ticket) routes every token: softmax,
//      top-k (ties -> lower expert index), gate weights (renormalised for
//      Mixtral), then the expert union: OR of per-token masks, ascending
//      unique-expert list, per-expert token ranks.  This is the real
//      counterpart of the reference's stand-ins draw_expert_set /
//      sample_active_experts (expert_model.hpp:100-139): union = distinct
//      routed experts, shared blocks always active on top.
// moe_combine_kernel (grid = T): residual += sum_r w[t][r] * Y[t][r]
//   (+ shared-gate * sum_b Y[t][k+b]) in fixed order, then the next
//   RMSNorm (next layer's attention input, or the final norm).
#pragma once

#include "common.cuh"

namespace cascade {

constexpr int kRouteThreads = 256;
constexpr int kMaxExperts = 128;   // expert_model.hpp:96 (kMaxRoutedExperts)
constexpr int kMaxTopK = 16;

struct RouteParams {
    const float* x;              // residual [T][d]
    const uint16_t* norm_w;      // [d] bf16
    const uint16_t* router_w;    // [E + shared_gate][d] bf16
    uint16_t* xn_bfrag;          // out: MoE input, B-frag
    float* logits;               // out: [T][E+1]
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
};

__global__ void __launch_bounds__(kRouteThreads) moe_route_kernel(RouteParams p) {
    __shared__ float red[32];
    __shared__ int s_last;
    extern __shared__ float xs[];  // [d] normalised input (bf16 values as fp32)
    const int t = blockIdx.x;
    if (t == 0 && threadIdx.x == 0 && p.stamp) *p.stamp = globaltimer();
    const float* x = p.x + (long long)t * p.d;
    float ss = 0.f;
    for (int i = threadIdx.x; i < p.d; i += blockDim.x) ss += x[i] * x[i];
    ss = block_sum(ss, red);
    const float rinv = 1.0f / sqrtf(ss / (float)p.d + p.eps);
    for (int i = threadIdx.x; i < p.d; i += blockDim.x) {
        const float v = (x[i] * rinv) * bits_to_f32(p.norm_w[i]);
        const uint16_t b = bf16_bits(v);
        p.xn_bfrag[bfrag_index(t, i)] = b;
        if (p.tap_xn) p.tap_xn[(long long)t * p.d + i] = b;
        xs[i] = bits_to_f32(b);
    }
    __syncthreads();
    const int n_rows = p.E + (p.shared_gate ? 1 : 0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = warp; e < n_rows; e += kRouteThreads / 32) {
        const uint32_t* w2 = reinterpret_cast<const uint32_t*>(p.router_w + (long long)e * p.d);
        float acc = 0.f;
        for (int i = lane; i < p.d / 2; i += 32) {
            const uint32_t ww = __ldg(w2 + i);
            acc = fmaf(xs[2 * i], __uint_as_float(ww << 16), acc);
            acc = fmaf(xs[2 * i + 1], __uint_as_float(ww & 0xFFFF0000u), acc);
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) p.logits[t * (p.E + 1) + e] = acc;
    }
    if (p.zero_nonlocal) {
        // EP: every (token, rank) row is written by exactly one rank's down
        // GEMV; the others must contribute exact zeros to the all-reduce.
        float* y = p.ycontrib + (long long)t * (p.k + p.S) * p.d;
        for (int i = threadIdx.x; i < (p.k + p.S) * p.d; i += blockDim.x) y[i] = 0.f;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(p.ticket, 1) == p.T - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();

    // ---- routing of all tokens (last CTA) ----
    __shared__ unsigned long long masks[kMaxT][2];
    for (int tt = warp; tt < p.T; tt += kRouteThreads / 32) {
        const float* lg = p.logits + tt * (p.E + 1);
        float v[kMaxExperts / 32];
        float m = -INFINITY;
#pragma unroll
        for (int q = 0; q < kMaxExperts / 32; ++q) {
            const int e = lane + 32 * q;
            v[q] = e < p.E ? __ldcg(lg + e) : -INFINITY;
            m = fmaxf(m, v[q]);
        }
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float z = 0.f;
#pragma unroll
        for (int q = 0; q < kMaxExperts / 32; ++q)
            if (lane + 32 * q < p.E) z += __expf(v[q] - m);
        for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
        unsigned long long m0 = 0, m1 = 0;
        float chosen_e[kMaxTopK];
        int chosen_i[kMaxTopK];
        for (int r = 0; r < p.k; ++r) {
            // warp argmax: larger logit first, lower index on ties
            float bv = -INFINITY;
            int bi = 0x7fffffff;
#pragma unroll
            for (int q = 0; q < kMaxExperts / 32; ++q) {
                const int e = lane + 32 * q;
                if (e < p.E && (v[q] > bv || (v[q] == bv && e < bi))) {
                    bv = v[q];
                    bi = e;
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
            chosen_e[r] = __expf(bv - m);
            chosen_i[r] = bi;
            if (bi < 64) m0 |= 1ull << bi;
            else m1 |= 1ull << (bi - 64);
        }
        if (lane == 0) {
            float zk = 0.f;
            for (int r = 0; r < p.k; ++r) zk += chosen_e[r];
            const float den = p.renorm ? zk : z;
            for (int r = 0; r < p.k; ++r) {
                p.topk_id[tt * p.k + r] = chosen_i[r];
                p.topk_w[tt * p.k + r] = chosen_e[r] / den;
            }
            float g = 1.0f;
            if (p.shared_gate) g = 1.0f / (1.0f + __expf(-__ldcg(lg + p.E)));
            p.gsh[tt] = g;
            masks[tt][0] = m0;
            masks[tt][1] = m1;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long u0 = 0, u1 = 0;
        for (int tt = 0; tt < p.T; ++tt) {
            u0 |= masks[tt][0];
            u1 |= masks[tt][1];
        }
        *p.union_size = __popcll(u0) + __popcll(u1);
        int n = 0;
        for (int e = p.e_lo; e < p.e_hi; ++e) {
            const bool on = e < 64 ? ((u0 >> e) & 1ull) : ((u1 >> (e - 64)) & 1ull);
            if (!on) continue;
            p.list[n] = e - p.e_lo;
            for (int tt = 0; tt < kMaxT; ++tt) {
                int rank = -1;
                if (tt < p.T)
                    for (int r = 0; r < p.k; ++r)
                        if (p.topk_id[tt * p.k + r] == e) rank = r;
                p.route_rank[n * kMaxT + tt] = rank;
            }
            ++n;
        }
        const int n_local_routed = p.e_hi - p.e_lo;
        int lb = 0;
        for (int b = 0; b < p.S; ++b) {
            if (b % p.ep_size != p.ep_rank) continue;
            p.list[n] = n_local_routed + lb;
            for (int tt = 0; tt < kMaxT; ++tt) p.route_rank[n * kMaxT + tt] = tt < p.T ? p.k + b : -1;
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
    float* tap_moe;              // optional [T][d] (the MoE contribution)
    uint16_t* tap_xn;            // optional [T][d] next-norm output
    float* tap_x;                // optional [T][d] residual after the add
    int T, d, k, S;
    float eps;
};

__global__ void __launch_bounds__(kRouteThreads) moe_combine_kernel(CombineParams p) {
    __shared__ float red[32];
    const int t = blockIdx.x;
    float* x = p.x + (long long)t * p.d;
    const float* y = p.ycontrib + (long long)t * (p.k + p.S) * p.d;
    const float g = p.gsh[t];
    float w[kMaxTopK];
    for (int r = 0; r < p.k; ++r) w[r] = p.topk_w[t * p.k + r];
    float ss = 0.f;
    for (int i = threadIdx.x; i < p.d; i += blockDim.x) {
        float acc = 0.f;
        for (int r = 0; r < p.k; ++r) acc += w[r] * y[(long long)r * p.d + i];
        if (p.S > 0) {
            float sh = 0.f;
            for (int b = 0; b < p.S; ++b) sh += y[(long long)(p.k + b) * p.d + i];
            acc += g * sh;
        }
        if (p.tap_moe) p.tap_moe[(long long)t * p.d + i] = acc;
        const float nx = x[i] + acc;
        x[i] = nx;
        if (p.tap_x) p.tap_x[(long long)t * p.d + i] = nx;
        ss += nx * nx;
    }
    ss = block_sum(ss, red);
    const float rinv = 1.0f / sqrtf(ss / (float)p.d + p.eps);
    for (int i = threadIdx.x; i < p.d; i += blockDim.x) {
        const uint16_t b = bf16_bits((x[i] * rinv) * bits_to_f32(p.norm_w[i]));
        p.xn_bfrag[bfrag_index(t, i)] = b;
        if (p.tap_xn) p.tap_xn[(long long)t * p.d + i] = b;
    }
}

// Step entry: token embedding + first RMSNorm; stamps the step start.
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
    unsigned long long* stamp;   // step start
    float* tap_x;                // optional
    uint16_t* tap_xn;            // optional
    int T, d;
    float eps;
};

__global__ void __launch_bounds__(kRouteThreads) embed_norm_kernel(EmbedParams p) {
    __shared__ float red[32];
    const int t = blockIdx.x;
    if (t == 0 && threadIdx.x == 0) *p.stamp = globaltimer();
    const int tok = (p.sp->mode == 0 && t == 0) ? p.st->pending : p.sp->tokens[t];
    if (threadIdx.x == 0) p.tokens_used[t] = tok;
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
        p.xn_bfrag[bfrag_index(t, i)] = b;
        if (p.tap_xn) p.tap_xn[(long long)t * p.d + i] = b;
    }
}

}  // namespace cascade
