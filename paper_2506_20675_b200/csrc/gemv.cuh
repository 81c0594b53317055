// gemv.cuh — the weight-streaming engine behind every linear layer of the
// verify step (QKV, O, routed + shared expert gate/up and down, LM head).
//
// Problem shape: Y[T, rows] = X[T, K] * W[rows, K]^T with T = K_spec+1 <= 16
// tokens, i.e. a batch of GEMVs whose cost is the weight bytes (arithmetic
// intensity T flop/B, far below the tensor-core ridge).  The design goal is
// to stream each *active* weight block from HBM exactly once at copy speed:
//
//  * Work = (active block, 64-row super-tile, 16-column k-step).  The flat
//    work range U*n_st*n_ks is split into one contiguous, equal-length range
//    per warp (stream-K), so every SM moves the same number of bytes no
//    matter how many experts the router activated (U is read from device
//    memory: the same captured graph serves every routing outcome).
//  * Each k-step a warp issues kTPW LDG.128 of A-fragments (512 B each, see
//    common.cuh) and one LDG.64 per n8 token tile, then kTPW*NT
//    mma.sync.m16n8k16 (fp32 accumulate).  kUnroll k-steps are loaded
//    before any math so ~8 KB per warp is in flight.
//  * A super-tile split between warps is finished by the last-arriving
//    warp, which sums the partials in worker order: deterministic for a
//    given (U, grid), no float atomics.
//  * The epilogue is fused: plain store, residual add, SiLU(gate)*up into
//    the next GEMV's B-frag layout, scatter into the expert-combine buffer,
//    or the LM-head argmax.
#pragma once

#include "common.cuh"

namespace cascade {

enum Epi : int {
    EPI_STORE = 0,   // out[tok*ld + row] = v
    EPI_ADD = 1,     // out[tok*ld + row] += v      (residual)
    EPI_GATEUP = 2,  // H[slot] (B-frag, bf16) = silu(gate) * up
    EPI_DOWN = 3,    // ycontrib[(tok*n_contrib + rank)*ld + row] = v
    EPI_ARGMAX = 4,  // keys[tok] = max(argmax_key(v, row)); optional logits store
};

struct GemvParams {
    const uint4* W;            // A-frag weights of local block 0
    long long w_block_stride;  // uint4 units between blocks
    const uint2* B;            // B-frag activations (list slot 0)
    long long b_block_stride;  // uint2 units between list slots (0: shared X)
    int* list;                 // active block ids, or nullptr (identity)
    int* count;                // device U, or nullptr (use n_blocks)
    int n_blocks;
    int n_st;                  // super-tiles per block
    int n_ks;                  // k-steps per block (K / 16)
    int T;                     // tokens in flight
    int min_seg;               // minimum k-steps per worker
    float4* partial;           // stream-K partials [workers][2][kTPW][NT][32]
    int* counters;             // per-unit arrival counters (zero between launches)
    float* out;                // EPI_STORE / EPI_ADD / EPI_DOWN / EPI_ARGMAX (opt.)
    int ld;                    // leading dimension of out
    uint16_t* hout;            // EPI_GATEUP output (B-frag bf16)
    long long h_block_stride;  // bf16 units between list slots
    int* route_rank;           // EPI_DOWN: [slot][16] -> rank in token's list or -1
    int n_contrib;             // EPI_DOWN
    unsigned long long* keys;  // EPI_ARGMAX
    unsigned long long* stamp; // optional globaltimer stamp at kernel start
    unsigned long long* trace; // in-graph trace slot
    int early_list;            // list/count final before griddepcontrol.wait (expert down projection)
    int l2_prologue;           // also L2-prefetch each warp's range before the wait: 0 off, 1 all, n > 1: the first n k-steps
    int trigger;               // griddepcontrol.launch_dependents right after the wait
    // Routed blocks: when topk_id is set, every CTA builds the expert union
    // itself from the router's top-k (no separate union kernel, no
    // cross-CTA synchronisation in the router); list / count / route_rank
    // above are then outputs, written by CTA 0 when `publish` is set.
    const int* topk_id;        // [T][k_top] routed expert ids (router output)
    int k_top, E, e_lo, e_hi;  // routed experts; local ones are [e_lo, e_hi)
    int S, ep_rank, ep_size;   // shared blocks; shared block b lives on rank b % ep_size
    int publish;
    int* union_size;           // out (publish): distinct routed experts of the step
    int invariant;             // 1: fixed pieces per block (batch-invariant sums); 0: stream-K over all blocks
    int unit_pieces;           // stream-K mode: one whole super-tile per CTA when the active super-tiles nearly fill the grid
    // SM-speed-weighted pieces: streaming rates differ by SM (a fixed
    // property of the part, +-3%; the slowest SM sets the kernel time), so
    // the work index of a CTA is (dense SM index, slot on that SM) and the
    // pieces of a grid-wide split are sized by the SM's measured rate.
    const int* sm_index;       // %smid -> dense SM index (or -1), nullptr: work index = blockIdx.x
    int* sm_slot;              // per-%smid arrival counters (parity = slot of the 2 CTAs of an SM)
    const int* cum;            // [grid + 1] cumulative piece weights, cum[grid] = 1 << 24 (nullptr: equal)
};

constexpr int kGemvThreads = 256;
constexpr int kGemvWarps = kGemvThreads / 32;
constexpr int kUnionExperts = 128;                 // expert_model.hpp:96 (kMaxRoutedExperts)
constexpr int kMaxSlots = kUnionExperts + 16;      // local routed + shared blocks

struct UnionSmem {
    int list[kMaxSlots];                 // slot -> local block id (ascending routed, then shared)
    int slot_of[kUnionExperts];          // routed expert -> slot (local only)
    signed char rank[kMaxSlots][kMaxT];  // slot, token -> rank in the token's contribution list, or -1
    int count;                           // active local blocks
    int union_size;                      // distinct routed experts (global)
};

// One warp: the expert union of the T tokens' top-k (the real counterpart
// of the reference's sample_active_experts, expert_model.hpp:120-139:
// union = distinct routed experts; shared blocks always active on top),
// as the ascending list of local blocks and per-(slot, token) ranks.
__device__ __forceinline__ void build_union(const GemvParams& p, UnionSmem& u) {
    const int lane = threadIdx.x & 31;
    const int n = p.T * p.k_top;  // <= 16 * 16
    int ev[8];
    unsigned long long m0 = 0, m1 = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int i = lane + 32 * j;
        ev[j] = i < n ? __ldcg(p.topk_id + i) : -1;
        if (ev[j] >= 0) {
            if (ev[j] < 64) m0 |= 1ull << ev[j];
            else m1 |= 1ull << (ev[j] - 64);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        m0 |= __shfl_xor_sync(0xffffffffu, m0, o);
        m1 |= __shfl_xor_sync(0xffffffffu, m1, o);
    }
    int base = 0;
#pragma unroll
    for (int q = 0; q < kUnionExperts / 32; ++q) {
        const int e = 32 * q + lane;
        const bool in = e < p.E && (((e < 64 ? (m0 >> e) : (m1 >> (e - 64))) & 1ull) != 0);
        const bool loc = in && e >= p.e_lo && e < p.e_hi;
        const unsigned b = __ballot_sync(0xffffffffu, loc);
        if (loc) {
            const int slot = base + __popc(b & ((1u << lane) - 1u));
            u.list[slot] = e - p.e_lo;
            u.slot_of[e] = slot;
        }
        base += __popc(b);
    }
    const int n_local = base;
    int nsh = 0;
    for (int b2 = 0; b2 < p.S; ++b2) {
        if (b2 % p.ep_size != p.ep_rank) continue;
        const int slot = n_local + nsh;
        if (lane == 0) u.list[slot] = (p.e_hi - p.e_lo) + nsh;
        if (lane < kMaxT) u.rank[slot][lane] = lane < p.T ? (signed char)(p.k_top + b2) : (signed char)-1;
        ++nsh;
    }
    for (int i = lane; i < n_local * kMaxT; i += 32) u.rank[i / kMaxT][i % kMaxT] = -1;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int i = lane + 32 * j;
        const int e = ev[j];
        if (e >= p.e_lo && e < p.e_hi) u.rank[u.slot_of[e]][i / p.k_top] = (signed char)(i % p.k_top);
    }
    if (lane == 0) {
        u.count = n_local + nsh;
        u.union_size = __popcll(m0) + __popcll(m1);
    }
    __syncwarp();
}

// CTA 0 of the gate/up launch publishes the union for the accept kernel,
// telemetry and the debug taps.
__device__ __forceinline__ void publish_union(const GemvParams& p, const UnionSmem& u) {
    for (int i = threadIdx.x; i < u.count * kMaxT; i += blockDim.x)
        p.route_rank[i] = u.rank[i / kMaxT][i % kMaxT];
    for (int i = threadIdx.x; i < u.count; i += blockDim.x) p.list[i] = u.list[i];
    if (threadIdx.x == 0) {
        *p.count = u.count;
        *p.union_size = u.union_size;
    }
}


__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

template <int NT, int EPI>
__device__ __forceinline__ void gemv_epilogue(const GemvParams& p, int bl, int st, int lane,
                                              float (&acc)[kTPW][NT][4], const signed char* rr) {
    const int g = lane >> 2, t = lane & 3;
    if constexpr (EPI == EPI_STORE || EPI == EPI_ADD) {
#pragma unroll
        for (int it = 0; it < kTPW; ++it) {
            const int row = st * kSTRows + it * 16 + g;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const int tok = nt * 8 + 2 * t;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int tk = tok + (c & 1);
                    const int r = row + 8 * (c >> 1);
                    if (tk < p.T) {
                        float* o = p.out + (long long)tk * p.ld + r;
                        if constexpr (EPI == EPI_ADD) *o += acc[it][nt][c];
                        else *o = acc[it][nt][c];
                    }
                }
            }
        }
    } else if constexpr (EPI == EPI_GATEUP) {
        // rows g (gate j) and g+8 (up j) of each tile share j.
        uint16_t* H = p.hout + (long long)bl * p.h_block_stride;
#pragma unroll
        for (int it = 0; it < kTPW; ++it) {
            const int j = st * (kSTRows / 2) + it * 8 + g;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int tk = nt * 8 + 2 * t + c;
                    const float gate = acc[it][nt][c];
                    const float up = acc[it][nt][2 + c];
                    const float h = tk < p.T ? silu(gate) * up : 0.0f;
                    H[bfrag_index(tk, j)] = bf16_bits(h);
                }
            }
        }
    } else if constexpr (EPI == EPI_DOWN) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int tk = nt * 8 + 2 * t + c;
                if (tk >= p.T) continue;
                const int rank = rr[tk];
                if (rank < 0) continue;
                float* o = p.out + ((long long)tk * p.n_contrib + rank) * p.ld;
#pragma unroll
                for (int it = 0; it < kTPW; ++it) {
                    const int row = st * kSTRows + it * 16 + g;
                    o[row] = acc[it][nt][c];
                    o[row + 8] = acc[it][nt][2 + c];
                }
            }
        }
    } else if constexpr (EPI == EPI_ARGMAX) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int tk = nt * 8 + 2 * t + c;
                unsigned long long best = 0ull;
#pragma unroll
                for (int it = 0; it < kTPW; ++it) {
                    const int row = st * kSTRows + it * 16 + g;
                    const unsigned long long k0 = argmax_key(acc[it][nt][c], row);
                    const unsigned long long k1 = argmax_key(acc[it][nt][2 + c], row + 8);
                    best = k0 > best ? k0 : best;
                    best = k1 > best ? k1 : best;
                    if (p.out != nullptr && tk < p.T) {
                        p.out[(long long)tk * p.ld + row] = acc[it][nt][c];
                        p.out[(long long)tk * p.ld + row + 8] = acc[it][nt][2 + c];
                    }
                }
                // reduce over the 8 lanes (g) that hold the same token
#pragma unroll
                for (int o = 4; o < 32; o <<= 1) {
                    const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
                    best = other > best ? other : best;
                }
                if (g == 0 && tk < p.T) atomicMax(p.keys + tk, best);
            }
        }
    }
}

// owner of flat position q when [0,total) is split into n ranges
// [floor(total*w/n), floor(total*(w+1)/n))
__device__ __forceinline__ int owner_of(long long q, long long total, int n) {
    return (int)(((q + 1) * n + total - 1) / total) - 1;
}

// piece boundaries of a split of [0, total) into n pieces: weighted by
// cum (n == grid) or equal
__device__ __forceinline__ long long piece_start(long long total, int q, int n, const int* cum) {
    if (cum != nullptr && n == (int)gridDim.x) return (total * (long long)__ldg(cum + q)) >> 24;
    return total * q / n;
}
__device__ __forceinline__ int piece_owner(long long pos, long long total, int n, const int* cum) {
    if (cum == nullptr || n != (int)gridDim.x) return owner_of(pos, total, n);
    int lo = 0, hi = n - 1;  // largest q with piece_start(q) <= pos
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (piece_start(total, mid, n, cum) <= pos) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Work index of this CTA: (dense SM index, slot) when the SM map is set.
// Each SM hosts exactly 2 CTAs of a 2*SMs grid (register-limited), and each
// launch adds 2 to the SM's counter, so its parity tells the two apart.
__device__ __forceinline__ int gemv_work_index(const GemvParams& p) {
    __shared__ int s_wi;
    if (p.sm_index == nullptr) return (int)blockIdx.x;
    if (threadIdx.x == 0) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        const int dense = p.sm_index[smid];
        const int slot = atomicAdd(p.sm_slot + smid, 1) & 1;
        s_wi = dense * 2 + slot;
    }
    __syncthreads();
    return s_wi;
}

template <int NT>
__device__ __forceinline__ void zero_acc(float (&acc)[kTPW][NT][4]) {
#pragma unroll
    for (int it = 0; it < kTPW; ++it)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[it][nt][c] = 0.f;
}

template <int NT>
__device__ __forceinline__ void add_acc(float (&acc)[kTPW][NT][4], const float4* src, bool cg) {
#pragma unroll
    for (int it = 0; it < kTPW; ++it)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const float4 v = cg ? __ldcg(src + (it * NT + nt) * 32) : src[(it * NT + nt) * 32];
            acc[it][nt][0] += v.x;
            acc[it][nt][1] += v.y;
            acc[it][nt][2] += v.z;
            acc[it][nt][3] += v.w;
        }
}

template <int NT>
__device__ __forceinline__ void store_acc(float4* dst, const float (&acc)[kTPW][NT][4], bool cg) {
#pragma unroll
    for (int it = 0; it < kTPW; ++it)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const float4 v = make_float4(acc[it][nt][0], acc[it][nt][1], acc[it][nt][2], acc[it][nt][3]);
            if (cg) __stcg(dst + (it * NT + nt) * 32, v);
            else dst[(it * NT + nt) * 32] = v;
        }
}

// Pieces per block: a fixed function of the block shape and the grid, so
// every super-tile is cut at the same k-steps whatever the router chose
// (U) and however many tokens ride along.  Sums are therefore identical
// for a token in any verify step (batch-invariant), which makes greedy
// speculative decoding bitwise lossless.  CTA c streams piece c of every
// active block when P == grid (equal bytes per CTA for any U).
__device__ __forceinline__ int block_pieces(const GemvParams& p, long long per_block) {
    // Small experts (OLMoE at K = 0: 256 gate/up super-tiles of 256 KB for
    // 296 CTAs): when the active super-tiles nearly fill the grid, one whole
    // super-tile per CTA removes every cross-CTA partial (global partial
    // store, fence, arrival atomic and reload) at the cost of idling the
    // surplus CTAs; HBM stays saturated with >= 80% of the CTAs streaming.
    if (p.unit_pieces && !p.invariant) {
        const long long units = per_block / p.n_ks;
        if (units <= (long long)gridDim.x && units * 5 >= (long long)gridDim.x * 4) return (int)units;
    }
    long long pm = per_block / ((long long)p.min_seg * kGemvWarps);
    if (pm < 1) pm = 1;
    return pm < (long long)gridDim.x ? (int)pm : (int)gridDim.x;
}
// Mode 0 (stream-K) treats the whole active range as one block: P = grid
// equal contiguous pieces, one per CTA, each split among the 8 warps.

template <int NT>
constexpr int gemv_smem_bytes() {
    return kGemvWarps * 2 * kTPW * NT * 32 * 16;
}

// Stream-K at two levels.  The flat work range is split into one
// contiguous range per CTA, and each CTA range into one contiguous range
// per warp.  A warp finishes every super-tile it covers completely
// (epilogue straight from registers).  Super-tiles split between warps of
// the same CTA are reduced through shared memory by their first
// contributor in warp order; only the (at most two) super-tiles that cross
// a CTA boundary go through global memory, where the last-arriving CTA
// sums the CTA partials in CTA order.  Every summation order is a pure
// function of (U, grid), so results are deterministic.
template <int NT, int EPI>
__global__ void __launch_bounds__(kGemvThreads, 2) stream_gemv_kernel(GemvParams p) {
    extern __shared__ float4 red[];  // [warp][slot][kTPW*NT*32]
    __shared__ long long seg_unit[kGemvWarps][2];
    __shared__ UnionSmem un;
    const bool routed = p.topk_id != nullptr;
    auto rk_row = [&](int bl) -> const signed char* { return routed ? un.rank[bl] : nullptr; };
    constexpr int kSlot = kTPW * NT * 32;
#ifndef CASCADE_KUNROLL1
#define CASCADE_KUNROLL1 4
#endif
#ifndef CASCADE_KUNROLL2
#define CASCADE_KUNROLL2 3
#endif
    constexpr int kUnroll = NT == 1 ? CASCADE_KUNROLL1 : CASCADE_KUNROLL2;  // k-steps of weights in flight per warp
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const uint64_t pol = policy_evict_first();

    // PDL prologue: a dense job's weights do not depend on the previous
    // kernel, so the first kUnroll k-steps of every warp are requested
    // *before* griddepcontrol.wait and stream in while the predecessor
    // (attention combine / expert combine) is still finishing.
    uint4 a[kUnroll][kTPW];
    bool pre = false;
    const bool dense = !routed && p.list == nullptr && p.count == nullptr;
    const int wi = gemv_work_index(p);
    if (routed && p.early_list) {
        // the router's top-k was written two kernels back (final): build the
        // union now so the prologue can address the first expert weights
        if (warp == 0) build_union(p, un);
        __syncthreads();
    }
    if (dense || p.early_list) {
        // weights addressable now: dense matrices always; the expert down
        // projection because its active list was written two kernels back
        // and the gate/up kernel triggers its dependents only after its own
        // griddepcontrol.wait.
        const int U0 = dense ? p.n_blocks : (routed ? un.count : __ldcg(p.count));
        // work blocks: each expert block (batch-invariant mode), or the whole
        // active range as one block (stream-K: equal bytes per CTA, splits depend on U)
        const long long pb0 = (long long)p.n_st * p.n_ks * (p.invariant ? 1 : U0);
        const int nb0 = p.invariant ? U0 : (U0 > 0 ? 1 : 0);
        const int P0 = block_pieces(p, pb0);
        long long wlo0 = 0, whi0 = 0;
        if (wi < nb0 * P0) {
            const int b0 = wi / P0, q0 = wi - b0 * P0;
            const long long clo0 = (long long)b0 * pb0 + piece_start(pb0, q0, P0, p.cum);
            const long long chi0 = (long long)b0 * pb0 + piece_start(pb0, q0 + 1, P0, p.cum);
            wlo0 = clo0 + (chi0 - clo0) * warp / kGemvWarps;
            whi0 = clo0 + (chi0 - clo0) * (warp + 1) / kGemvWarps;
        }
        if (whi0 > wlo0) {
            const long long unit0 = wlo0 / p.n_ks;
            const int ks00 = (int)(wlo0 - unit0 * p.n_ks);
            const long long rem0 = whi0 - wlo0;
            const int ks10 = rem0 < (long long)(p.n_ks - ks00) ? ks00 + (int)rem0 : p.n_ks;
            long long pf_from = wlo0;
            if (ks10 - ks00 >= kUnroll) {
                const int bl0 = (int)(unit0 / p.n_st);
                const int st0 = (int)(unit0 - (long long)bl0 * p.n_st);
                const int blk0 = routed ? un.list[bl0] : (p.list ? __ldcg(p.list + bl0) : bl0);
                const uint4* A0 = p.W + (long long)blk0 * p.w_block_stride +
                                  (long long)st0 * p.n_ks * (kTPW * 32) + lane;
#pragma unroll
                for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                    for (int it = 0; it < kTPW; ++it)
                        a[u][it] = ldg_stream(A0 + ((long long)(ks00 + u) * kTPW + it) * 32, pol);
                pre = true;
                pf_from = wlo0 + kUnroll;
            }
            if (p.l2_prologue && lane == 0) {
                // the rest of this warp's range -> L2 while the predecessor drains
                const long long pf_to = p.l2_prologue > 1 && wlo0 + p.l2_prologue < whi0 ? wlo0 + p.l2_prologue : whi0;
                for (long long pos = pf_from; pos < pf_to;) {
                    const long long unit = pos / p.n_ks;
                    const int ks = (int)(pos - unit * p.n_ks);
                    long long n = p.n_ks - ks;
                    if (pf_to - pos < n) n = pf_to - pos;
                    const int bl = (int)(unit / p.n_st);
                    const int st = (int)(unit - (long long)bl * p.n_st);
                    const int blk = routed ? un.list[bl] : (p.list ? __ldcg(p.list + bl) : bl);
                    const char* src = reinterpret_cast<const char*>(
                        p.W + (long long)blk * p.w_block_stride + ((long long)st * p.n_ks + ks) * (kTPW * 32));
                    const unsigned long long bytes = (unsigned long long)n * kTPW * 32 * 16;
                    for (unsigned long long off = 0; off < bytes; off += 65536) {
                        const unsigned long long sz = bytes - off < 65536 ? bytes - off : 65536;
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + off), "r"((uint32_t)sz)
                                     : "memory");
                    }
                    pos += n;
                }
            }
        }
    }
    griddep_wait();
    if (p.trigger) griddep_launch();
    CTA_TRACE(p.trace);
    if (p.stamp != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *p.stamp = globaltimer();
    if (routed && !p.early_list) {
        if (warp == 0) build_union(p, un);
        __syncthreads();
    }
    if (routed && p.publish && blockIdx.x == 0) publish_union(p, un);
    const int U = routed ? un.count : (p.count ? *p.count : p.n_blocks);
    const long long per_block = (long long)p.n_st * p.n_ks * (p.invariant ? 1 : U);
    const int n_blocks_w = p.invariant ? U : (U > 0 ? 1 : 0);
    const int P = block_pieces(p, per_block);
    const int n_items = n_blocks_w * P;
    float acc[kTPW][NT][4];
    constexpr int kMaxPend = 2 * kMaxSlots;  // <= 2 boundary super-tiles per item
    __shared__ int4 pend[kMaxPend];
    __shared__ int n_pend;
    if (threadIdx.x == 0) n_pend = 0;
    __syncthreads();
    for (int item = wi; item < n_items; item += gridDim.x) {
        const int b = item / P, q = item - b * P;
        // this piece of block b, in flat (unit, k-step) positions
        const long long base = (long long)b * per_block;
        const long long clo = base + piece_start(per_block, q, P, p.cum), chi = base + piece_start(per_block, q + 1, P, p.cum);
        const long long wlo = clo + (chi - clo) * warp / kGemvWarps;
        const long long whi = clo + (chi - clo) * (warp + 1) / kGemvWarps;
        if (lane == 0) {
            seg_unit[warp][0] = -1;
            seg_unit[warp][1] = -1;
        }
        __syncwarp();

        long long pos = wlo;
        while (pos < whi) {
            const long long unit = pos / p.n_ks;
            const int ks0 = (int)(pos - unit * p.n_ks);
            const long long rem = whi - pos;
            const int ks1 = rem < (long long)(p.n_ks - ks0) ? ks0 + (int)rem : p.n_ks;
            const int bl = (int)(unit / p.n_st);
            const int st = (int)(unit - (long long)bl * p.n_st);
            const int blk = routed ? un.list[bl] : (p.list ? p.list[bl] : bl);
            const uint4* A = p.W + (long long)blk * p.w_block_stride + (long long)st * p.n_ks * (kTPW * 32) + lane;
            const uint2* Bp = p.B + (long long)bl * p.b_block_stride + lane;
            zero_acc<NT>(acc);
            int s = ks0;
            for (; s + kUnroll <= ks1; s += kUnroll) {
                uint2 bb[kUnroll][NT];
                if (!pre) {
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                        for (int it = 0; it < kTPW; ++it)
                            a[u][it] = ldg_stream(A + ((long long)(s + u) * kTPW + it) * 32, pol);
                }
                pre = false;
#pragma unroll
                for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) bb[u][nt] = ldg_act(Bp + ((s + u) * 2 + nt) * 32);
#pragma unroll
                for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                    for (int it = 0; it < kTPW; ++it)
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) mma_bf16_16816(acc[it][nt], a[u][it], bb[u][nt]);
            }
            for (; s < ks1; ++s) {
                uint4 a1[kTPW];
                uint2 bb[NT];
#pragma unroll
                for (int it = 0; it < kTPW; ++it) a1[it] = ldg_stream(A + ((long long)s * kTPW + it) * 32, pol);
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) bb[nt] = ldg_act(Bp + (s * 2 + nt) * 32);
#pragma unroll
                for (int it = 0; it < kTPW; ++it)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) mma_bf16_16816(acc[it][nt], a1[it], bb[nt]);
            }
            const bool first_seg = pos == wlo;
            pos += ks1 - ks0;
            if (ks0 == 0 && ks1 == p.n_ks) {
                gemv_epilogue<NT, EPI>(p, bl, st, lane, acc, rk_row(bl));
            } else {
                const int slot = first_seg ? 0 : 1;
                store_acc<NT>(red + (warp * 2 + slot) * kSlot + lane, acc, false);
                if (lane == 0) seg_unit[warp][slot] = unit;
            }
        }
        __syncthreads();

        // ---- piece-level reduction of split super-tiles (owner = first contributor)
        for (int slot = 0; slot < 2; ++slot) {
            const long long unit = seg_unit[warp][slot];
            if (unit < 0) continue;
            bool owner = true;
            for (int w = 0; w < warp && owner; ++w) owner = seg_unit[w][0] != unit && seg_unit[w][1] != unit;
            if (!owner) continue;
            zero_acc<NT>(acc);
            add_acc<NT>(acc, red + (warp * 2 + slot) * kSlot + lane, false);
            for (int w = warp + 1; w < kGemvWarps; ++w)
                for (int s2 = 0; s2 < 2; ++s2)
                    if (seg_unit[w][s2] == unit) add_acc<NT>(acc, red + (w * 2 + s2) * kSlot + lane, false);
            const long long ustart = unit * p.n_ks, uend = ustart + p.n_ks;
            const int bl = (int)(unit / p.n_st);
            const int st = (int)(unit - (long long)bl * p.n_st);
            if (ustart >= clo && uend <= chi) {
                gemv_epilogue<NT, EPI>(p, bl, st, lane, acc, rk_row(bl));
                continue;
            }
            // crosses a piece boundary: store the piece partial now, count the
            // arrival after the CTA's last item (one fence for all of them)
            const int first = piece_owner(ustart - base, per_block, P, p.cum);
            const int last = piece_owner(uend - 1 - base, per_block, P, p.cum);
            const int gslot = (q == first) ? 1 : 0;
            store_acc<NT>(p.partial + (((long long)b * P + q) * 2 + gslot) * kSlot + lane, acc, true);
            if (lane == 0) {
                const int i = atomicAdd(&n_pend, 1);
                if (i < kMaxPend) pend[i] = make_int4((int)unit, b, first, last);
            }
        }
        __syncthreads();  // red[] / seg_unit reused by the next item
    }
    // ---- cross-piece reductions: every piece partial of this CTA is stored;
    //      one fence, then the arrivals; the last arriving piece of a
    //      super-tile sums the piece partials in piece order
    __threadfence();
    __syncthreads();
    const int np = n_pend < kMaxPend ? n_pend : kMaxPend;
    for (int e = warp; e < np; e += kGemvWarps) {
        const int4 pe = pend[e];
        const long long unit = pe.x;
        const int b = pe.y, first = pe.z, last = pe.w;
        int prev = 0;
        if (lane == 0) prev = atomicAdd(p.counters + unit, 1);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev != last - first) continue;
        __threadfence();
        zero_acc<NT>(acc);
        for (int j = first; j <= last; ++j)
            add_acc<NT>(acc, p.partial + (((long long)b * P + j) * 2 + (j == first ? 1 : 0)) * kSlot + lane, true);
        if (lane == 0) p.counters[unit] = 0;
        const int bl = (int)(unit / p.n_st);
        const int st = (int)(unit - (long long)bl * p.n_st);
        gemv_epilogue<NT, EPI>(p, bl, st, lane, acc, rk_row(bl));
    }
}

// CUDA-core alternative for a single token (T = 1, K = 0 steps): the lane's
// A-fragment holds rows g and g+8 at k = 2t..2t+1 and 2t+8..2t+9 of the
// k-step; the token's activations at the same k come from lane t of the
// B-fragment (token 0 lives in lanes 0-3).  Eight FMAs per tile, no tensor
// core; the four partial sums of a row (the quad's lanes t = 0..3) are
// added after the segment (fma_quad_to_acc), which leaves the mma.sync
// accumulator layout so the reductions and epilogues are shared.
__device__ __forceinline__ void fma_tile_t1(float (&pr)[2], const uint4& a, const uint2& b) {
    const float x0 = __uint_as_float(b.x << 16), x1 = __uint_as_float(b.x & 0xFFFF0000u);
    const float x8 = __uint_as_float(b.y << 16), x9 = __uint_as_float(b.y & 0xFFFF0000u);
    float r0 = pr[0], r1 = pr[1];
    r0 = fmaf(__uint_as_float(a.x << 16), x0, r0);
    r0 = fmaf(__uint_as_float(a.x & 0xFFFF0000u), x1, r0);
    r0 = fmaf(__uint_as_float(a.z << 16), x8, r0);
    r0 = fmaf(__uint_as_float(a.z & 0xFFFF0000u), x9, r0);
    r1 = fmaf(__uint_as_float(a.y << 16), x0, r1);
    r1 = fmaf(__uint_as_float(a.y & 0xFFFF0000u), x1, r1);
    r1 = fmaf(__uint_as_float(a.w << 16), x8, r1);
    r1 = fmaf(__uint_as_float(a.w & 0xFFFF0000u), x9, r1);
    pr[0] = r0;
    pr[1] = r1;
}
template <int NT>
__device__ __forceinline__ void fma_quad_to_acc(float (&pr)[kTPW][2], float (&acc)[kTPW][NT][4]) {
#pragma unroll
    for (int it = 0; it < kTPW; ++it)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            float v = pr[it][h];
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            acc[it][0][h * 2] = v;      // rows g / g+8, token 2t (token 0 on lanes t = 0)
            acc[it][0][h * 2 + 1] = 0.f;
        }
}

// One phase of the fused expert FFN (expert_ffn_kernel): the stream-K work
// of stream_gemv_kernel for one matrix.  Phase 0 (gate/up) counts each
// finished super-tile of slot bl in s_done[bl]; phase 1 (down) waits, per
// slot, until ready[bl] reaches target (every gate/up super-tile of that
// expert published) and reads its B operand (SiLU(gate)*up, written in this
// launch) from L2.
template <int NT, int EPI, bool WAIT, bool FMA = false>
__device__ __forceinline__ void ffn_phase(const GemvParams& p, const UnionSmem& un, int wi, int* s_done,
                                          const int* ready, int target) {
    static_assert(!FMA || NT == 1, "the CUDA-core path serves one token");
    extern __shared__ float4 red[];
    __shared__ long long seg_unit[kGemvWarps][2];
    const bool routed = true;
    auto rk_row = [&](int bl) -> const signed char* { return un.rank[bl]; };
    constexpr int kSlot = kTPW * NT * 32;
    constexpr int kUnroll = NT == 1 ? CASCADE_KUNROLL1 : CASCADE_KUNROLL2;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const uint64_t pol = policy_evict_first();
    uint4 a[kUnroll][kTPW];
    bool pre = false;
    unsigned long long ready_mask[WAIT ? (kMaxSlots + 63) / 64 : 1] = {};
    bool waited = false;
    // CTA-wide readiness: one warp polls a slot's global counter (the first
    // to need it claims s_poll[slot]); the others watch the shared bit.  A
    // poll per warp on one counter line (2368 warps) delayed the release by
    // microseconds behind the publishing atomics.
    __shared__ unsigned int s_ready_bits[(kMaxSlots + 31) / 32];
    __shared__ int s_poll[kMaxSlots];
    if constexpr (WAIT) {
        for (int i = threadIdx.x; i < (kMaxSlots + 31) / 32; i += blockDim.x) s_ready_bits[i] = 0u;
        for (int i = threadIdx.x; i < kMaxSlots; i += blockDim.x) s_poll[i] = 0;
    }
    (void)kSlot;
    const int U = routed ? un.count : (p.count ? *p.count : p.n_blocks);
    const long long per_block = (long long)p.n_st * p.n_ks * (p.invariant ? 1 : U);
    const int n_blocks_w = p.invariant ? U : (U > 0 ? 1 : 0);
    const int P = block_pieces(p, per_block);
    const int n_items = n_blocks_w * P;
    float acc[kTPW][NT][4];
    constexpr int kMaxPend = 2 * kMaxSlots;  // <= 2 boundary super-tiles per item
    __shared__ int4 pend[kMaxPend];
    __shared__ int n_pend;
    if (threadIdx.x == 0) n_pend = 0;
    __syncthreads();
    for (int item = wi; item < n_items; item += gridDim.x) {
        const int b = item / P, q = item - b * P;
        // this piece of block b, in flat (unit, k-step) positions
        const long long base = (long long)b * per_block;
        const long long clo = base + piece_start(per_block, q, P, p.cum), chi = base + piece_start(per_block, q + 1, P, p.cum);
        const long long wlo = clo + (chi - clo) * warp / kGemvWarps;
        const long long whi = clo + (chi - clo) * (warp + 1) / kGemvWarps;
        if (lane == 0) {
            seg_unit[warp][0] = -1;
            seg_unit[warp][1] = -1;
        }
        __syncwarp();
        if constexpr (WAIT) {
            // Down phase: the weights do not depend on the gate/up results, so
            // the first p.l2_prologue k-steps of this warp's range stream into
            // L2 while the CTA waits for its slots' readiness.
            if (p.l2_prologue > 0 && item == wi && lane == 0) {
                const long long pf_to = wlo + p.l2_prologue < whi ? wlo + p.l2_prologue : whi;
                for (long long q = wlo; q < pf_to;) {
                    const long long unit = q / p.n_ks;
                    const int ks = (int)(q - unit * p.n_ks);
                    long long n = p.n_ks - ks;
                    if (pf_to - q < n) n = pf_to - q;
                    const int bl = (int)(unit / p.n_st);
                    const int st = (int)(unit - (long long)bl * p.n_st);
                    const char* src = reinterpret_cast<const char*>(
                        p.W + (long long)un.list[bl] * p.w_block_stride + ((long long)st * p.n_ks + ks) * (kTPW * 32));
                    const unsigned long long bytes = (unsigned long long)n * kTPW * 32 * 16;
                    for (unsigned long long off = 0; off < bytes; off += 65536) {
                        const unsigned long long sz = bytes - off < 65536 ? bytes - off : 65536;
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + off), "r"((uint32_t)sz)
                                     : "memory");
                    }
                    q += n;
                }
            }
        }

        long long pos = wlo;
        while (pos < whi) {
            const long long unit = pos / p.n_ks;
            const int ks0 = (int)(pos - unit * p.n_ks);
            const long long rem = whi - pos;
            const int ks1 = rem < (long long)(p.n_ks - ks0) ? ks0 + (int)rem : p.n_ks;
            const int bl = (int)(unit / p.n_st);
            const int st = (int)(unit - (long long)bl * p.n_st);
            const int blk = routed ? un.list[bl] : (p.list ? p.list[bl] : bl);
            if constexpr (WAIT) {
                if (!((ready_mask[bl >> 6] >> (bl & 63)) & 1ull)) {
                    if (lane == 0) {
                        volatile unsigned int* bits = s_ready_bits;
                        const unsigned int bit = 1u << (bl & 31);
                        const bool poller = !(bits[bl >> 5] & bit) && atomicCAS(&s_poll[bl], 0, 1) == 0;
                        long long spins = 0;
                        for (;;) {
                            if (bits[bl >> 5] & bit) break;
                            if (poller) {
                                int v;
                                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];"
                                             : "=r"(v)
                                             : "l"(ready + (long long)bl * kReadyStride)
                                             : "memory");
                                if (v >= target) {
                                    __threadfence_block();
                                    atomicOr(&s_ready_bits[bl >> 5], bit);
                                    break;
                                }
                            }
                            if (++spins > (1ll << 24)) __trap();  // a lost producer must not hang the GPU (~seconds)
                            __nanosleep(poller ? 32 : 64);
                        }
                        __threadfence_block();
                    }
                    __syncwarp();
                    if (!waited) {
                        cta_phase(p.trace, 3);  // first readiness wait of this warp released
                        phase_stamp(p.trace, 5);
                    }
                    waited = true;
                    ready_mask[bl >> 6] |= 1ull << (bl & 63);
                }
            }
            const uint4* A = p.W + (long long)blk * p.w_block_stride + (long long)st * p.n_ks * (kTPW * 32) + lane;
            // FMA: every lane reads token 0's B-fragment entry of its quad position (lane t)
            const uint2* Bp = p.B + (long long)bl * p.b_block_stride + (FMA ? (lane & 3) : lane);
            zero_acc<NT>(acc);
            float pr[kTPW][2];
            if constexpr (FMA) {
#pragma unroll
                for (int it = 0; it < kTPW; ++it) pr[it][0] = pr[it][1] = 0.f;
            }
            int s = ks0;
            for (; s + kUnroll <= ks1; s += kUnroll) {
                uint2 bb[kUnroll][NT];
                if (!pre) {
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                        for (int it = 0; it < kTPW; ++it)
                            a[u][it] = ldg_stream(A + ((long long)(s + u) * kTPW + it) * 32, pol);
                }
                pre = false;
#pragma unroll
                for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) bb[u][nt] = WAIT ? ldcg_act(Bp + ((s + u) * 2 + nt) * 32) : ldg_act(Bp + ((s + u) * 2 + nt) * 32);
#pragma unroll
                for (int u = 0; u < kUnroll; ++u)
#pragma unroll
                    for (int it = 0; it < kTPW; ++it) {
                        if constexpr (FMA) fma_tile_t1(pr[it], a[u][it], bb[u][0]);
                        else {
#pragma unroll
                            for (int nt = 0; nt < NT; ++nt) mma_bf16_16816(acc[it][nt], a[u][it], bb[u][nt]);
                        }
                    }
            }
            for (; s < ks1; ++s) {
                uint4 a1[kTPW];
                uint2 bb[NT];
#pragma unroll
                for (int it = 0; it < kTPW; ++it) a1[it] = ldg_stream(A + ((long long)s * kTPW + it) * 32, pol);
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) bb[nt] = WAIT ? ldcg_act(Bp + (s * 2 + nt) * 32) : ldg_act(Bp + (s * 2 + nt) * 32);
#pragma unroll
                for (int it = 0; it < kTPW; ++it) {
                    if constexpr (FMA) fma_tile_t1(pr[it], a1[it], bb[0]);
                    else {
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) mma_bf16_16816(acc[it][nt], a1[it], bb[nt]);
                    }
                }
            }
            if constexpr (FMA) fma_quad_to_acc<NT>(pr, acc);
            const bool first_seg = pos == wlo;
            pos += ks1 - ks0;
            if (ks0 == 0 && ks1 == p.n_ks) {
                gemv_epilogue<NT, EPI>(p, bl, st, lane, acc, rk_row(bl));
                if constexpr (!WAIT) { if (lane == 0) atomicAdd(s_done + bl, 1); }
            } else {
                const int slot = first_seg ? 0 : 1;
                store_acc<NT>(red + (warp * 2 + slot) * kSlot + lane, acc, false);
                if (lane == 0) seg_unit[warp][slot] = unit;
            }
        }
        if (item == wi) {
            phase_stamp(p.trace, WAIT ? 6 : 1);  // CTA 0, warp 0: its range streamed
            warp_stamp(p.trace, WAIT ? 1 : 0);   // CTAs 0-1, every warp (scripts/warp_spread.py)
        }
        __syncthreads();

        // ---- piece-level reduction of split super-tiles (owner = first contributor)
        for (int slot = 0; slot < 2; ++slot) {
            const long long unit = seg_unit[warp][slot];
            if (unit < 0) continue;
            bool owner = true;
            for (int w = 0; w < warp && owner; ++w) owner = seg_unit[w][0] != unit && seg_unit[w][1] != unit;
            if (!owner) continue;
            zero_acc<NT>(acc);
            add_acc<NT>(acc, red + (warp * 2 + slot) * kSlot + lane, false);
            for (int w = warp + 1; w < kGemvWarps; ++w)
                for (int s2 = 0; s2 < 2; ++s2)
                    if (seg_unit[w][s2] == unit) add_acc<NT>(acc, red + (w * 2 + s2) * kSlot + lane, false);
            const long long ustart = unit * p.n_ks, uend = ustart + p.n_ks;
            const int bl = (int)(unit / p.n_st);
            const int st = (int)(unit - (long long)bl * p.n_st);
            if (ustart >= clo && uend <= chi) {
                gemv_epilogue<NT, EPI>(p, bl, st, lane, acc, rk_row(bl));
                if constexpr (!WAIT) { if (lane == 0) atomicAdd(s_done + bl, 1); }
                continue;
            }
            // crosses a piece boundary: store the piece partial now, count the
            // arrival after the CTA's last item (one fence for all of them)
            const int first = piece_owner(ustart - base, per_block, P, p.cum);
            const int last = piece_owner(uend - 1 - base, per_block, P, p.cum);
            const int gslot = (q == first) ? 1 : 0;
            store_acc<NT>(p.partial + (((long long)b * P + q) * 2 + gslot) * kSlot + lane, acc, true);
            if (lane == 0) {
                const int i = atomicAdd(&n_pend, 1);
                if (i < kMaxPend) pend[i] = make_int4((int)unit, b, first, last);
            }
        }
        __syncthreads();  // red[] / seg_unit reused by the next item
        if (item == wi) phase_stamp(p.trace, WAIT ? 7 : 2);  // CTA 0: piece-level reductions done
    }
    // ---- cross-piece reductions: every piece partial of this CTA is stored;
    //      one fence, then the arrivals; the last arriving piece of a
    //      super-tile sums the piece partials in piece order
    // The barrier orders every warp's partial stores before the arrivals;
    // each arrival is an acq_rel atomic by one lane (release: this CTA's
    // partials; acquire: the other pieces' partials for the last arriver),
    // instead of a gpu-scope fence by every thread (~1 us after a streaming
    // phase, profiles/r02b).
    __syncthreads();
    const int np = n_pend < kMaxPend ? n_pend : kMaxPend;
    for (int e = warp; e < np; e += kGemvWarps) {
        const int4 pe = pend[e];
        const long long unit = pe.x;
        const int b = pe.y, first = pe.z, last = pe.w;
        int prev = 0;
        if (lane == 0) prev = atomic_add_acq_rel(p.counters + unit, 1);
        prev = __shfl_sync(0xffffffffu, prev, 0);
        if (prev != last - first) continue;
        __syncwarp();
        zero_acc<NT>(acc);
        for (int j = first; j <= last; ++j)
            add_acc<NT>(acc, p.partial + (((long long)b * P + j) * 2 + (j == first ? 1 : 0)) * kSlot + lane, true);
        if (lane == 0) p.counters[unit] = 0;
        const int bl = (int)(unit / p.n_st);
        const int st = (int)(unit - (long long)bl * p.n_st);
        gemv_epilogue<NT, EPI>(p, bl, st, lane, acc, rk_row(bl));
        if constexpr (!WAIT) { if (lane == 0) atomicAdd(s_done + bl, 1); }
    }
    phase_stamp(p.trace, WAIT ? 8 : 3);  // CTA 0, warp 0: cross-CTA reductions done
}

struct FfnParams {
    GemvParams gu, dn;         // expert gate/up (EPI_GATEUP) and down (EPI_DOWN) launches' parameters
    int* ready;                // [slots] published gate/up super-tiles (zeroed by the combine kernel)
    int n_st_gu;               // gate/up super-tiles per expert
    int dn_l2_stages;          // ring engine: down stages L2-prefetched at the gate/up -> down transition
};

// Fused expert FFN: gate/up (+SiLU) and down in one launch of 2 CTAs per SM
// (all co-resident), so the down projection needs no second launch, no
// kernel-boundary gap and no late-starting CTAs.  A CTA finishes its
// gate/up range, publishes the super-tiles it completed per expert (one
// fence), and streams its down range; a down segment of expert b starts
// once every gate/up super-tile of b is published.
template <int NT, bool FMA = false>
__global__ void __launch_bounds__(kGemvThreads, 2) expert_ffn_kernel(FfnParams f) {
    __shared__ UnionSmem un;
    __shared__ int s_done[kMaxSlots];
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kMaxSlots; i += blockDim.x) s_done[i] = 0;
    griddep_wait();
    if (f.gu.trigger) griddep_launch();
    CTA_TRACE(f.gu.trace);
    if (warp == 0) build_union(f.gu, un);
    __syncthreads();
    phase_stamp(f.gu.trace, 0);  // CTA 0: union built (phases 1-3 gate/up, 4 published, 5-8 down)
    if (f.gu.publish && blockIdx.x == 0) publish_union(f.gu, un);
    ffn_phase<NT, EPI_GATEUP, false, FMA>(f.gu, un, (int)blockIdx.x, s_done, nullptr, 0);
    cta_phase(f.gu.trace, 2);  // gate/up range of this CTA streamed
    __syncthreads();  // every h store of the CTA is ordered before the release adds below
    for (int i = threadIdx.x; i < un.count; i += blockDim.x)
        if (s_done[i] > 0) red_add_release(f.ready + (long long)i * kReadyStride, s_done[i]);
    phase_stamp(f.gu.trace, 4);
    ffn_phase<NT, EPI_DOWN, true, FMA>(f.dn, un, (int)blockIdx.x, nullptr, f.ready, f.n_st_gu);
}

}  // namespace cascade
