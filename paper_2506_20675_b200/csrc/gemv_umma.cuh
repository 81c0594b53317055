// gemv_umma.cuh — the weight-streaming engine of the verify step on the
// 5th-generation tensor cores: TMA bulk copies -> shared-memory ring ->
// tcgen05.mma (one issuing thread) -> TMEM accumulators -> tcgen05.ld
// epilogue.  Every linear layer of the step (QKV, O, routed + shared expert
// gate/up and down, LM head) is Y[T, rows] = X[T, K] * W[rows, K]^T with
// T = K_spec + 1 <= 16 tokens: the cost is the weight bytes, so the kernel
// is built to keep HBM streaming at copy speed and nothing else.
//
// Layouts (written by init.cuh / the activation producers):
//  * A (weights): 128-row units; per unit, per 16-column k-step, the UMMA
//    K-major no-swizzle canonical tile [kc 2][row 128][8 bf16] (4 KB):
//    core matrices of 8 rows x 16 B, 8-row groups 128 B apart (SBO), the
//    two 8-column halves 2 KB apart (LBO).  A unit's k-steps are
//    contiguous, so any k-range of a unit is one bulk copy.
//  * B (activations, 16 token slots): per k-step [kc 2][tok 16][8 bf16]
//    (512 B; SBO 128 B, LBO 256 B).  Token slots >= T hold don't-care
//    values: a token's column never mixes with another's, so N = 16 always
//    and results do not depend on T.
//
// Warp roles (192 threads, one CTA per SM; 108 KB of smem = three 32 KB
// weight stages + activations (scripts/umma_probe.cu sweep, profiles/r01),
// small enough that every kernel of the step runs in the same 132 KB
// shared-memory carveout and the SMs never reconfigure L1 between them):
//  * warps 0-3: epilogue — warp w owns TMEM lanes 32w..32w+31 = rows of
//    the unit; tcgen05.ld.32x32b.x16 gives each thread its row for all 16
//    tokens; fused epilogues (store, residual add, SiLU(gate)*up into the
//    next GEMV's B layout, expert-output scatter, LM-head argmax).
//  * warp 4 lane 0: TMA producer.  Weights of dense matrices (and of the
//    expert down projection, whose active list is final once the gate/up
//    kernel passed its griddepcontrol.wait) are requested BEFORE
//    griddepcontrol.wait, so the first 96 KB per SM (14 MB over the chip)
//    stream in while the previous latency-bound kernel is still running.
//  * warp 5: TMEM allocation (32 columns = two 128x16 fp32 accumulators,
//    double-buffered against the epilogue); lane 0 issues tcgen05.mma
//    (M=128, N=16, K=16, bf16 in, fp32 accumulate) and tcgen05.commit to
//    the ring's empty barriers and the accumulator-full barriers.
//
// Work split, invariant to routing and to T: each active block (expert)
// is cut into P equal pieces of its flat (unit, k-step) range, P fixed by
// the block shape; item (block slot b, piece q) goes to CTA
// (b*P + q) mod grid.  With P = grid every CTA streams exactly U pieces
// whatever the router chose.  A unit split between pieces is reduced by
// the last-arriving piece in piece order.  Every sum is therefore a fixed
// function of (row, token): no float atomics, deterministic, and a token's
// logits do not depend on how many drafts ride along (lossless greedy
// speculative decoding needs exactly that).
#pragma once

#include "common.cuh"

namespace cascade {

constexpr int kURows = 128;                       // UMMA M: rows per unit
constexpr int kUTok = 16;                         // UMMA N: token slots
constexpr int kUKsA = kURows * 16 * 2;            // 4 KB of weights per k-step
constexpr int kUKsB = kUTok * 16 * 2;             // 512 B of activations per k-step
#ifndef CASCADE_USTAGE_KS
#define CASCADE_USTAGE_KS 8
#endif
#ifndef CASCADE_USTAGES
#define CASCADE_USTAGES 3
#endif
constexpr int kUStageKs = CASCADE_USTAGE_KS;      // k-steps per ring stage
constexpr int kUStages = CASCADE_USTAGES;         // 96 KB of weights in flight per SM
constexpr int kUStageA = kUStageKs * kUKsA;       // 16 KB
constexpr int kUStageBytes = kUStageA + kUStageKs * kUKsB;  // + 2 KB
constexpr int kUThreads = 192;
constexpr int kUMinPieceKs = 16;                  // >= 64 KB of weights per piece
constexpr int kUPartialFloats = kURows * kUTok;   // one split-unit partial (8 KB)

constexpr int gemv_umma_smem_bytes() { return kUStages * kUStageBytes; }

// element (row, col) of a [rows, K] weight matrix in the A layout (bf16 index)
__host__ __device__ __forceinline__ long long umma_a_index(long long row, int col, int n_ks) {
    const long long unit = row >> 7;
    const int r = (int)(row & 127);
    const int s = col >> 4, kc = (col >> 3) & 1, e = col & 7;
    return (((unit * n_ks + s) * 2 + kc) * kURows + r) * 8 + e;
}
// element (tok, k) of a [16, K] activation in the B layout (bf16 index)
__host__ __device__ __forceinline__ long long umma_b_index(int tok, int k) {
    const int s = k >> 4, kc = (k >> 3) & 1, e = k & 7;
    return (((long long)s * 2 + kc) * kUTok + tok) * 8 + e;
}

enum UEpi : int {
    UEPI_STORE = 0,   // out[tok*ld + row] = v
    UEPI_ADD = 1,     // out[tok*ld + row] += v      (residual)
    UEPI_GATEUP = 2,  // H[slot] (B layout, bf16) = silu(gate) * up
    UEPI_DOWN = 3,    // ycontrib[(tok*n_contrib + rank)*ld + row] = v
    UEPI_ARGMAX = 4,  // keys[tok] = max(argmax_key(v, row)); optional logits store
};

struct UGemvParams {
    const uint16_t* W;         // A layout, local block 0
    long long w_block_stride;  // bf16 elements between blocks
    const uint16_t* B;         // B layout activations, list slot 0
    long long b_block_stride;  // bf16 elements between list slots (0: shared X)
    const int* list;           // active block ids, or nullptr (identity)
    const int* count;          // device U, or nullptr (use n_blocks)
    int n_blocks;
    int n_st;                  // units per block (rows / 128)
    int n_ks;                  // k-steps per unit (K / 16)
    int T;                     // tokens in flight
    int early_list;            // list/count final before griddepcontrol.wait
    float* partial;            // [slots][P][2][128][16]
    int* counters;             // [slots][n_st] arrival counters (zero between launches)
    float* out;
    int ld;
    uint16_t* hout;            // UEPI_GATEUP output (B layout)
    long long h_block_stride;  // bf16 elements between list slots
    const int* route_rank;     // UEPI_DOWN: [slot][16] -> rank in token's list or -1
    int n_contrib;
    unsigned long long* keys;  // UEPI_ARGMAX
    unsigned long long* stamp; // optional globaltimer stamp at kernel start
    unsigned long long* trace; // in-graph trace slot
    unsigned long long* dbg;   // optional phase stamps (scripts/umma_probe.cu)
    int no_prologue;           // A/B: issue nothing before griddepcontrol.wait
    int ring_stages;           // dense_gemv_cluster_kernel: ring depth (<= kCMaxStages)
    int stage_ks;              // dense_gemv_cluster_kernel: k-steps per ring stage (<= kCMaxStageKs)
    int pf_self;               // dense_gemv_cluster_kernel: L2-prefetch the k-range beyond the ring before the wait
    int no_trigger;            // 1: dependents launch at exit, not right after the wait
    int pf_ahead;              // rolling L2 prefetch: weights of the stage this many stages ahead of the ring
};

// phase stamps for the probe: slot i <- globaltimer (CTA 0), or max/min over CTAs
__device__ __forceinline__ void udbg(const UGemvParams& p, int i) {
    if (p.dbg != nullptr && blockIdx.x == 0) p.dbg[i] = globaltimer_raw();
}

// ---------------------------------------------------------------- PTX
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mb_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nUW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra UW_%=;\n}\n" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void l2_prefetch_bulk(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void nbar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major, no swizzle (Blackwell version 1)
__device__ __forceinline__ uint64_t umma_desc(const void* smem, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((su32(smem) >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version
    return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}
// instruction descriptor: D f32, A/B bf16, both K-major, N = 16, M = 128
constexpr uint32_t kUIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kUTok >> 3) << 17) |
                             ((uint32_t)(kURows >> 4) << 24);

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(kUIdesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// ---------------------------------------------------------------- work split
struct UWork {
    int P;                // pieces per block
    long long per_block;  // k-steps per block
    int n_items;          // U * P
};
__device__ __forceinline__ UWork uwork(const UGemvParams& p, int U) {
    UWork w;
    w.per_block = (long long)p.n_st * p.n_ks;
    // dense: spread over every SM; routed blocks: pieces of >= half a unit
    // so a unit is reduced from at most ~3 partials
    long long min_piece = kUMinPieceKs;
    if (p.list != nullptr && p.n_ks / 2 > min_piece) min_piece = p.n_ks / 2;
    long long pm = w.per_block / min_piece;
    if (pm < 1) pm = 1;
    w.P = pm < (long long)gridDim.x ? (int)pm : (int)gridDim.x;
    w.n_items = U * w.P;
    return w;
}
__device__ __forceinline__ long long piece_lo(const UWork& w, int q) { return w.per_block * q / w.P; }
__device__ __forceinline__ int piece_of(const UWork& w, long long pos) {
    return (int)(((pos + 1) * w.P + w.per_block - 1) / w.per_block) - 1;
}

__device__ __forceinline__ float silu_f(float x) { return x / (1.0f + __expf(-x)); }

// Epilogue of one unit row (thread = row r of the unit, v = 16 token values).
template <int EPI>
__device__ __forceinline__ void uepilogue(const UGemvParams& p, int b, int st, int r, float (&v)[16]) {
    const int lane = threadIdx.x & 31;
    const long long row = (long long)st * kURows + r;
    if constexpr (EPI == UEPI_ADD) {
        // residual add: every token's old value is loaded before any store (a
        // load-add-store per token in sequence could not be reordered by the
        // compiler - the token rows might alias - and put T dependent L2
        // round trips into the O projection's epilogue)
        if (p.T == 1) {
            p.out[row] += v[0];
        } else {
            float old[16];
#pragma unroll
            for (int t = 0; t < 16; ++t)
                if (t < p.T) old[t] = p.out[(long long)t * p.ld + row];
#pragma unroll
            for (int t = 0; t < 16; ++t)
                if (t < p.T) p.out[(long long)t * p.ld + row] = old[t] + v[t];
        }
    } else if constexpr (EPI == UEPI_STORE) {
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            if (t >= p.T) break;
            p.out[(long long)t * p.ld + row] = v[t];
        }
    } else if constexpr (EPI == UEPI_GATEUP) {
        // 16-row groups: rows 0-7 gate j..j+7, rows 8-15 up j..j+7 (same warp)
        float up[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) up[t] = __shfl_down_sync(0xffffffffu, v[t], 8);
        if ((r & 15) < 8) {
            const int j = st * (kURows / 2) + (r >> 4) * 8 + (r & 7);
            uint16_t* H = p.hout + (long long)b * p.h_block_stride;
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                const float h = t < p.T ? silu_f(v[t]) * up[t] : 0.0f;
                H[umma_b_index(t, j)] = bf16_bits(h);
            }
        }
    } else if constexpr (EPI == UEPI_DOWN) {
        const int* rr = p.route_rank + b * kMaxT;
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            if (t >= p.T) break;
            const int rank = rr[t];
            if (rank >= 0) p.out[((long long)t * p.n_contrib + rank) * p.ld + row] = v[t];
        }
    } else if constexpr (EPI == UEPI_ARGMAX) {
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            if (t >= p.T) break;
            if (p.out != nullptr) p.out[(long long)t * p.ld + row] = v[t];
            unsigned long long best = argmax_key(v[t], (int)row);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
                best = other > best ? other : best;
            }
            if (lane == 0) atomicMax(p.keys + t, best);
        }
    }
    (void)lane;
}

// PROBE != 0 only in scripts/umma_probe.cu (bottleneck isolation): 1 = no
// tcgen05.mma (plain arrivals), 2 = no activation copies.
template <int EPI, int PROBE = 0>
__global__ void __launch_bounds__(kUThreads, 1) stream_gemv_umma_kernel(UGemvParams p) {
    extern __shared__ __align__(1024) unsigned char ring[];
    __shared__ __align__(8) uint64_t full_bar[kUStages];
    __shared__ __align__(8) uint64_t empty_bar[kUStages];
    __shared__ __align__(8) uint64_t accf_bar[2];
    __shared__ __align__(8) uint64_t acce_bar[2];
    __shared__ uint32_t tmem_base_sh;
    __shared__ int last_sh;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kUStages; ++i) {
            mb_init(&full_bar[i], 1);
            mb_init(&empty_bar[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mb_init(&accf_bar[i], 1);
            mb_init(&acce_bar[i], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tmem_base_sh))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    if (threadIdx.x == 0) {
        udbg(p, 0);
        if (p.dbg) atomicMin(p.dbg + 10, globaltimer_raw());
    }

    const bool dense = p.list == nullptr && p.count == nullptr;
    const bool early = dense || p.early_list;  // weights addressable before griddepcontrol.wait
    const int grid = gridDim.x;

    if (warp == 4) {
        // ------------------------------------------------------------ TMA producer
        {
            uint64_t pol_a, pol_b;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_a));
            asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_b));
            int U = early ? (dense ? p.n_blocks : *p.count) : 0;
            UWork w = uwork(p, U);
            int item = blockIdx.x;
            long long pos = 0, hi = 0;
            int b = 0;
            int i = 0;            // stage sequence number
            int n_pre = 0;        // stages whose B copy is still owed (prologue)
            long long pre_b_off[kUStages];
            int pre_b_slot[kUStages];
            uint32_t pre_b_bytes[kUStages];
            // next stage of this CTA's item sequence; false when done
            auto next_stage = [&](int& bb, long long& p0, int& n) -> bool {
                while (pos >= hi) {
                    if (item >= w.n_items) return false;
                    b = item / w.P;
                    const int q = item - b * w.P;
                    pos = piece_lo(w, q);
                    hi = piece_lo(w, q + 1);
                    item += grid;
                }
                const long long unit_end = (pos / p.n_ks + 1) * p.n_ks;
                long long lim = (hi < unit_end ? hi : unit_end) - pos;
                n = lim < kUStageKs ? (int)lim : kUStageKs;
                p0 = pos;
                bb = b;
                pos += n;
                return true;
            };
            auto issue = [&](int limit, bool with_b) {
                int bb, n;
                long long p0;
                while (i < limit && next_stage(bb, p0, n)) {
                    const int slot = i % kUStages;
                    if (i >= kUStages) mb_wait(&empty_bar[slot], ((i / kUStages) - 1) & 1);
                    const int blk = p.list ? p.list[bb] : bb;
                    const uint16_t* a = p.W + (long long)blk * p.w_block_stride + p0 * (kUKsA / 2);
                    const long long ks = p0 % p.n_ks;
                    const long long b_off = (long long)bb * p.b_block_stride + ks * (kUKsB / 2);
                    unsigned char* dst = ring + (size_t)slot * kUStageBytes;
                    mb_expect_tx(&full_bar[slot], (uint32_t)n * (PROBE == 2 ? kUKsA : kUKsA + kUKsB));
                    bulk_g2s(dst, a, (uint32_t)n * kUKsA, &full_bar[slot], pol_a);
                    if (with_b && p.pf_ahead > 0) {
                        // rolling L2 prefetch: the piece's weights pf_ahead stages ahead
                        // (flat (unit, k-step) positions are contiguous in the A layout)
                        const long long f0 = p0 + (long long)p.pf_ahead * kUStageKs;
                        if (f0 < hi) {
                            const long long f1 = f0 + kUStageKs < hi ? f0 + kUStageKs : hi;
                            l2_prefetch_bulk(p.W + (long long)blk * p.w_block_stride + f0 * (kUKsA / 2), (uint32_t)(f1 - f0) * kUKsA);
                        }
                    }
                    if (PROBE == 2) {
                    } else if (with_b) {
                        bulk_g2s(dst + kUStageA, p.B + b_off, (uint32_t)n * kUKsB, &full_bar[slot], pol_b);
                    } else {
                        pre_b_off[n_pre] = b_off;
                        pre_b_slot[n_pre] = slot;
                        pre_b_bytes[n_pre] = (uint32_t)n * kUKsB;
                        ++n_pre;
                    }
                    ++i;
                }
            };
            if (early && lane == 0 && !p.no_prologue) issue(kUStages, false);  // PDL prologue: weights overlap the predecessor's tail
            griddep_wait();
            if (!p.no_trigger) griddep_launch();
            if (lane != 0) goto producer_done;
            udbg(p, 1);
            for (int j = 0; j < (PROBE == 2 ? 0 : n_pre); ++j)
                bulk_g2s(ring + (size_t)pre_b_slot[j] * kUStageBytes + kUStageA, p.B + pre_b_off[j], pre_b_bytes[j],
                         &full_bar[pre_b_slot[j]], pol_b);
            if (!early) {
                U = p.count ? *p.count : p.n_blocks;
                w = uwork(p, U);
            }
            if (p.pf_ahead > 0 && pos < hi) {
                // fill the prefetch window once (the per-stage prefetch keeps it pf_ahead stages deep)
                const int blk = p.list ? p.list[b] : b;
                const long long f1 = pos + (long long)p.pf_ahead * kUStageKs < hi ? pos + (long long)p.pf_ahead * kUStageKs : hi;
                for (long long f = pos; f < f1; f += kUStageKs) {
                    const long long e = f + kUStageKs < f1 ? f + kUStageKs : f1;
                    l2_prefetch_bulk(p.W + (long long)blk * p.w_block_stride + f * (kUKsA / 2), (uint32_t)(e - f) * kUKsA);
                }
            }
            issue(0x7fffffff, true);
            udbg(p, 2);
        }
    producer_done:;
    } else if (warp == 5) {
        // ------------------------------------------------------------ MMA issuer
        griddep_wait();
        if (!p.no_trigger) griddep_launch();
        if (lane == 0) {
            const int U = p.count ? *p.count : p.n_blocks;
            const UWork w = uwork(p, U);
            int i = 0, v = -1;
            udbg(p, 3);
            for (int item = blockIdx.x; item < w.n_items; item += grid) {
                const int q = item % w.P;
                long long pos = piece_lo(w, q);
                const long long hi = piece_lo(w, q + 1);
                while (pos < hi) {
                    const long long unit_end = (pos / p.n_ks + 1) * p.n_ks;
                    const long long seg_end = hi < unit_end ? hi : unit_end;
                    ++v;
                    const int a = v & 1;
                    if (v >= 2) mb_wait(&acce_bar[a], ((v >> 1) - 1) & 1);
                    tc_fence_after();
                    const uint32_t d = tmem + (uint32_t)(a * kUTok);
                    bool first = true;
                    while (pos < seg_end) {
                        const long long lim = seg_end - pos;
                        const int n = lim < kUStageKs ? (int)lim : kUStageKs;
                        const int slot = i % kUStages;
                        mb_wait(&full_bar[slot], (i / kUStages) & 1);
                        tc_fence_after();
                        const unsigned char* st = ring + (size_t)slot * kUStageBytes;
                        if (PROBE == 1) {
                            mb_arrive(&empty_bar[slot]);
                        } else {
                            for (int j = 0; j < n; ++j) {
                                const uint64_t da = umma_desc(st + j * kUKsA, 2048, 128);
                                const uint64_t db = umma_desc(st + kUStageA + j * kUKsB, 256, 128);
                                umma_bf16(d, da, db, first ? 0u : 1u);
                                first = false;
                            }
                            umma_commit(&empty_bar[slot]);
                        }
                        pos += n;
                        ++i;
                    }
                    if (PROBE == 1) mb_arrive(&accf_bar[a]);
                    else umma_commit(&accf_bar[a]);
                }
            }
            udbg(p, 4);
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ epilogue (warps 0-3)
        griddep_wait();
        if (!p.no_trigger) griddep_launch();
        trace_start(p.trace);
        if (p.stamp != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *p.stamp = globaltimer();
        if (threadIdx.x == 0) udbg(p, 5);
        const int U = p.count ? *p.count : p.n_blocks;
        const UWork w = uwork(p, U);
        const int r = warp * 32 + lane;  // TMEM lane = unit row
        int v = -1;
        for (int item = blockIdx.x; item < w.n_items; item += grid) {
            const int b = item / w.P;
            const int q = item - b * w.P;
            const long long lo = piece_lo(w, q), hi = piece_lo(w, q + 1);
            for (long long u = lo / p.n_ks; u * p.n_ks < hi; ++u) {
                const long long us = u * p.n_ks, ue = us + p.n_ks;
                ++v;
                const int a = v & 1;
                mb_wait(&accf_bar[a], (v >> 1) & 1);
                tc_fence_after();
                float val[16];
                if (v == 0 && threadIdx.x == 0) udbg(p, 6);
                tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(a * kUTok), val);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mb_arrive(&acce_bar[a]);
                const int st = (int)u;
                if (us >= lo && ue <= hi) {
                    uepilogue<EPI>(p, b, st, r, val);
                    continue;
                }
                // unit split between pieces: publish, last arriver reduces in piece order
                const int which = (u == lo / p.n_ks) ? 0 : 1;
                float* mine = p.partial + (((long long)b * w.P + q) * 2 + which) * kUPartialFloats + r * kUTok;
#pragma unroll
                for (int t = 0; t < 16; t += 4)
                    __stcg(reinterpret_cast<float4*>(mine + t), make_float4(val[t], val[t + 1], val[t + 2], val[t + 3]));
                __threadfence();
                nbar(1, 128);
                const int q0 = piece_of(w, us), q1 = piece_of(w, ue - 1);
                if (threadIdx.x == 0) last_sh = atomicAdd(p.counters + (long long)b * p.n_st + u, 1) == q1 - q0;
                nbar(1, 128);
                if (!last_sh) continue;
                __threadfence();
#pragma unroll
                for (int t = 0; t < 16; ++t) val[t] = 0.f;
                for (int qq = q0; qq <= q1; ++qq) {
                    const int wh = (u == piece_lo(w, qq) / p.n_ks) ? 0 : 1;
                    const float* src = p.partial + (((long long)b * w.P + qq) * 2 + wh) * kUPartialFloats + r * kUTok;
#pragma unroll
                    for (int t = 0; t < 16; t += 4) {
                        const float4 x = __ldcg(reinterpret_cast<const float4*>(src + t));
                        val[t] += x.x;
                        val[t + 1] += x.y;
                        val[t + 2] += x.z;
                        val[t + 3] += x.w;
                    }
                }
                if (threadIdx.x == 0) p.counters[(long long)b * p.n_st + u] = 0;
                uepilogue<EPI>(p, b, st, r, val);
            }
        }
    }
    if (threadIdx.x == 0) udbg(p, 7);
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0 && p.dbg) atomicMax(p.dbg + 9, globaltimer_raw());
    if (threadIdx.x == 0) {
        unsigned long long* c = cta_trace_slot(p.trace);
        if (c != nullptr) c[1] = globaltimer_raw();
    }
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem) : "memory");
    }
}


// ---------------------------------------------------------------- cluster split-K (dense, few units)
// Dense matrices with fewer 128-row units than SMs (QKV, O projection) are
// split along K inside a thread-block cluster: unit u = cluster u, CTA rank
// r of C streams k-steps [n_ks*r/C, n_ks*(r+1)/C).  The C partial
// accumulators are reduced through distributed shared memory instead of
// global partials + fences + atomics (the last-arriver chain of the
// stream-K path costs ~4 global round trips at the end of every launch):
// every CTA sends row i of its partial to the CTA that owns row i
// (owner = i*C/128) with st.async, completing on the owner's mbarrier, and
// the owner sums the C partials in rank order and runs the epilogue for
// its rows.  Deterministic; the split depends only on the matrix shape.
constexpr int kCMaxC = 8;
constexpr int kCMaxStages = 6;
constexpr int kCRecvFloats = (kURows + kCMaxC) * kUTok;  // sum over ranks of owned rows * 16

// Ring stages of the split-K engine are sized at launch: QKV, whose
// predecessor (the one-CTA residual combine) leaves the SMs free, streams
// 3 x 64 KB stages (225 KB of shared memory); the O projection keeps
// 3 x 32 KB so that its CTAs fit beside the attention CTAs they follow and
// prefetch their weights under them (PDL prologue).
constexpr int kCMaxStageKs = 16;
__host__ __device__ constexpr int dense_cluster_stage_bytes(int stage_ks) { return stage_ks * (kUKsA + kUKsB); }
constexpr int dense_cluster_smem_bytes(int stages, int stage_ks = kUStageKs) {
    return stages * dense_cluster_stage_bytes(stage_ks) + kCRecvFloats * 4;
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_v4(uint32_t raddr, float4 v, uint32_t rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
        "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(rbar)
        : "memory");
}
__device__ __forceinline__ void cluster_sync_relaxed() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// first row owned by rank j of C (rows i with i*C/128 == j)
__device__ __forceinline__ int owner_row0(int j, int C) { return (kURows * j + C - 1) / C; }

template <int EPI>
__global__ void __launch_bounds__(kUThreads, 1) dense_gemv_cluster_kernel(UGemvParams p) {
    static_assert(EPI == UEPI_STORE || EPI == UEPI_ADD, "cluster split-K: row-local epilogues only");
    extern __shared__ __align__(1024) unsigned char ring[];
    const int NS = p.ring_stages;
    const int SK = p.stage_ks;                          // k-steps per stage
    const int SB = dense_cluster_stage_bytes(SK), SA = SK * kUKsA;
    float* recv = reinterpret_cast<float*>(ring + (size_t)NS * SB);  // [src][own row][16]
    __shared__ __align__(8) uint64_t full_bar[kCMaxStages];
    __shared__ __align__(8) uint64_t empty_bar[kCMaxStages];
    __shared__ __align__(8) uint64_t acc_bar;
    __shared__ __align__(8) uint64_t recv_bar;
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int C = (int)(gridDim.x / (unsigned)p.n_st);  // cluster size
    const int rank = (int)cluster_rank();
    const int unit = (int)cluster_id_x();
    const int ks_lo = p.n_ks * rank / C, ks_hi = p.n_ks * (rank + 1) / C;
    const int my_row0 = owner_row0(rank, C), my_rows = owner_row0(rank + 1, C) - my_row0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            mb_init(&full_bar[i], 1);
            mb_init(&empty_bar[i], 1);
        }
        mb_init(&acc_bar, 1);
        mb_init(&recv_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mb_expect_tx(&recv_bar, (uint32_t)(C * my_rows * kUTok * 4));
    }
    if (warp == 5) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tmem_base_sh))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // every CTA's receive barrier is initialised before anyone can send
    cluster_sync_relaxed();
    const uint32_t tmem = tmem_base_sh;

    if (warp == 4) {
        // ------------------------------------------------------------ TMA producer
        uint64_t pol_a, pol_b;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_a));
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_b));
        const uint16_t* a_base = p.W + ((long long)unit * p.n_ks) * (kUKsA / 2);
        const int n_stages = (ks_hi - ks_lo + SK - 1) / SK;
        auto stage_n = [&](int i) { return min(SK, ks_hi - (ks_lo + i * SK)); };
        // PDL prologue: the weights do not depend on the predecessor
        const int n_pre = min(NS, n_stages);
        if (lane == 0 && !p.no_prologue) {
            for (int i = 0; i < n_pre; ++i) {
                const int n = stage_n(i);
                mb_expect_tx(&full_bar[i], (uint32_t)n * (kUKsA + kUKsB));
                bulk_g2s(ring + (size_t)i * SB, a_base + (long long)(ks_lo + i * SK) * (kUKsA / 2),
                         (uint32_t)n * kUKsA, &full_bar[i], pol_a);
            }
            if (p.pf_self) {
                // the rest of this CTA's weights -> L2 while the latency-bound predecessor runs
                const char* src = reinterpret_cast<const char*>(a_base + (long long)(ks_lo + n_pre * SK) * (kUKsA / 2));
                const long long bytes = (long long)(ks_hi - (ks_lo + n_pre * SK)) * kUKsA;
                for (long long off = 0; off < bytes; off += 32768) {
                    const uint32_t sz = (uint32_t)(bytes - off < 32768 ? bytes - off : 32768);
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + off), "r"(sz) : "memory");
                }
            }
        }
        griddep_wait();
        if (!p.no_trigger) griddep_launch();
        if (lane == 0) {
            // rolling L2 prefetch: the ring holds NS stages in flight per SM (the
            // shared carveout caps it), so the weights of the next pf_ahead stages
            // are requested into L2 ahead of their ring slot
            auto pf_stage = [&](int j) {
                if (j < n_stages)
                    l2_prefetch_bulk(a_base + (long long)(ks_lo + j * SK) * (kUKsA / 2), (uint32_t)stage_n(j) * kUKsA);
            };
            const int i0 = p.no_prologue ? 0 : n_pre;
            for (int j = i0; j < i0 + p.pf_ahead; ++j) pf_stage(j);
            for (int i = 0; i < n_stages; ++i) {
                const int slot = i % NS;
                const int n = stage_n(i);
                const int ks = ks_lo + i * SK;
                unsigned char* dst = ring + (size_t)slot * SB;
                if (i >= i0 && p.pf_ahead > 0) pf_stage(i + p.pf_ahead);
                if (i >= n_pre || p.no_prologue) {
                    if (i >= NS) mb_wait(&empty_bar[slot], ((i / NS) - 1) & 1);
                    mb_expect_tx(&full_bar[slot], (uint32_t)n * (kUKsA + kUKsB));
                    bulk_g2s(dst, a_base + (long long)ks * (kUKsA / 2), (uint32_t)n * kUKsA, &full_bar[slot], pol_a);
                }
                bulk_g2s(dst + SA, p.B + (long long)ks * (kUKsB / 2), (uint32_t)n * kUKsB, &full_bar[slot], pol_b);
            }
        }
    } else if (warp == 5) {
        // ------------------------------------------------------------ MMA issuer
        griddep_wait();
        if (!p.no_trigger) griddep_launch();
        if (lane == 0) {
            const int n_stages = (ks_hi - ks_lo + SK - 1) / SK;
            bool first = true;
            for (int i = 0; i < n_stages; ++i) {
                const int slot = i % NS;
                const int n = min(SK, ks_hi - (ks_lo + i * SK));
                mb_wait(&full_bar[slot], (i / NS) & 1);
                tc_fence_after();
                const unsigned char* st = ring + (size_t)slot * SB;
                for (int j = 0; j < n; ++j) {
                    const uint64_t da = umma_desc(st + j * kUKsA, 2048, 128);
                    const uint64_t db = umma_desc(st + SA + j * kUKsB, 256, 128);
                    umma_bf16(tmem, da, db, first ? 0u : 1u);
                    first = false;
                }
                umma_commit(&empty_bar[slot]);
            }
            umma_commit(&acc_bar);
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ epilogue (warps 0-3, thread = row)
        griddep_wait();
        if (!p.no_trigger) griddep_launch();
        trace_start(p.trace);
        if (p.stamp != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *p.stamp = globaltimer();
        phase_stamp(p.trace, 0);  // CTA 0 (diagnostic): 1 accumulator ready, 2 partials received, 3 epilogue done
        const int r = warp * 32 + lane;
        mb_wait(&acc_bar, 0);
        tc_fence_after();
        phase_stamp(p.trace, 1);
        float val[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), val);
        tc_fence_before();
        // send row r's partial to its owner
        const int own = r * C / kURows;
        const uint32_t laddr = su32(recv + ((size_t)rank * (owner_row0(own + 1, C) - owner_row0(own, C)) +
                                            (r - owner_row0(own, C))) * kUTok);
        // recv layout of owner `own`: [src rank][own rows][16]
        const uint32_t raddr = mapa_shared(laddr, (uint32_t)own);
        const uint32_t rbar = mapa_shared(su32(&recv_bar), (uint32_t)own);
#pragma unroll
        for (int q = 0; q < 4; ++q)
            st_async_v4(raddr + q * 16, make_float4(val[4 * q], val[4 * q + 1], val[4 * q + 2], val[4 * q + 3]), rbar);
        if (r >= my_row0 && r < my_row0 + my_rows) {
            mb_wait(&recv_bar, 0);
            phase_stamp(p.trace, 2);
            float acc[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) acc[t] = 0.f;
            for (int src = 0; src < C; ++src) {
                const float4* f = reinterpret_cast<const float4*>(recv + ((size_t)src * my_rows + (r - my_row0)) * kUTok);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float4 x = f[q];
                    acc[4 * q] += x.x;
                    acc[4 * q + 1] += x.y;
                    acc[4 * q + 2] += x.z;
                    acc[4 * q + 3] += x.w;
                }
            }
            uepilogue<EPI>(p, 0, unit, r, acc);
            phase_stamp(p.trace, 3);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long* c = cta_trace_slot(p.trace);
        if (c != nullptr) c[1] = globaltimer_raw();
    }
    if (warp == 5) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem) : "memory");
    }
}

}  // namespace cascade
