// ffn_ring.cuh — fused expert FFN (gate/up + SiLU, then down) with one TMA
// stream per CTA (option; CASCADE_FFN_RING=1).
//
// The register-direct engine (gemv.cuh expert_ffn_kernel) splits a CTA's
// piece of the flat (slot, super-tile, k-step) range into 8 contiguous warp
// ranges, each warp streaming its own LDG.128s.  The memory system serves
// the 16 warps of an SM unevenly: per layer the last warp of a CTA ends
// 4.5 us (Mixtral K=0) to 10 us (K=8) after the first (scripts/warp_spread.py,
// profiles/r02b), and the piece-level reduction, the cross-CTA partials and
// the readiness publish all wait for it.
//
// Here one CTA per SM streams its piece through a 6 x 16 KB shared-memory
// ring with cp.async.bulk (one producer lane, 96 KB in flight per SM: HBM
// saturates with every SM streaming, profiles/r02b/per_sm_bw_probe.txt), in
// piece order, so there is a single stream per SM and no straggler warp.
//  * 4 stream warps consume every stage in lockstep with the ring, warp w
//    taking k-steps 2w, 2w+1 of each 8-k-step stage (A-fragments from shared
//    memory, conflict-free LDS.128; B-fragments from L1/L2); each keeps its
//    partial of the current super-tile in registers;
//  * at the end of a super-tile's part in the piece the 4 partials go to a
//    shared buffer and a finaliser warp sums them in warp order (so every
//    sum is a fixed function of (U, grid)) and runs the epilogue (SiLU*up
//    into the down projection's B operand, or the expert-output scatter),
//    the cross-CTA piece partial + acq_rel arrival for a super-tile shared
//    with a neighbouring piece, and for gate/up the release add on the
//    slot's readiness counter, while the stream warps go on with the next
//    super-tile;
//  * the producer runs straight on into the down projection's stages (the
//    weights do not depend on the gate/up results), so the ring holds down
//    weights while the stream warps wait for a slot's readiness.
#pragma once

#include "gemv.cuh"
#include "gemv_umma.cuh"

namespace cascade {

constexpr int kRingStream = 4;                   // stream (consumer) warps 0-3
constexpr int kRingProducerWarp = kRingStream;   // warp 4: weight (A) producer
constexpr int kRingFinalWarp = kRingStream + 1;  // warp 5: finaliser
constexpr int kRingBWarp = kRingStream + 2;      // warp 6 (T > 8 only): B-operand producer
constexpr int kRingStages = 3;
constexpr int kBStepBytes = 2 * 32 * 8;          // B-frag bytes per k-step (both n8 token tiles)

// Per token-tile geometry.  Up to 8 tokens (NT = 1) the token block fits
// L1 and each stream warp loads its B-fragments itself (one stage of
// look-ahead); with 9-16 tokens (NT = 2, up to 128 KB) it does not, and a
// CTA sweeps the whole k-range once per super-tile, so every B load would
// go to L2 under the weight stream: there the stage carries the B slice
// too, copied by a second producer (which also owns the down phase's
// readiness wait), and stages are 12 k-steps to fit the 132 KB carveout.
template <int NT>
struct RingCfg {
    static constexpr bool kBInStage = NT == 2;
    static constexpr int kWarpKs = NT == 1 ? 4 : 3;                 // k-steps of a stage per stream warp
    static constexpr int kStageKs = kWarpKs * kRingStream;            // 16 / 12
    static constexpr int kABytes = kStageKs * kTPW * 32 * 16;         // 32 / 24 KB of weights
    static constexpr int kStageBytes = kABytes + (kBInStage ? kStageKs * kBStepBytes : 0);
    static constexpr int kThreads = 32 * (kRingStream + (kBInStage ? 3 : 2));
    static constexpr int kSmem = kRingStages * kStageBytes + kRingStream * kTPW * NT * 32 * 16;
};
constexpr int kRingMaxThreads = RingCfg<2>::kThreads;
template <int NT>
constexpr int ffn_ring_smem_bytes() { return RingCfg<NT>::kSmem; }
template <int NT>
constexpr int ffn_ring_threads() { return RingCfg<NT>::kThreads; }

// Geometry of one phase's split (the same pieces as ffn_phase: stream-K,
// batch-invariant, or one super-tile per CTA).
struct RingGeo {
    long long per_block;
    int P, n_items;
};
__device__ __forceinline__ RingGeo ring_geo(const GemvParams& p, int U) {
    RingGeo g;
    g.per_block = (long long)p.n_st * p.n_ks * (p.invariant ? 1 : U);
    const int n_blocks_w = p.invariant ? U : (U > 0 ? 1 : 0);
    g.P = block_pieces(p, g.per_block);
    g.n_items = n_blocks_w * g.P;
    return g;
}

// One stage of the walk: k-steps [ks, ks+n) of super-tile st of slot bl
// (flat unit index `unit`); `ends` marks the last stage of the super-tile's
// part in the current piece.
struct RingStage {
    long long unit;
    int ks, n, bl, st;
    bool ends;
};

// Walks this CTA's stages of one phase: item (block, piece), then stages of
// <= sk k-steps that never cross a super-tile.  Inside a piece the
// two super-tiles shared with the neighbouring pieces go first (the tail
// part, then the head part, then the interior), so their cross-CTA partials
// and arrivals are finished early, under the rest of the stream, and a
// phase ends on an interior super-tile whose finalisation needs no global
// round trip but the readiness publish.  The position advances
// incrementally (64-bit divisions only at segment starts: per 32 KB stage
// they would cost more than the stage's MMAs).
struct RingWalk {
    RingGeo g;
    int n_ks, n_st, item, b, q, sk;
    long long base, clo, chi, pos, seg_end;
    long long seg_lo[3], seg_hi[3];
    int seg, n_seg;
    long long unit;
    int ks, bl, st;
    __device__ void start(const GemvParams& p, int U, int stage_ks) {
        g = ring_geo(p, U);
        n_ks = p.n_ks;
        n_st = p.n_st;
        sk = stage_ks;
        item = (int)blockIdx.x - (int)gridDim.x;
        pos = seg_end = 0;
        seg = n_seg = 0;
    }
    __device__ void enter(long long at) {
        pos = at;
        unit = pos / n_ks;
        ks = (int)(pos - unit * n_ks);
        bl = (int)(unit / n_st);
        st = (int)(unit - (long long)bl * n_st);
    }
    __device__ bool next(const GemvParams& p, RingStage& sg) {
        while (pos >= seg_end) {
            if (seg + 1 < n_seg) {
                ++seg;
            } else {
                item += gridDim.x;
                if (item >= g.n_items) return false;
                b = item / g.P;
                q = item - b * g.P;
                base = (long long)b * g.per_block;
                clo = base + piece_start(g.per_block, q, g.P, p.cum);
                chi = base + piece_start(g.per_block, q + 1, g.P, p.cum);
                if (chi <= clo) {
                    n_seg = 0;
                    continue;
                }
                const long long h1 = (clo / n_ks + 1) * n_ks;   // end of the head super-tile
                const long long t0 = (chi - 1) / n_ks * n_ks;    // start of the tail super-tile
                n_seg = 0;
                if (h1 >= chi) {  // the piece lies in one super-tile
                    seg_lo[n_seg] = clo, seg_hi[n_seg++] = chi;
                } else {
                    seg_lo[n_seg] = t0 > clo ? t0 : clo, seg_hi[n_seg++] = chi;     // tail part
                    if (t0 > clo) seg_lo[n_seg] = clo, seg_hi[n_seg++] = h1;      // head part
                    if (t0 > h1) seg_lo[n_seg] = h1, seg_hi[n_seg++] = t0;        // interior
                }
                seg = 0;
            }
            enter(seg_lo[seg]);
            seg_end = seg_hi[seg];
        }
        const int rem_unit = n_ks - ks;
        const long long rem_seg = seg_end - pos;
        int n = rem_unit < sk ? rem_unit : sk;
        if (rem_seg < n) n = (int)rem_seg;
        sg.unit = unit;
        sg.ks = ks;
        sg.n = n;
        sg.bl = bl;
        sg.st = st;
        sg.ends = n == rem_unit || n == rem_seg;
        pos += n;
        ks += n;
        if (ks == n_ks) {
            ks = 0;
            ++unit;
            if (++st == n_st) {
                st = 0;
                ++bl;
            }
        }
        return true;
    }
};

struct RingSmem {
    uint64_t full[kRingStages], empty[kRingStages];
    uint64_t red_full, red_empty;
    int a_issued;  // stages whose weight copy (and expect_tx) the A producer issued
    unsigned int ready_bits[(kMaxSlots + 31) / 32];
    int poll[kMaxSlots];
};

template <int NT>
__device__ __forceinline__ void ring_producer(const FfnParams& f, const UnionSmem& un, unsigned char* ring, RingSmem& rs) {
    using C = RingCfg<NT>;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    int i = 0;
#pragma unroll 1
    for (int phase = 0; phase < 2; ++phase) {
        const GemvParams& p = phase ? f.dn : f.gu;
        RingWalk w;
        w.start(p, un.count, C::kStageKs);
        RingStage sg;
        if (phase == 1 && f.dn_l2_stages > 0) {
            // Down weights do not depend on gate/up, and HBM idles while the
            // CTAs cross from gate/up to down: optionally the down stages
            // right behind the ring's first ones go to L2 now (A/B: no gain).
            RingWalk pw;
            pw.start(p, un.count, C::kStageKs);
            RingStage ps;
            int k = 0;
            while (k < kRingStages + f.dn_l2_stages && pw.next(p, ps)) {
                if (k++ < kRingStages) continue;
                const uint4* src = p.W + (long long)un.list[ps.bl] * p.w_block_stride + ((long long)ps.st * p.n_ks + ps.ks) * (kTPW * 32);
                l2_prefetch_bulk(src, (uint32_t)ps.n * kTPW * 32 * 16);
            }
        }
        while (w.next(p, sg)) {
            const int n = sg.n;
            const uint4* src = p.W + (long long)un.list[sg.bl] * p.w_block_stride + ((long long)sg.st * p.n_ks + sg.ks) * (kTPW * 32);
            const int slot = i % kRingStages;
            if (i >= kRingStages) mb_wait(&rs.empty[slot], ((i / kRingStages) - 1) & 1);
            mb_expect_tx(&rs.full[slot], (uint32_t)n * (kTPW * 32 * 16 + (C::kBInStage ? kBStepBytes : 0)));
            bulk_g2s(ring + (size_t)slot * C::kStageBytes, src, (uint32_t)n * kTPW * 32 * 16, &rs.full[slot], pol);
            ++i;
            if constexpr (C::kBInStage) {
                // the slot is free and its transaction count is set: the B
                // producer may copy this stage's token slice
                asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(su32(&rs.a_issued)), "r"(i) : "memory");
            }
        }
    }
}

// B-operand producer (T > 8): copies each stage's token slice into the stage
// right behind the weight copy; in the down phase it first waits for the
// slot's readiness (every gate/up super-tile of that expert published), so
// the stream warps never poll.
template <int NT>
__device__ __forceinline__ void ring_b_producer(const FfnParams& f, const UnionSmem& un, unsigned char* ring, RingSmem& rs) {
    using C = RingCfg<NT>;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    unsigned long long ready_mask[(kMaxSlots + 63) / 64] = {};
    int i = 0;
#pragma unroll 1
    for (int phase = 0; phase < 2; ++phase) {
        const GemvParams& p = phase ? f.dn : f.gu;
        RingWalk w;
        w.start(p, un.count, C::kStageKs);
        RingStage sg;
        while (w.next(p, sg)) {
            const int bl = sg.bl;
            if (phase == 1 && !((ready_mask[bl >> 6] >> (bl & 63)) & 1ull)) {
                long long spins = 0;
                for (;;) {
                    int v;
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f.ready + (long long)bl * kReadyStride) : "memory");
                    if (v >= f.n_st_gu) break;
                    if (++spins > (1ll << 24)) __trap();  // a lost producer must not hang the GPU (~seconds)
                    __nanosleep(32);
                }
                // the h stores of other CTAs (generic proxy) before this CTA's bulk copy of them
                asm volatile("fence.proxy.async.global;" ::: "memory");
                ready_mask[bl >> 6] |= 1ull << (bl & 63);
            }
            const int slot = i % kRingStages;
            ++i;
            for (;;) {
                int v;
                asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(su32(&rs.a_issued)) : "memory");
                if (v >= i) break;
                __nanosleep(20);
            }
            const uint2* src = p.B + (long long)bl * p.b_block_stride + (long long)sg.ks * (kBStepBytes / 8);
            bulk_g2s(ring + (size_t)slot * C::kStageBytes + C::kABytes, src, (uint32_t)sg.n * kBStepBytes, &rs.full[slot], pol);
        }
    }
}

// readiness of slot bl (down phase): one poller per CTA and slot, the other
// warps watch the shared bit (as ffn_phase)
__device__ __forceinline__ void ring_wait_ready(const FfnParams& f, RingSmem& rs, int bl,
                                                unsigned long long (&ready_mask)[(kMaxSlots + 63) / 64]) {
    if ((ready_mask[bl >> 6] >> (bl & 63)) & 1ull) return;
    if ((threadIdx.x & 31) == 0) {
        volatile unsigned int* bits = rs.ready_bits;
        const unsigned int bit = 1u << (bl & 31);
        const bool poller = !(bits[bl >> 5] & bit) && atomicCAS(&rs.poll[bl], 0, 1) == 0;
        long long spins = 0;
        for (;;) {
            if (bits[bl >> 5] & bit) break;
            if (poller) {
                int v;
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f.ready + (long long)bl * kReadyStride) : "memory");
                if (v >= f.n_st_gu) {
                    __threadfence_block();
                    atomicOr(&rs.ready_bits[bl >> 5], bit);
                    break;
                }
            }
            if (++spins > (1ll << 24)) __trap();  // a lost producer must not hang the GPU (~seconds)
            __nanosleep(poller ? 32 : 64);
        }
        __threadfence_block();
    }
    __syncwarp();
    ready_mask[bl >> 6] |= 1ull << (bl & 63);
}

// Stream warp w: its k-steps of every stage of both phases (4w..4w+3 of 16
// for NT = 1, 3w..3w+2 of 12 for NT = 2).
template <int NT>
__device__ __forceinline__ void ring_stream(const FfnParams& f, const UnionSmem& un, const unsigned char* ring,
                                            float4* red, RingSmem& rs) {
    using C = RingCfg<NT>;
    constexpr int WK = C::kWarpKs;
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    constexpr int kSlot = kTPW * NT * 32;
    float acc[kTPW][NT][4];
    zero_acc<NT>(acc);
    int i = 0, uc = 0;
    unsigned long long ready_mask[(kMaxSlots + 63) / 64] = {};
#pragma unroll 1
    for (int phase = 0; phase < 2; ++phase) {
        const GemvParams& p = phase ? f.dn : f.gu;
        const bool down = phase == 1;
        RingWalk wk;
        wk.start(p, un.count, C::kStageKs);
        const int k0 = WK * w;
        // NT = 1: B-fragments from L1 with one stage of look-ahead (a stage
        // whose slot still needs its readiness wait loads after it)
        auto load_b = [&](const RingStage& g, uint2 (&bb)[WK][NT]) {
            const uint2* Bp = p.B + (long long)g.bl * p.b_block_stride + lane;
#pragma unroll
            for (int k = 0; k < WK; ++k)
                if (k0 + k < g.n)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
                        bb[k][nt] = down ? ldcg_act(Bp + ((g.ks + k0 + k) * 2 + nt) * 32) : ldg_act(Bp + ((g.ks + k0 + k) * 2 + nt) * 32);
        };
        RingStage sg, sn;
        uint2 bb[WK][NT], bn[WK][NT];
        bool first_stage = true;
        bool have = wk.next(p, sg);
        if (have && !C::kBInStage) {
            if (down) ring_wait_ready(f, rs, sg.bl, ready_mask);
            load_b(sg, bb);
        }
        while (have) {
            const bool have_n = wk.next(p, sn);
            bool pre = false;
            if constexpr (!C::kBInStage) {
                pre = have_n && (!down || ((ready_mask[sn.bl >> 6] >> (sn.bl & 63)) & 1ull));
                if (pre) load_b(sn, bn);
            }
            const int n = sg.n;
            const int slot = i % kRingStages;
            mb_wait(&rs.full[slot], (i / kRingStages) & 1);
            ++i;
            const unsigned char* stage = ring + (size_t)slot * C::kStageBytes;
            if constexpr (C::kBInStage) {
                const uint2* Bs = reinterpret_cast<const uint2*>(stage + C::kABytes) + lane;
#pragma unroll
                for (int k = 0; k < WK; ++k)
                    if (k0 + k < n)
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) bb[k][nt] = Bs[((k0 + k) * 2 + nt) * 32];
            }
            const uint4* S = reinterpret_cast<const uint4*>(stage) + lane;
#pragma unroll
            for (int k = 0; k < WK; ++k) {
                if (k0 + k < n) {
                    uint4 a[kTPW];
#pragma unroll
                    for (int it = 0; it < kTPW; ++it) a[it] = S[((k0 + k) * kTPW + it) * 32];
#pragma unroll
                    for (int it = 0; it < kTPW; ++it)
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) mma_bf16_16816(acc[it][nt], a[it], bb[k][nt]);
                }
            }
            __syncwarp();
            if (lane == 0) mb_arrive(&rs.empty[slot]);
            if (first_stage) {
                phase_stamp(f.gu.trace, down ? 4 : 1);  // CTA 0 warp 0: first stage of the phase consumed
                first_stage = false;
            }
            if (sg.ends) {
                // hand this warp's partial of the super-tile to the finaliser
                if (uc > 0) mb_wait(&rs.red_empty, (uc - 1) & 1);
                store_acc<NT>(red + w * kSlot + lane, acc, false);
                __syncwarp();
                if (lane == 0) mb_arrive(&rs.red_full);
                zero_acc<NT>(acc);
                ++uc;
            }
            if (!have_n) {
                phase_stamp(f.gu.trace, down ? 5 : 2);  // CTA 0 warp 0: last stage of the phase consumed
                break;
            }
            sg = sn;
            if constexpr (!C::kBInStage) {
                if (pre) {
#pragma unroll
                    for (int k = 0; k < WK; ++k)
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) bb[k][nt] = bn[k][nt];
                } else {
                    ring_wait_ready(f, rs, sg.bl, ready_mask);
                    load_b(sg, bb);
                }
            }
        }
    }
}

// Finaliser warp: sums the 4 stream partials of each finished super-tile
// part in warp order and completes it.
template <int NT>
__device__ __forceinline__ void ring_finalise(const FfnParams& f, const UnionSmem& un, const float4* red, RingSmem& rs) {
    const int lane = threadIdx.x & 31;
    constexpr int kSlot = kTPW * NT * 32;
    float acc[kTPW][NT][4];
    int uc = 0;
#pragma unroll 1
    for (int phase = 0; phase < 2; ++phase) {
        const GemvParams& p = phase ? f.dn : f.gu;
        const bool down = phase == 1;
        RingWalk wk;
        wk.start(p, un.count, RingCfg<NT>::kStageKs);
        RingStage sg;
        while (wk.next(p, sg)) {
            if (!sg.ends) continue;
            const long long unit = sg.unit;
            const int bl = sg.bl, st = sg.st;
            mb_wait(&rs.red_full, uc & 1);
            zero_acc<NT>(acc);
#pragma unroll 1
            for (int s = 0; s < kRingStream; ++s) add_acc<NT>(acc, red + s * kSlot + lane, false);
            __syncwarp();
            if (lane == 0) mb_arrive(&rs.red_empty);
            ++uc;
            const signed char* rr = un.rank[bl];
            const long long ustart = unit * p.n_ks, uend = ustart + p.n_ks;
            if (ustart < wk.clo || uend > wk.chi) {
                // shared with a neighbouring piece: piece partial + acq_rel
                // arrival; the last arriver sums the pieces in piece order
                const int first = piece_owner(ustart - wk.base, wk.g.per_block, wk.g.P, p.cum);
                const int last = piece_owner(uend - 1 - wk.base, wk.g.per_block, wk.g.P, p.cum);
                const int gslot = (wk.q == first) ? 1 : 0;
                store_acc<NT>(p.partial + (((long long)wk.b * wk.g.P + wk.q) * 2 + gslot) * kSlot + lane, acc, true);
                __syncwarp();
                int prev = 0;
                if (lane == 0) prev = atomic_add_acq_rel(p.counters + unit, 1);
                prev = __shfl_sync(0xffffffffu, prev, 0);
                if (prev != last - first) continue;
                __syncwarp();
                zero_acc<NT>(acc);
                for (int jj = first; jj <= last; ++jj)
                    add_acc<NT>(acc, p.partial + (((long long)wk.b * wk.g.P + jj) * 2 + (jj == first ? 1 : 0)) * kSlot + lane, true);
                if (lane == 0) p.counters[unit] = 0;
            }
            if (down) {
                gemv_epilogue<NT, EPI_DOWN>(p, bl, st, lane, acc, rr);
            } else {
                gemv_epilogue<NT, EPI_GATEUP>(p, bl, st, lane, acc, rr);
                __syncwarp();  // the super-tile's h stores precede the release
                if (lane == 0) red_add_release(f.ready + (long long)bl * kReadyStride, 1);
            }
        }
        if (phase == 0) cta_phase(f.gu.trace, 2);  // gate/up super-tiles of this CTA finalised
        if (lane == 0) phase_stamp_cta0(f.gu.trace, phase ? 6 : 3);  // CTA 0 finaliser: phase finalised (0 union, 1-2 / 4-5 stream, 3 / 6 final)
    }
}

template <int NT>
__global__ void __launch_bounds__(kRingMaxThreads, 1) expert_ffn_ring_kernel(FfnParams f) {
    using C = RingCfg<NT>;
    extern __shared__ __align__(1024) unsigned char ring[];
    float4* red = reinterpret_cast<float4*>(ring + (size_t)kRingStages * C::kStageBytes);
    __shared__ UnionSmem un;
    __shared__ RingSmem rs;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kRingStages; ++i) {
            mb_init(&rs.full[i], 1);
            mb_init(&rs.empty[i], kRingStream);
        }
        mb_init(&rs.red_full, kRingStream);
        mb_init(&rs.red_empty, 1);
        rs.a_issued = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < (kMaxSlots + 31) / 32; i += blockDim.x) rs.ready_bits[i] = 0u;
    for (int i = threadIdx.x; i < kMaxSlots; i += blockDim.x) rs.poll[i] = 0;
    griddep_wait();
    if (f.gu.trigger) griddep_launch();
    CTA_TRACE(f.gu.trace);
    if (warp == 0) build_union(f.gu, un);
    __syncthreads();
    phase_stamp(f.gu.trace, 0);
    if (f.gu.publish && blockIdx.x == 0) publish_union(f.gu, un);
    if (warp == kRingProducerWarp) {
        if ((threadIdx.x & 31) == 0) ring_producer<NT>(f, un, ring, rs);
    } else if (warp == kRingFinalWarp) {
        ring_finalise<NT>(f, un, red, rs);
    } else if (warp == kRingBWarp) {
        if constexpr (C::kBInStage) {
            if ((threadIdx.x & 31) == 0) ring_b_producer<NT>(f, un, ring, rs);
        }
    } else {
        ring_stream<NT>(f, un, ring, red, rs);
    }
}

}  // namespace cascade
