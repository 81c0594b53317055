// attention.cuh — causal GQA attention of the T = K+1 in-flight tokens over
// the request's KV cache, with RoPE and the KV append fused in
// (SURVEY.md §8(a2) stage K4; replaces the constant attention_time term of
// iteration_cost, proj/include/specsim/expert_model.hpp:159).
//
// Split-KV ("flash-decoding"): work item = (chunk, kv head).  Chunks
// 0..nch-1 cover the committed cache [0, ctx) in kChunk-key slices; chunk
// nch is the T new tokens themselves, whose keys/values are rotated,
// rounded to bf16, appended to the cache and used under the causal mask.
// All G = H/KV query heads of a KV head share the item (R = G*T rows), so
// every K/V byte is read once per step.  QK^T and PV run on mma.m16n8k16
// (bf16 in, fp32 accumulate); one warp owns a 16-row tile and keeps S and
// O in registers (the S accumulator is re-packed as the P A-fragment).
// Every item writes (max, sum, unnormalised o) per query row; the combine
// kernel merges chunks in fixed order and writes the O-projection input in
// B-frag layout.  ctx is read from device memory, so one captured graph
// serves every context length.
#pragma once

#include "common.cuh"
#include "gemv_umma.cuh"

namespace cascade {

constexpr int kChunk = 64;
constexpr int kAttnThreads = 128;
constexpr int kAttnMaxRows = 128;  // G * T

struct AttnParams {
    const float* qkv;        // [T][(H + 2KV) * hd] fp32
    uint16_t* kc;            // [KV][max_ctx][hd] bf16 (this layer)
    uint16_t* vc;
    const int* ctx_ptr;      // committed cache length
    const float2* rope;      // [T][hd/2] (cos, sin) at position ctx + t (embed kernel)
    float* part;             // [KV][R][max_chunks][hd + 2]
    int T, H, KV, max_ctx, max_chunks;
    float scale;             // 1/sqrt(hd)
    const void* pf;          // weights to prefetch into L2 (the O projection)
    unsigned long long pf_bytes;
    unsigned long long* trace;
    // fused chunk combine: the last item of a KV head to finish merges that
    // head's chunk partials and writes the O-projection input
    int fused;
    int* arrive;             // [KV] item arrivals (zero between launches)
    uint16_t* out_bfrag;     // [T][H*hd] bf16, UMMA B layout (umma) or B-frag
    int umma;
    int ksplit;              // key-split chunk tiles (attn_ksplit_pass; hd >= 64)
};

// rotate_half RoPE on the pair (i, i + hd/2)
__device__ __forceinline__ void rope_pair(float& a, float& b, float2 cs) {
    const float x0 = a, x1 = b;
    a = x0 * cs.x - x1 * cs.y;
    b = x1 * cs.x + x0 * cs.y;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    return (uint32_t)bf16_bits(lo) | ((uint32_t)bf16_bits(hi) << 16);
}

// hi/lo bf16 split of a pair: x ~= hi + lo with ~16 significant bits
__device__ __forceinline__ void split_bf16x2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
    const uint16_t h0 = bf16_bits(x0), h1 = bf16_bits(x1);
    hi = (uint32_t)h0 | ((uint32_t)h1 << 16);
    lo = (uint32_t)bf16_bits(x0 - bits_to_f32(h0)) | ((uint32_t)bf16_bits(x1 - bits_to_f32(h1)) << 16);
}

__device__ __forceinline__ void mma_bf16_regs(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                              uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int HD>
constexpr int attn_smem_bytes(int qrows = kAttnMaxRows) {
    return (2 * qrows + 2 * kChunk) * (HD + 8) * 2 + 3 * (16 * (kChunk + 8) * 4 + 64 * 4);  // + key-split scratch (kAttnKsplitSmem)
}

// Two-term bf16 operands.  q and P enter the tensor cores as hi + lo bf16
// pairs (hi = bf16(x), lo = bf16(x - hi)), so QK^T and PV carry ~16
// mantissa bits instead of 8: the attention result no longer depends on
// which keys share a 64-key chunk (i.e. on T), and matches an fp32/fp64
// softmax to ~1e-5.  K and V are bf16 in the cache, so they need one term.
//
// smem (bf16, row stride HD+8 -> conflict-free fragment loads):
//   q_hi [kAttnMaxRows][HD+8] | q_lo [..] | k [kChunk][HD+8] | v [kChunk][HD+8]
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Key-split chunk tiles (p.ksplit, hd >= 64).  The four warps share every
// 16-row tile: warp w computes S for keys [16w, 16w+16) (32 mma instead of
// 128), the chunk row max is exchanged through shared memory so every warp
// exponentiates against the same max (P bitwise equal to the one-warp
// tile), P is staged in fp32, and warp w then runs PV over all 64 keys
// for dims [hd/4 * w, hd/4 * (w+1)) (32 mma instead of 128), splitting P
// into its hi/lo bf16 terms as it loads the fragments.  Up to kAttnKsMt
// row tiles go through one pass (two barriers per pass; the V fragments
// are loaded once per pass).  Warp 0 forms the row sums from the staged P
// in the one-warp tile's order, so the chunk partials (max, sum, o) are
// bitwise those of the one-warp tile.
constexpr int kAttnPLd = kChunk + 8;  // P row stride (fp32): conflict-free 8-byte fragment loads
constexpr int kAttnKsMt = 3;          // row tiles per pass (4: register spills)
constexpr int kAttnKsplitSmem = kAttnKsMt * (16 * kAttnPLd * 4 + 64 * 4);
static_assert(attn_smem_bytes<128>(16) == (2 * 16 + 2 * kChunk) * 136 * 2 + kAttnKsplitSmem, "key-split scratch");

template <int HD, int NM>
__device__ __forceinline__ void attn_ksplit_pass(const AttnParams& p, const uint16_t* qs, const uint16_t* qsl,
                                                 const uint16_t* ks, const uint16_t* vs, uint16_t* scratch,
                                                 int mt0, int R, int nkeys, int key0, int ctx, int kvh, int c) {
    constexpr int LD = HD + 8;
    constexpr int NKS = HD / 16;
    constexpr int NDW = HD / 32;  // n8 dim tiles per warp in PV
    constexpr int MB = NM;  // row tiles of this pass
    constexpr int PT = 16 * kAttnPLd;  // one P tile (fp32)
    float* pe = reinterpret_cast<float*>(scratch);  // [kAttnKsMt][16][kAttnPLd] P (fp32)
    float* red_m = pe + kAttnKsMt * PT;              // [kAttnKsMt][4 warps][16 rows]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;
    {
        constexpr int nm = NM;
        float s[MB][2][4];
#pragma unroll
        for (int u = 0; u < MB; ++u)
#pragma unroll
            for (int nn = 0; nn < 2; ++nn)
#pragma unroll
                for (int q = 0; q < 4; ++q) s[u][nn][q] = 0.f;
#pragma unroll
        for (int kst = 0; kst < NKS; ++kst) {
            const int i0 = kst * 16 + 2 * t4;
            uint32_t b[2][2];
#pragma unroll
            for (int nn = 0; nn < 2; ++nn) {
                const int n = 2 * warp + nn;
                b[nn][0] = *reinterpret_cast<const uint32_t*>(ks + (n * 8 + g) * LD + i0);
                b[nn][1] = *reinterpret_cast<const uint32_t*>(ks + (n * 8 + g) * LD + i0 + 8);
            }
#pragma unroll
            for (int u = 0; u < MB; ++u) {
                if (u >= nm) break;
                const int r0 = (mt0 + u) * 16;
                const uint32_t a0 = *reinterpret_cast<const uint32_t*>(qs + (r0 + g) * LD + i0);
                const uint32_t a1 = *reinterpret_cast<const uint32_t*>(qs + (r0 + g + 8) * LD + i0);
                const uint32_t a2 = *reinterpret_cast<const uint32_t*>(qs + (r0 + g) * LD + i0 + 8);
                const uint32_t a3 = *reinterpret_cast<const uint32_t*>(qs + (r0 + g + 8) * LD + i0 + 8);
                const uint32_t l0 = *reinterpret_cast<const uint32_t*>(qsl + (r0 + g) * LD + i0);
                const uint32_t l1 = *reinterpret_cast<const uint32_t*>(qsl + (r0 + g + 8) * LD + i0);
                const uint32_t l2 = *reinterpret_cast<const uint32_t*>(qsl + (r0 + g) * LD + i0 + 8);
                const uint32_t l3 = *reinterpret_cast<const uint32_t*>(qsl + (r0 + g + 8) * LD + i0 + 8);
#pragma unroll
                for (int nn = 0; nn < 2; ++nn) {
                    mma_bf16_regs(s[u][nn], l0, l1, l2, l3, b[nn][0], b[nn][1]);
                    mma_bf16_regs(s[u][nn], a0, a1, a2, a3, b[nn][0], b[nn][1]);
                }
            }
        }
        if (mt0 == 0) phase_stamp(p.trace, 4);  // CTA 0 (diagnostic): 4 S done, 5 max exchanged, 6 P staged, 7 PV done
        // mask + this quarter's row max
#pragma unroll
        for (int u = 0; u < MB; ++u) {
            if (u >= nm) break;
            const int ra = (mt0 + u) * 16 + g, rb = ra + 8;
            const int ta = ra % p.T, tb = rb % p.T;
            float ma = -INFINITY, mb = -INFINITY;
#pragma unroll
            for (int nn = 0; nn < 2; ++nn)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int j = (2 * warp + nn) * 8 + 2 * t4 + (q & 1);
                    const int tt = (q < 2) ? ta : tb;
                    const bool ok = j < nkeys && key0 + j <= ctx + tt;  // causal on absolute positions
                    if (!ok) s[u][nn][q] = -INFINITY;
                    if (q < 2) ma = fmaxf(ma, s[u][nn][q]);
                    else mb = fmaxf(mb, s[u][nn][q]);
                }
#pragma unroll
            for (int o = 1; o < 4; o <<= 1) {
                ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, o));
                mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, o));
            }
            if (t4 == 0) {
                red_m[u * 64 + warp * 16 + g] = ma;
                red_m[u * 64 + warp * 16 + g + 8] = mb;
            }
        }
        __syncthreads();
        if (mt0 == 0) phase_stamp(p.trace, 5);
        // exponentiate against the chunk max, P -> smem
#pragma unroll
        for (int u = 0; u < MB; ++u) {
            if (u >= nm) break;
            const float* rm = red_m + u * 64;
            const float ma = fmaxf(fmaxf(rm[g], rm[16 + g]), fmaxf(rm[32 + g], rm[48 + g]));
            const float mb = fmaxf(fmaxf(rm[8 + g], rm[24 + g]), fmaxf(rm[40 + g], rm[56 + g]));
            float* peu = pe + u * PT;
#pragma unroll
            for (int nn = 0; nn < 2; ++nn) {
                float e[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float m = (q < 2) ? ma : mb;
                    e[q] = (s[u][nn][q] == -INFINITY) ? 0.f : __expf(s[u][nn][q] - m);
                }
                const int col = (2 * warp + nn) * 8 + 2 * t4;
                *reinterpret_cast<float2*>(peu + g * kAttnPLd + col) = make_float2(e[0], e[1]);
                *reinterpret_cast<float2*>(peu + (g + 8) * kAttnPLd + col) = make_float2(e[2], e[3]);
            }
        }
        __syncthreads();
        if (mt0 == 0) phase_stamp(p.trace, 6);
        // O = P V for this warp's dims, all row tiles of the pass
        float o[MB][NDW][4];
#pragma unroll
        for (int u = 0; u < MB; ++u)
#pragma unroll
            for (int n = 0; n < NDW; ++n)
#pragma unroll
                for (int q = 0; q < 4; ++q) o[u][n][q] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            uint32_t bv[NDW / 2][4];
#pragma unroll
            for (int n2 = 0; n2 < NDW / 2; ++n2) {
                const int jrow = kk * 16 + (lane & 15);
                const int col = (warp * NDW + 2 * n2) * 8 + ((lane >> 4) << 3);
                const uint32_t addr = (uint32_t)__cvta_generic_to_shared(vs + jrow * LD + col);
                asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                             : "=r"(bv[n2][0]), "=r"(bv[n2][1]), "=r"(bv[n2][2]), "=r"(bv[n2][3])
                             : "r"(addr));
            }
            const int cA = kk * 16 + 2 * t4;
#pragma unroll
            for (int u = 0; u < MB; ++u) {
                if (u >= nm) break;
                const float* peu = pe + u * PT;
                const float2 e0 = *reinterpret_cast<const float2*>(peu + g * kAttnPLd + cA);
                const float2 e1 = *reinterpret_cast<const float2*>(peu + (g + 8) * kAttnPLd + cA);
                const float2 e2 = *reinterpret_cast<const float2*>(peu + g * kAttnPLd + cA + 8);
                const float2 e3 = *reinterpret_cast<const float2*>(peu + (g + 8) * kAttnPLd + cA + 8);
                uint32_t a0, a1, a2, a3, l0, l1, l2, l3;
                split_bf16x2(e0.x, e0.y, a0, l0);
                split_bf16x2(e1.x, e1.y, a1, l1);
                split_bf16x2(e2.x, e2.y, a2, l2);
                split_bf16x2(e3.x, e3.y, a3, l3);
#pragma unroll
                for (int n2 = 0; n2 < NDW / 2; ++n2) {
                    mma_bf16_regs(o[u][2 * n2], l0, l1, l2, l3, bv[n2][0], bv[n2][1]);
                    mma_bf16_regs(o[u][2 * n2], a0, a1, a2, a3, bv[n2][0], bv[n2][1]);
                    mma_bf16_regs(o[u][2 * n2 + 1], l0, l1, l2, l3, bv[n2][2], bv[n2][3]);
                    mma_bf16_regs(o[u][2 * n2 + 1], a0, a1, a2, a3, bv[n2][2], bv[n2][3]);
                }
            }
        }
        if (mt0 == 0) phase_stamp(p.trace, 7);
#pragma unroll
        for (int u = 0; u < MB; ++u) {
            if (u >= nm) break;
            const float* rm = red_m + u * 64;
            const int ra = (mt0 + u) * 16 + g, rb = ra + 8;
            float la = 0.f, lb = 0.f;
            if (warp == 0) {  // row sums in the one-warp tile's order: per lane over the 8 key tiles, then the quad
                const float* peu = pe + u * PT;
#pragma unroll
                for (int n = 0; n < 8; ++n) {
                    const float2 ea = *reinterpret_cast<const float2*>(peu + g * kAttnPLd + n * 8 + 2 * t4);
                    const float2 eb = *reinterpret_cast<const float2*>(peu + (g + 8) * kAttnPLd + n * 8 + 2 * t4);
                    la += ea.x;
                    la += ea.y;
                    lb += eb.x;
                    lb += eb.y;
                }
#pragma unroll
                for (int o = 1; o < 4; o <<= 1) {
                    la += __shfl_xor_sync(0xffffffffu, la, o);
                    lb += __shfl_xor_sync(0xffffffffu, lb, o);
                }
            }
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int r = half ? rb : ra;
                if (r >= R) continue;
                float* out = p.part + (((long long)kvh * R + r) * p.max_chunks + c) * (HD + 2);
#pragma unroll
                for (int n = 0; n < NDW; ++n) {
                    const int i = (warp * NDW + n) * 8 + 2 * t4;
                    *reinterpret_cast<float2*>(out + 2 + i) = make_float2(o[u][n][half * 2 + 0], o[u][n][half * 2 + 1]);
                }
                if (warp == 0 && t4 == 0) {
                    const int rr = g + 8 * half;
                    out[0] = fmaxf(fmaxf(rm[rr], rm[16 + rr]), fmaxf(rm[32 + rr], rm[48 + rr]));
                    out[1] = half ? lb : la;
                }
            }
        }
    }
}

// Transposed key-split pass (p.ksplit == 2): S^T = K Q^T and O^T = V^T P^T
// on mma.m16n8k16, so the query rows are the n8 dimension and a chunk item
// with R rows costs ceil(R/8) row tiles instead of 2*ceil(R/16) (Mixtral
// at K <= 1 and OLMoE / Qwen at K <= 7 have R <= 8: half the mma of the
// key split above).  Warp w owns keys [16w, 16w+16) for S^T and dims
// [hd/4 * w, hd/4 * (w+1)) for O^T; the row max is exchanged through
// shared memory, P is staged in fp32 (split into hi/lo bf16 as the B
// fragments load), and the row sums are formed in the one-warp tile's
// order.  kAttnTRows rows per pass.
constexpr int kAttnTRows = 32;
static_assert(kAttnTRows * kAttnPLd * 4 + kAttnTRows * 4 * 4 <= kAttnKsplitSmem, "transposed pass scratch");

template <int HD, int NB>
__device__ __forceinline__ void attn_tpass(const AttnParams& p, const uint16_t* qs, const uint16_t* qsl,
                                           const uint16_t* ks, const uint16_t* vs, uint16_t* scratch, int nr0,
                                           int R, int nkeys, int key0, int ctx, int kvh, int c) {
    constexpr int LD = HD + 8;
    constexpr int NKS = HD / 16;
    constexpr int MD = HD / 64;  // 16-dim m-tiles per warp in O^T
    float* pe = reinterpret_cast<float*>(scratch);  // [kAttnTRows][kAttnPLd] P (fp32), by query row
    float* red_m = pe + kAttnTRows * kAttnPLd;       // [kAttnTRows][4 warps]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const int kw = warp * 16;
    float s[NB][4];
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
        for (int q = 0; q < 4; ++q) s[nb][q] = 0.f;
#pragma unroll
    for (int kst = 0; kst < NKS; ++kst) {
        const int i0 = kst * 16 + 2 * t4;
        const uint32_t a0 = *reinterpret_cast<const uint32_t*>(ks + (kw + g) * LD + i0);
        const uint32_t a1 = *reinterpret_cast<const uint32_t*>(ks + (kw + g + 8) * LD + i0);
        const uint32_t a2 = *reinterpret_cast<const uint32_t*>(ks + (kw + g) * LD + i0 + 8);
        const uint32_t a3 = *reinterpret_cast<const uint32_t*>(ks + (kw + g + 8) * LD + i0 + 8);
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
            const int row = (nr0 + nb) * 8 + g;
            const uint32_t bh0 = *reinterpret_cast<const uint32_t*>(qs + row * LD + i0);
            const uint32_t bh1 = *reinterpret_cast<const uint32_t*>(qs + row * LD + i0 + 8);
            const uint32_t bl0 = *reinterpret_cast<const uint32_t*>(qsl + row * LD + i0);
            const uint32_t bl1 = *reinterpret_cast<const uint32_t*>(qsl + row * LD + i0 + 8);
            mma_bf16_regs(s[nb], a0, a1, a2, a3, bl0, bl1);
            mma_bf16_regs(s[nb], a0, a1, a2, a3, bh0, bh1);
        }
    }
    if (nr0 == 0) phase_stamp(p.trace, 4);
    // mask; this key quarter's max of each row (lanes of equal t4 share rows)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) {
        float m2[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = (nr0 + nb) * 8 + 2 * t4 + h;
            const int tt = r % p.T;
#pragma unroll
            for (int q = h; q < 4; q += 2) {
                const int j = kw + g + (q >= 2 ? 8 : 0);
                if (!(j < nkeys && key0 + j <= ctx + tt)) s[nb][q] = -INFINITY;
            }
            m2[h] = fmaxf(s[nb][h], s[nb][h + 2]);
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) m2[h] = fmaxf(m2[h], __shfl_xor_sync(0xffffffffu, m2[h], o));
        }
        if (g == 0) {
            red_m[(nb * 8 + 2 * t4) * 4 + warp] = m2[0];
            red_m[(nb * 8 + 2 * t4 + 1) * 4 + warp] = m2[1];
        }
    }
    __syncthreads();
    if (nr0 == 0) phase_stamp(p.trace, 5);
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int rl = nb * 8 + 2 * t4 + h;
            const float m = fmaxf(fmaxf(red_m[rl * 4], red_m[rl * 4 + 1]), fmaxf(red_m[rl * 4 + 2], red_m[rl * 4 + 3]));
#pragma unroll
            for (int q = h; q < 4; q += 2) {
                const float e = (s[nb][q] == -INFINITY) ? 0.f : __expf(s[nb][q] - m);
                pe[rl * kAttnPLd + kw + g + (q >= 2 ? 8 : 0)] = e;
            }
        }
    __syncthreads();
    if (nr0 == 0) phase_stamp(p.trace, 6);
    // O^T = V^T P^T for this warp's dims
    float o[MD][NB][4];
#pragma unroll
    for (int md = 0; md < MD; ++md)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
#pragma unroll
            for (int q = 0; q < 4; ++q) o[md][nb][q] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        uint32_t av[MD][4];
#pragma unroll
        for (int md = 0; md < MD; ++md) {
            const int d0 = (warp * MD + md) * 16;
            const int key = kk * 16 + (lane & 7) + ((lane >> 4) << 3);
            const int dim = d0 + (((lane >> 3) & 1) << 3);
            const uint32_t addr = (uint32_t)__cvta_generic_to_shared(vs + key * LD + dim);
            asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                         : "=r"(av[md][0]), "=r"(av[md][1]), "=r"(av[md][2]), "=r"(av[md][3])
                         : "r"(addr));
        }
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
            const float* pr = pe + (nb * 8 + g) * kAttnPLd + kk * 16 + 2 * t4;
            const float2 e0 = *reinterpret_cast<const float2*>(pr);
            const float2 e1 = *reinterpret_cast<const float2*>(pr + 8);
            uint32_t bh0, bl0, bh1, bl1;
            split_bf16x2(e0.x, e0.y, bh0, bl0);
            split_bf16x2(e1.x, e1.y, bh1, bl1);
#pragma unroll
            for (int md = 0; md < MD; ++md) {
                mma_bf16_regs(o[md][nb], av[md][0], av[md][1], av[md][2], av[md][3], bl0, bl1);
                mma_bf16_regs(o[md][nb], av[md][0], av[md][1], av[md][2], av[md][3], bh0, bh1);
            }
        }
    }
    if (nr0 == 0) phase_stamp(p.trace, 7);
    // row max / sum (sum in the one-warp tile's order: per lane over the 8
    // key tiles, then the quad)
    for (int rl = threadIdx.x >> 2; rl < NB * 8; rl += kAttnThreads / 4) {
        const float* pr = pe + rl * kAttnPLd + 2 * t4;
        float l = 0.f;
#pragma unroll
        for (int n = 0; n < 8; ++n) {
            const float2 e = *reinterpret_cast<const float2*>(pr + n * 8);
            l += e.x;
            l += e.y;
        }
        l += __shfl_xor_sync(0xffffffffu, l, 1);
        l += __shfl_xor_sync(0xffffffffu, l, 2);
        const int r = nr0 * 8 + rl;
        if (t4 == 0 && r < R) {
            float* out = p.part + (((long long)kvh * R + r) * p.max_chunks + c) * (HD + 2);
            out[0] = fmaxf(fmaxf(red_m[rl * 4], red_m[rl * 4 + 1]), fmaxf(red_m[rl * 4 + 2], red_m[rl * 4 + 3]));
            out[1] = l;
        }
    }
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = (nr0 + nb) * 8 + 2 * t4 + h;
            if (r >= R) continue;
            float* out = p.part + (((long long)kvh * R + r) * p.max_chunks + c) * (HD + 2) + 2;
#pragma unroll
            for (int md = 0; md < MD; ++md) {
                const int d0 = (warp * MD + md) * 16;
                out[d0 + g] = o[md][nb][h];
                out[d0 + g + 8] = o[md][nb][h + 2];
            }
        }
}

template <int HD>
__global__ void __launch_bounds__(kAttnThreads) attn_partial_kernel(AttnParams p) {
    constexpr int LD = HD + 8;
    constexpr int HALF = HD / 2;
    constexpr int NKS = HD / 16;      // k-steps of QK^T
    constexpr int NDT = HD / 8;       // n8 dim tiles of PV
    extern __shared__ __align__(16) uint16_t sm[];
    uint16_t* qs = sm;
    const int qrows = ((p.H / p.KV) * p.T + 15) / 16 * 16;  // staged query rows (smem sized per T)
    uint16_t* qsl = qs + qrows * LD;
    uint16_t* ks = qsl + qrows * LD;
    uint16_t* vs = ks + kChunk * LD;

    const int G = p.H / p.KV;
    const int R = G * p.T;
    // The committed cache (and its length, written by the previous step's
    // accept kernel) does not depend on the predecessor (the QKV GEMV): the
    // first item's K/V chunk is requested with cp.async before the wait.
    const int ctx = *p.ctx_ptr;
    auto issue_kv = [&](int item) {
        const int c = item / p.KV;
        const int kvh = item - c * p.KV;
        const int key0 = c * kChunk;
        const int nkeys = max(0, min(kChunk, ctx - key0));  // cached keys of the chunk (the rest are new)
        constexpr int V8 = HD / 8;  // 16-byte pieces per row
        const long long base = ((long long)kvh * p.max_ctx + key0) * HD;
        // slots >= nkeys belong to new keys (written by the item itself)
        for (int e = threadIdx.x; e < nkeys * V8; e += blockDim.x) {
            const int j = e / V8, q = e - j * V8;
            cp_async16(ks + j * LD + q * 8, p.kc + base + (long long)e * 8, 16);
            cp_async16(vs + j * LD + q * 8, p.vc + base + (long long)e * 8, 16);
        }
        cp_async_commit();
    };
    // Chunks are 64 absolute key positions: chunk c covers [64c, 64c+64) of
    // the cache + the T new keys, so a token's keys are grouped (and its
    // softmax summed) identically whatever the step width (batch-invariant).
    const int nch = (ctx + p.T + kChunk - 1) / kChunk;
    bool kv_pending = false;
    if ((int)blockIdx.x < nch * p.KV) {
        issue_kv(blockIdx.x);
        kv_pending = true;
    }
    griddep_wait();
    griddep_launch_early(kLateAttn);
    CTA_TRACE(p.trace);
    phase_stamp(p.trace, 0);  // CTA 0 (diagnostic): 1 queries staged, 2 K/V ready, 3 partials stored
    prefetch_l2(p.pf, p.pf_bytes);
    const int n_items = nch * p.KV;
    const int QD = (p.H + 2 * p.KV) * HD;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const int n_mt = (R + 15) / 16;

    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int c = item / p.KV;
        const int kvh = item - c * p.KV;
        const int key0 = c * kChunk;
        const int nkeys = min(kChunk, ctx + p.T - key0);      // keys of this chunk
        const int n_cached = max(0, min(kChunk, ctx - key0));  // the first n_cached come from the cache
        const bool has_new = n_cached < nkeys;

        __syncthreads();
        // queries (rotated at their own positions, scaled, two bf16 terms):
        // work item = (row, 4 consecutive dims i..i+3 and their rotate_half
        // partners i+HALF..), every global load of a batch of 4 items issued
        // before any math (this kernel is latency-bound).
        {
            constexpr int Q4 = HALF / 4;
            const int n_q = n_mt * 16 * Q4;
#ifndef CASCADE_ATTN_QB
#define CASCADE_ATTN_QB 4
#endif
            constexpr int kQB = CASCADE_ATTN_QB;  // query items per thread with loads in flight together
            for (int e0 = 0; e0 < n_q; e0 += kQB * kAttnThreads) {
                float4 qa[kQB], qb[kQB], ca[kQB], cb[kQB];
#pragma unroll
                for (int u = 0; u < kQB; ++u) {
                    const int e = e0 + u * kAttnThreads + threadIdx.x;
                    const int r = e / Q4, i = (e - r * Q4) * 4;
                    qa[u] = qb[u] = ca[u] = cb[u] = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (e < n_q && r < R) {
                        const int gi = r / p.T, t = r - gi * p.T;
                        const float* q = p.qkv + (long long)t * QD + (kvh * G + gi) * HD;
                        qa[u] = *reinterpret_cast<const float4*>(q + i);
                        qb[u] = *reinterpret_cast<const float4*>(q + i + HALF);
                        const float4* rp = reinterpret_cast<const float4*>(p.rope + t * HALF + i);
                        ca[u] = rp[0];  // (cos, sin) of dims i, i+1
                        cb[u] = rp[1];  // (cos, sin) of dims i+2, i+3
                    }
                }
#pragma unroll
                for (int u = 0; u < kQB; ++u) {
                    const int e = e0 + u * kAttnThreads + threadIdx.x;
                    if (e >= n_q) continue;
                    const int r = e / Q4, i = (e - r * Q4) * 4;
                    float a4[4] = {qa[u].x, qa[u].y, qa[u].z, qa[u].w};
                    float b4[4] = {qb[u].x, qb[u].y, qb[u].z, qb[u].w};
                    const float2 cs[4] = {make_float2(ca[u].x, ca[u].y), make_float2(ca[u].z, ca[u].w),
                                          make_float2(cb[u].x, cb[u].y), make_float2(cb[u].z, cb[u].w)};
                    uint32_t ah[2], al[2], bh[2], bl[2];
#pragma unroll
                    for (int k2 = 0; k2 < 4; ++k2) {
                        rope_pair(a4[k2], b4[k2], cs[k2]);
                        a4[k2] *= p.scale;
                        b4[k2] *= p.scale;
                    }
                    split_bf16x2(a4[0], a4[1], ah[0], al[0]);
                    split_bf16x2(a4[2], a4[3], ah[1], al[1]);
                    split_bf16x2(b4[0], b4[1], bh[0], bl[0]);
                    split_bf16x2(b4[2], b4[3], bh[1], bl[1]);
                    *reinterpret_cast<uint2*>(qs + r * LD + i) = make_uint2(ah[0], ah[1]);
                    *reinterpret_cast<uint2*>(qs + r * LD + i + HALF) = make_uint2(bh[0], bh[1]);
                    *reinterpret_cast<uint2*>(qsl + r * LD + i) = make_uint2(al[0], al[1]);
                    *reinterpret_cast<uint2*>(qsl + r * LD + i + HALF) = make_uint2(bl[0], bl[1]);
                }
            }
        }
        if (item == (int)blockIdx.x) phase_stamp(p.trace, 1);
        if (has_new) {
            // the new keys of this chunk (positions ctx .. ctx+T-1, rotated)
            // and their values -> bf16, appended to the cache and staged at
            // their chunk slots; slots past the chunk's keys are zero
            constexpr int Q4 = HALF / 4;
            for (int e = threadIdx.x; e < (kChunk - n_cached) * Q4; e += kAttnThreads) {
                const int jl = n_cached + e / Q4, i = (e - (e / Q4) * Q4) * 4;  // chunk slot
                const int j = key0 + jl - ctx;                                  // new-token index
                uint2 ka = make_uint2(0, 0), kb = ka, va = ka, vb = ka;
                if (jl < nkeys) {
                    const float* kr = p.qkv + (long long)j * QD + p.H * HD + kvh * HD;
                    const float* vr = p.qkv + (long long)j * QD + (p.H + p.KV) * HD + kvh * HD;
                    const float4 k0 = *reinterpret_cast<const float4*>(kr + i);
                    const float4 k1 = *reinterpret_cast<const float4*>(kr + i + HALF);
                    const float4 v0 = *reinterpret_cast<const float4*>(vr + i);
                    const float4 v1 = *reinterpret_cast<const float4*>(vr + i + HALF);
                    const float4* rp = reinterpret_cast<const float4*>(p.rope + j * HALF + i);
                    const float4 c0 = rp[0], c1 = rp[1];
                    float a4[4] = {k0.x, k0.y, k0.z, k0.w};
                    float b4[4] = {k1.x, k1.y, k1.z, k1.w};
                    rope_pair(a4[0], b4[0], make_float2(c0.x, c0.y));
                    rope_pair(a4[1], b4[1], make_float2(c0.z, c0.w));
                    rope_pair(a4[2], b4[2], make_float2(c1.x, c1.y));
                    rope_pair(a4[3], b4[3], make_float2(c1.z, c1.w));
                    ka = make_uint2(pack_bf16x2(a4[0], a4[1]), pack_bf16x2(a4[2], a4[3]));
                    kb = make_uint2(pack_bf16x2(b4[0], b4[1]), pack_bf16x2(b4[2], b4[3]));
                    va = make_uint2(pack_bf16x2(v0.x, v0.y), pack_bf16x2(v0.z, v0.w));
                    vb = make_uint2(pack_bf16x2(v1.x, v1.y), pack_bf16x2(v1.z, v1.w));
                    const long long base = ((long long)kvh * p.max_ctx + ctx + j) * HD;
                    *reinterpret_cast<uint2*>(p.kc + base + i) = ka;
                    *reinterpret_cast<uint2*>(p.kc + base + i + HALF) = kb;
                    *reinterpret_cast<uint2*>(p.vc + base + i) = va;
                    *reinterpret_cast<uint2*>(p.vc + base + i + HALF) = vb;
                }
                *reinterpret_cast<uint2*>(ks + jl * LD + i) = ka;
                *reinterpret_cast<uint2*>(ks + jl * LD + i + HALF) = kb;
                *reinterpret_cast<uint2*>(vs + jl * LD + i) = va;
                *reinterpret_cast<uint2*>(vs + jl * LD + i + HALF) = vb;
            }
        }
        if (n_cached > 0 && !kv_pending) {
            issue_kv(item);  // later items: the copy overlaps the query staging above
        }
        kv_pending = false;
        cp_async_wait_all();
        __syncthreads();
        if (item == (int)blockIdx.x) phase_stamp(p.trace, 2);

        bool done_ksplit = false;
        if constexpr (HD >= 64) {
            if (p.ksplit) {
                if (p.ksplit == 2) {
                    const int NR = (R + 7) / 8;
                    uint16_t* scr = vs + kChunk * LD;
                    for (int nr0 = 0; nr0 < NR; nr0 += kAttnTRows / 8) {
                        if (nr0 > 0) __syncthreads();  // the previous pass's readers of P / red_m are done
                        switch (min(kAttnTRows / 8, NR - nr0)) {
                            case 1: attn_tpass<HD, 1>(p, qs, qsl, ks, vs, scr, nr0, R, nkeys, key0, ctx, kvh, c); break;
                            case 2: attn_tpass<HD, 2>(p, qs, qsl, ks, vs, scr, nr0, R, nkeys, key0, ctx, kvh, c); break;
                            case 3: attn_tpass<HD, 3>(p, qs, qsl, ks, vs, scr, nr0, R, nkeys, key0, ctx, kvh, c); break;
                            default: attn_tpass<HD, 4>(p, qs, qsl, ks, vs, scr, nr0, R, nkeys, key0, ctx, kvh, c); break;
                        }
                    }
                } else
                for (int mt0 = 0; mt0 < n_mt; mt0 += kAttnKsMt) {
                    if (mt0 > 0) __syncthreads();  // the previous pass's readers of P / red_m are done
                    uint16_t* scr = vs + kChunk * LD;
                    switch (min(kAttnKsMt, n_mt - mt0)) {
                        case 1: attn_ksplit_pass<HD, 1>(p, qs, qsl, ks, vs, scr, mt0, R, nkeys, key0, ctx, kvh, c); break;
                        case 2: attn_ksplit_pass<HD, 2>(p, qs, qsl, ks, vs, scr, mt0, R, nkeys, key0, ctx, kvh, c); break;
                        default: attn_ksplit_pass<HD, 3>(p, qs, qsl, ks, vs, scr, mt0, R, nkeys, key0, ctx, kvh, c); break;

                    }
                }
                done_ksplit = true;
            }
        }
        for (int mt = warp; mt < (done_ksplit ? 0 : n_mt); mt += kAttnThreads / 32) {
            const int r0 = mt * 16;
            // S = Q K^T  (16 rows x 64 keys)
            float s[8][4];
#pragma unroll
            for (int n = 0; n < 8; ++n)
#pragma unroll
                for (int q = 0; q < 4; ++q) s[n][q] = 0.f;
#pragma unroll
            for (int kst = 0; kst < NKS; ++kst) {
                const int i0 = kst * 16 + 2 * t4;
                const uint32_t a0 = *reinterpret_cast<const uint32_t*>(qs + (r0 + g) * LD + i0);
                const uint32_t a1 = *reinterpret_cast<const uint32_t*>(qs + (r0 + g + 8) * LD + i0);
                const uint32_t a2 = *reinterpret_cast<const uint32_t*>(qs + (r0 + g) * LD + i0 + 8);
                const uint32_t a3 = *reinterpret_cast<const uint32_t*>(qs + (r0 + g + 8) * LD + i0 + 8);
                const uint32_t l0 = *reinterpret_cast<const uint32_t*>(qsl + (r0 + g) * LD + i0);
                const uint32_t l1 = *reinterpret_cast<const uint32_t*>(qsl + (r0 + g + 8) * LD + i0);
                const uint32_t l2 = *reinterpret_cast<const uint32_t*>(qsl + (r0 + g) * LD + i0 + 8);
                const uint32_t l3 = *reinterpret_cast<const uint32_t*>(qsl + (r0 + g + 8) * LD + i0 + 8);
#pragma unroll
                for (int n = 0; n < 8; ++n) {
                    const uint32_t b0 = *reinterpret_cast<const uint32_t*>(ks + (n * 8 + g) * LD + i0);
                    const uint32_t b1 = *reinterpret_cast<const uint32_t*>(ks + (n * 8 + g) * LD + i0 + 8);
                    mma_bf16_regs(s[n], l0, l1, l2, l3, b0, b1);
                    mma_bf16_regs(s[n], a0, a1, a2, a3, b0, b1);
                }
            }
            // mask + row softmax statistics (rows r0+g and r0+g+8)
            const int ra = r0 + g, rb = r0 + g + 8;
            const int ta = ra % p.T, tb = rb % p.T;
            float ma = -INFINITY, mb = -INFINITY;
#pragma unroll
            for (int n = 0; n < 8; ++n)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int j = n * 8 + 2 * t4 + (q & 1);
                    const int tt = (q < 2) ? ta : tb;
                    const bool ok = j < nkeys && key0 + j <= ctx + tt;  // causal on absolute positions
                    if (!ok) s[n][q] = -INFINITY;
                    if (q < 2) ma = fmaxf(ma, s[n][q]);
                    else mb = fmaxf(mb, s[n][q]);
                }
#pragma unroll
            for (int o = 1; o < 4; o <<= 1) {
                ma = fmaxf(ma, __shfl_xor_sync(0xffffffffu, ma, o));
                mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, o));
            }
            float la = 0.f, lb = 0.f;
#pragma unroll
            for (int n = 0; n < 8; ++n)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float m = (q < 2) ? ma : mb;
                    const float e = (s[n][q] == -INFINITY) ? 0.f : __expf(s[n][q] - m);
                    s[n][q] = e;
                    if (q < 2) la += e;
                    else lb += e;
                }
#pragma unroll
            for (int o = 1; o < 4; o <<= 1) {
                la += __shfl_xor_sync(0xffffffffu, la, o);
                lb += __shfl_xor_sync(0xffffffffu, lb, o);
            }
            // O = P V  (16 rows x HD)
            float o[NDT][4];
#pragma unroll
            for (int n = 0; n < NDT; ++n)
#pragma unroll
                for (int q = 0; q < 4; ++q) o[n][q] = 0.f;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                uint32_t a0, a1, a2, a3, l0, l1, l2, l3;
                split_bf16x2(s[2 * kk][0], s[2 * kk][1], a0, l0);
                split_bf16x2(s[2 * kk][2], s[2 * kk][3], a1, l1);
                split_bf16x2(s[2 * kk + 1][0], s[2 * kk + 1][1], a2, l2);
                split_bf16x2(s[2 * kk + 1][2], s[2 * kk + 1][3], a3, l3);
#pragma unroll
                for (int n = 0; n < NDT; n += 2) {
                    // ldmatrix.x4.trans: lanes 0-15 -> rows of dims n*8, lanes 16-31 -> dims n*8+8
                    const int jrow = kk * 16 + (lane & 15);
                    const int col = n * 8 + ((lane >> 4) << 3);
                    const uint32_t addr =
                        (uint32_t)__cvta_generic_to_shared(vs + jrow * LD + col);
                    uint32_t b0, b1, b2, b3;
                    asm volatile(
                        "ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                        : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                        : "r"(addr));
                    mma_bf16_regs(o[n], l0, l1, l2, l3, b0, b1);
                    mma_bf16_regs(o[n], a0, a1, a2, a3, b0, b1);
                    mma_bf16_regs(o[n + 1], l0, l1, l2, l3, b2, b3);
                    mma_bf16_regs(o[n + 1], a0, a1, a2, a3, b2, b3);
                }
            }
            // partials
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int r = half ? rb : ra;
                if (r >= R) continue;
                float* out = p.part + (((long long)kvh * R + r) * p.max_chunks + c) * (HD + 2);
#pragma unroll
                for (int n = 0; n < NDT; ++n) {
                    const int i = n * 8 + 2 * t4;
                    out[2 + i] = o[n][half * 2 + 0];
                    out[2 + i + 1] = o[n][half * 2 + 1];
                }
                if (t4 == 0) {
                    out[0] = half ? mb : ma;
                    out[1] = half ? lb : la;
                }
            }
        }
        if (item == (int)blockIdx.x) phase_stamp(p.trace, 3);
        if (p.fused) {
            // arrival of this item; the last of the KV head's nch items
            // merges the head's chunk partials (fixed chunk order)
            __shared__ int s_last;
            __threadfence();
            __syncthreads();
            if (threadIdx.x == 0) s_last = atomicAdd(p.arrive + kvh, 1) == nch - 1;
            __syncthreads();
            if (s_last) {
                __threadfence();
                const int nck = nch;
                float* scale = reinterpret_cast<float*>(sm);  // [R][nck] exp(m_c - M_r), then L_r at [R*nck + r]
                float* Lr = scale + R * nck;  // [R]
                float* lv = Lr + R;           // [R][nck] chunk sums l_c
                const float* base = p.part + (long long)kvh * R * p.max_chunks * (HD + 2);
                for (int r = warp; r < R; r += kAttnThreads / 32) {
                    const float* pr = base + (long long)r * p.max_chunks * (HD + 2);
                    float m = -INFINITY;
                    for (int c2 = lane; c2 < nck; c2 += 32) m = fmaxf(m, __ldcg(pr + (long long)c2 * (HD + 2)));
                    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
                    for (int c2 = lane; c2 < nck; c2 += 32) {
                        scale[r * nck + c2] = __expf(__ldcg(pr + (long long)c2 * (HD + 2)) - m);
                        lv[r * nck + c2] = __ldcg(pr + (long long)c2 * (HD + 2) + 1);
                    }
                    __syncwarp();
                    if (lane == 0) {  // sequential in chunk order (same expression as attn_combine_kernel)
                        float l = 0.f;
                        for (int c2 = 0; c2 < nck; ++c2) l = fmaf(lv[r * nck + c2], scale[r * nck + c2], l);
                        Lr[r] = l;
                    }
                }
                __syncthreads();
                // (row, 4 dims) per thread-item, the chunk loads of a batch of
                // 9 chunks in flight together
                constexpr int H4 = HD / 4;
#ifndef CASCADE_ATTN_MB
#define CASCADE_ATTN_MB 9
#endif
                constexpr int kMB = CASCADE_ATTN_MB;  // chunk partials in flight per (row, 4 dims)
                for (int idx = threadIdx.x; idx < R * H4; idx += kAttnThreads) {
                    const int r = idx / H4, i = (idx - r * H4) * 4;
                    const float* pr = base + (long long)r * p.max_chunks * (HD + 2) + 2 + i;
                    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
                    for (int c0 = 0; c0 < nck; c0 += kMB) {
                        float4 v9[kMB];
#pragma unroll
                        for (int u = 0; u < kMB; ++u)
                            if (c0 + u < nck) {
                                const float* q = pr + (long long)(c0 + u) * (HD + 2);  // 8-byte aligned: two float2
                                const float2 lo = __ldcg(reinterpret_cast<const float2*>(q));
                                const float2 hi = __ldcg(reinterpret_cast<const float2*>(q + 2));
                                v9[u] = make_float4(lo.x, lo.y, hi.x, hi.y);
                            }
#pragma unroll
                        for (int u = 0; u < kMB; ++u)
                            if (c0 + u < nck) {
                                const float sc = scale[r * nck + c0 + u];
                                acc.x = fmaf(v9[u].x, sc, acc.x);
                                acc.y = fmaf(v9[u].y, sc, acc.y);
                                acc.z = fmaf(v9[u].z, sc, acc.z);
                                acc.w = fmaf(v9[u].w, sc, acc.w);
                            }
                    }
                    const float L = Lr[r];
                    const int gi = r / p.T, t = r - gi * p.T;
                    const int k = (kvh * G + gi) * HD + i;
                    const uint32_t w0 = pack_bf16x2(acc.x / L, acc.y / L), w1 = pack_bf16x2(acc.z / L, acc.w / L);
                    if (p.umma) {
                        *reinterpret_cast<uint2*>(p.out_bfrag + umma_b_index(t, k)) = make_uint2(w0, w1);
                    } else {
                        *reinterpret_cast<uint32_t*>(p.out_bfrag + bfrag_index(t, k)) = w0;
                        *reinterpret_cast<uint32_t*>(p.out_bfrag + bfrag_index(t, k + 2)) = w1;
                    }
                }
                if (threadIdx.x == 0) p.arrive[kvh] = 0;
            }
        }
    }
}

// Merge chunk partials in fixed order; write bf16 O-proj input (B-frag).
// One CTA per (token, head); the per-chunk (max, sum) pairs are staged in
// shared memory so every o-load of the merge is independent.
struct AttnCombineParams {
    const float* part;
    const int* ctx_ptr;
    uint16_t* out_bfrag;   // [H*hd] B-frag
    float* tap;            // optional fp32 [T][H*hd]
    int T, H, KV, hd, max_chunks;
    unsigned long long* trace;
    int umma;              // out_bfrag in the UMMA B layout (O projection on tcgen05)
};

constexpr int kMaxChunksSmem = 1024;

__global__ void attn_combine_kernel(AttnCombineParams p) {
    griddep_wait();
    griddep_launch_early(kLateAttnCombine);
    CTA_TRACE(p.trace);
    __shared__ float scale_c[kMaxChunksSmem];
    __shared__ float red[32];
    const int t = blockIdx.x, h = blockIdx.y;
    const int G = p.H / p.KV;
    const int kvh = h / G, gi = h - kvh * G;
    const int R = G * p.T;
    const int r = gi * p.T + t;
    const int ctx = *p.ctx_ptr;
    const int nch = (ctx + p.T + kChunk - 1) / kChunk;  // 64-key chunks of absolute positions (attn_partial_kernel)
    const int stride = p.hd + 2;
    const float* base = p.part + ((long long)kvh * R + r) * p.max_chunks * stride;
    // every load of the first kCB chunks is issued up front: (max, sum) of
    // chunk c by thread c, the o-vectors of dim i by thread i
    constexpr int kCB = 32;
    const int i = threadIdx.x;  // blockDim.x == hd
    float mc = -INFINITY, lc = 0.f;
    if ((int)threadIdx.x < nch) {
        mc = base[(long long)threadIdx.x * stride];
        lc = base[(long long)threadIdx.x * stride + 1];
    }
    float ov[kCB];
#pragma unroll
    for (int c = 0; c < kCB; ++c) ov[c] = c < nch ? base[(long long)c * stride + 2 + i] : 0.f;
    float m = mc;
    for (int c = threadIdx.x + blockDim.x; c < nch; c += blockDim.x) m = fmaxf(m, base[(long long)c * stride]);
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    float M = -INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) M = fmaxf(M, red[w]);
    __syncthreads();
    // scale_c = exp(m_c - M); L = sum_c l_c * scale_c summed sequentially in
    // chunk order (the fused combine in attn_partial_kernel computes the
    // identical expression, so the result does not depend on the path)
    __shared__ float s_L;
    __shared__ float l_c[kMaxChunksSmem];
    for (int c = threadIdx.x; c < nch; c += blockDim.x) {
        scale_c[c] = __expf(base[(long long)c * stride] - M);
        l_c[c] = base[(long long)c * stride + 1];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float L0 = 0.f;
        for (int c = 0; c < nch; ++c) L0 = fmaf(l_c[c], scale_c[c], L0);
        s_L = L0;
    }
    (void)mc;
    (void)lc;
    __syncthreads();
    const float L = s_L;
    float o = 0.f;
#pragma unroll
    for (int c = 0; c < kCB; ++c)
        if (c < nch) o = fmaf(ov[c], scale_c[c], o);
    for (int c0 = kCB; c0 < nch; c0 += kCB) {
#pragma unroll
        for (int c = 0; c < kCB; ++c) ov[c] = c0 + c < nch ? base[(long long)(c0 + c) * stride + 2 + i] : 0.f;
#pragma unroll
        for (int c = 0; c < kCB; ++c)
            if (c0 + c < nch) o = fmaf(ov[c], scale_c[c0 + c], o);
    }
    const float v = o / L;
    const int k = h * p.hd + i;
    p.out_bfrag[p.umma ? umma_b_index(t, k) : bfrag_index(t, k)] = bf16_bits(v);
    if (p.tap) p.tap[(long long)t * p.H * p.hd + k] = v;
}

}  // namespace cascade
