// combine_ops.cuh — the residual combine + RMSNorm arithmetic shared by
// moe_combine_kernel (moe.cuh) and the QKV GEMV that folds the combine of a
// one-token step into its prologue (gemv_umma.cuh dense_gemv_cluster_kernel):
// one fixed operation order with explicit fma / round-to-nearest adds, so
// contraction choices cannot differ between the two kernels and their
// results are bitwise equal (batch-invariant mode relies on it).
#pragma once

#include "common.cuh"

namespace cascade {

#ifndef CASCADE_ROW_THREADS
#define CASCADE_ROW_THREADS 512
#endif
constexpr int kRowThreads = CASCADE_ROW_THREADS;  // route / combine: one CTA per token row
constexpr int kRowG = 8192 / (8 * kRowThreads);   // 8-column groups per thread (d <= 8192)
static_assert(kRowThreads == 512, "block_sum512_emulated mirrors a 512-thread combine");

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    return (uint32_t)bf16_bits(lo) | ((uint32_t)bf16_bits(hi) << 16);
}
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ void moe_acc_add(float4& acc, float w, const float4& y) {
    acc.x = fmaf(w, y.x, acc.x);
    acc.y = fmaf(w, y.y, acc.y);
    acc.z = fmaf(w, y.z, acc.z);
    acc.w = fmaf(w, y.w, acc.w);
}
__device__ __forceinline__ void moe_sh_add(float4& sh, const float4& y) {
    sh.x = __fadd_rn(sh.x, y.x);
    sh.y = __fadd_rn(sh.y, y.y);
    sh.z = __fadd_rn(sh.z, y.z);
    sh.w = __fadd_rn(sh.w, y.w);
}
// residual + contribution (the shared experts' sum gated by g); moe = the contribution
__device__ __forceinline__ float4 moe_finish(const float4& x0, float4 acc, const float4& sh, float g, bool shared, float4& moe) {
    if (shared) {
        acc.x = fmaf(g, sh.x, acc.x);
        acc.y = fmaf(g, sh.y, acc.y);
        acc.z = fmaf(g, sh.z, acc.z);
        acc.w = fmaf(g, sh.w, acc.w);
    }
    moe = acc;
    return make_float4(__fadd_rn(x0.x, acc.x), __fadd_rn(x0.y, acc.y), __fadd_rn(x0.z, acc.z), __fadd_rn(x0.w, acc.w));
}
__device__ __forceinline__ float ss_add(float ss, const float4& v) {
    float t = __fmul_rn(v.x, v.x);
    t = fmaf(v.y, v.y, t);
    t = fmaf(v.z, v.z, t);
    t = fmaf(v.w, v.w, t);
    return __fadd_rn(ss, t);
}
// 8 normalised columns (a: 0-3, b: 4-7) as packed bf16
__device__ __forceinline__ uint4 xn_pack8(const float4& a, const float4& b, float rinv, const uint4& nw) {
    return make_uint4(pack_bf16(__fmul_rn(__fmul_rn(a.x, rinv), bf16_lo(nw.x)), __fmul_rn(__fmul_rn(a.y, rinv), bf16_hi(nw.x))),
                      pack_bf16(__fmul_rn(__fmul_rn(a.z, rinv), bf16_lo(nw.y)), __fmul_rn(__fmul_rn(a.w, rinv), bf16_hi(nw.y))),
                      pack_bf16(__fmul_rn(__fmul_rn(b.x, rinv), bf16_lo(nw.z)), __fmul_rn(__fmul_rn(b.y, rinv), bf16_hi(nw.z))),
                      pack_bf16(__fmul_rn(__fmul_rn(b.z, rinv), bf16_lo(nw.w)), __fmul_rn(__fmul_rn(b.w, rinv), bf16_hi(nw.w))));
}

// block_sum (common.cuh) over the 512 threads of moe_combine_kernel, given
// their per-thread partials in shared memory, computed by one warp in the
// same butterfly order (every lane ends with the same value)
__device__ __forceinline__ float block_sum512_emulated(const float* part, float* red16) {
    const int lane = threadIdx.x & 31;
    for (int w = 0; w < 16; ++w) {
        float v = part[32 * w + lane];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red16[w] = v;
    }
    __syncwarp();
    float s = lane < 16 ? red16[lane] : 0.f;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

}  // namespace cascade
