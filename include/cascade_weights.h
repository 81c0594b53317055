/* cascade_weights.h — the counter-hash weight generator shared by the CUDA
 * library and the CPU oracle.
 *
 * Random-init weights for the BASELINE configs (Mixtral-8x7B is 93 GB of
 * bf16) are never moved between host and device: every element is a pure
 * function of (seed, tensor id, logical row, logical col), evaluated with
 * integer arithmetic plus at most two IEEE-rounded fp32 operations, so the
 * GPU initialiser and the oracle produce bit-identical bf16 values.  The
 * mixing function is the splitmix64 finaliser the reference already uses
 * for seeding (proj/include/specsim/engine.hpp:74-79).
 *
 * Value of element (r, c) of a [rows, cols] tensor:
 *     h = mix(mix(seed ^ mix(tid)) + r*cols + c)
 *     u = ((h >> 40) - 2^23) * 2^-23            in [-1, 1), exact in fp32
 *     linear / router / embedding:  w = bf16(u * scale)
 *     norm weights:                 w = bf16(1 + 0.1*u)
 * with scale = sqrt(3 / fan_in) (std 1/sqrt(fan_in)), times router_scale
 * for router rows, and sqrt(3) for the embedding (std 1).
 *
 * C and CUDA; no dependencies.  Compile users with -ffp-contract=off.
 */
#ifndef CASCADE_WEIGHTS_H_
#define CASCADE_WEIGHTS_H_

#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define CASCADE_HD __host__ __device__ __forceinline__
#else
#define CASCADE_HD static inline
#endif

/* tensor kinds */
enum {
    CASCADE_T_EMBED = 1,       /* [V, d]                        */
    CASCADE_T_ATTN_NORM = 2,   /* [d] per layer                 */
    CASCADE_T_FFN_NORM = 3,    /* [d] per layer                 */
    CASCADE_T_WQ = 4,          /* [H*hd, d]                     */
    CASCADE_T_WK = 5,          /* [KV*hd, d]                    */
    CASCADE_T_WV = 6,          /* [KV*hd, d]                    */
    CASCADE_T_WO = 7,          /* [d, H*hd]                     */
    CASCADE_T_ROUTER = 8,      /* [E, d]                        */
    CASCADE_T_SHARED_GATE = 9, /* [1, d]  (Qwen sigmoid gate)   */
    CASCADE_T_W_GATE = 10,     /* [f, d] per expert block       */
    CASCADE_T_W_UP = 11,       /* [f, d] per expert block       */
    CASCADE_T_W_DOWN = 12,     /* [d, f] per expert block       */
    CASCADE_T_FINAL_NORM = 13, /* [d]                           */
    CASCADE_T_LM_HEAD = 14     /* [V, d]                        */
};

CASCADE_HD uint64_t cascade_mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

CASCADE_HD uint64_t cascade_tensor_id(int kind, int layer, int expert) {
    return ((uint64_t)(uint32_t)kind << 48) | ((uint64_t)(uint32_t)layer << 24) |
           (uint64_t)(uint32_t)expert;
}

/* per-tensor key: hoisted out of the element loop */
CASCADE_HD uint64_t cascade_tensor_key(uint64_t seed, uint64_t tid) {
    return cascade_mix64(seed ^ cascade_mix64(tid));
}

/* u in [-1, 1), exactly representable in fp32 */
CASCADE_HD float cascade_unit(uint64_t key, uint64_t index) {
    const uint64_t h = cascade_mix64(key + index);
    const int32_t q = (int32_t)(h >> 40) - 0x800000;
    return (float)q * (1.0f / 8388608.0f);
}

/* round-to-nearest-even fp32 -> bf16 bits (values are finite here) */
CASCADE_HD uint16_t cascade_f32_to_bf16(float f) {
    union { float f; uint32_t u; } v;
    v.f = f;
    uint32_t u = v.u;
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

CASCADE_HD float cascade_bf16_to_f32(uint16_t b) {
    union { float f; uint32_t u; } v;
    v.u = ((uint32_t)b) << 16;
    return v.f;
}

/* bf16 bits of one weight element.  `scale` < 0 selects the norm rule. */
CASCADE_HD uint16_t cascade_weight_bits(uint64_t key, uint64_t index, float scale) {
    const float u = cascade_unit(key, index);
#if defined(__CUDA_ARCH__)
    const float w = scale < 0.0f ? __fadd_rn(1.0f, __fmul_rn(0.1f, u)) : __fmul_rn(u, scale);
#else
    volatile float t = scale < 0.0f ? 0.1f * u : u * scale; /* one rounding, no contraction */
    const float w = scale < 0.0f ? 1.0f + t : t;
#endif
    return cascade_f32_to_bf16(w);
}

/* Init scale of a tensor kind (host side; the device receives the float).
 * Returns a negative value for norm weights. */
static inline float cascade_kind_scale(int kind, int fan_in, float router_scale) {
    switch (kind) {
    case CASCADE_T_ATTN_NORM:
    case CASCADE_T_FFN_NORM:
    case CASCADE_T_FINAL_NORM:
        return -1.0f;
    case CASCADE_T_EMBED:
        return 1.7320508075688772f; /* sqrt(3): std 1 */
    case CASCADE_T_ROUTER:
    case CASCADE_T_SHARED_GATE: {
        volatile float s = sqrtf(3.0f / (float)fan_in);
        return s * router_scale;
    }
    default:
        return sqrtf(3.0f / (float)fan_in);
    }
}

#endif /* CASCADE_WEIGHTS_H_ */
