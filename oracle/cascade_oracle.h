/* cascade_oracle.h — CPU oracle for the MoE verification step.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker for the CUDA path
 * in paper_2506_20675_b200/csrc; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path never calls it (no CPU fallback exists).
 *
 * What it restates.  The reference (/root/reference/proj, `specsim`) prices
 * the verification step instead of computing it, so its numerics have no
 * reference implementation ("parity unpinned" for logits).
 * The reference pins the *semantics* this oracle follows:
 *   - per token, top_k DISTINCT routed experts           expert_model.hpp:100-112
 *   - union = distinct routed experts, shared blocks
 *     counted once on top (popcount + shared)           expert_model.hpp:126-138
 *   - acceptance = causal prefix, 0 <= accepted <= K,
 *     emitted = accepted + 1                            workload.hpp:80-86
 *   - a smaller offered K truncates the prefix          trace.hpp:69-74
 *   - ties resolve to the lower index                   controller.hpp:124-125
 * and the numerics follow the public model definitions (RMSNorm, GQA
 * attention with RoPE, softmax top-k router, SwiGLU experts) in fp64 with
 * bf16 rounding exactly where the device rounds (norm outputs, KV cache,
 * attention output, SiLU(gate)*up).  Weights come from the same counter
 * hash as the device (include/cascade_weights.h), generated lazily.
 */
#ifndef CASCADE_ORACLE_H_
#define CASCADE_ORACLE_H_

#include <stdint.h>

#include "cascade.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_model orc_model;
typedef struct orc_session orc_session;

orc_model* orc_model_create(const cascade_geometry* g, uint64_t seed, int nthreads);
void orc_model_destroy(orc_model* m);
void orc_model_drop_cache(orc_model* m);
/* bytes of generated weights currently cached */
uint64_t orc_cached_bytes(const orc_model* m);

/* Copies logical rows [row0, row0+nrows) of a tensor (bf16 bits). */
int orc_tensor(orc_model* m, int kind, int layer, int expert, int row0, int nrows, uint16_t* out);
/* Pre-generates (and caches) every tensor of one layer touched by experts
 * `experts[0..n)` (routed ids, shared blocks are E..E+S-1). */
int orc_prepare_layer(orc_model* m, int layer, const int32_t* experts, int n);

/* ---- stages (teacher-forcing API; x = fp32 residual rows [T][d]) ---- */
int orc_rmsnorm(orc_model* m, int kind, int layer, const float* x, int T, uint16_t* out);
int orc_router(orc_model* m, int layer, const uint16_t* xn, int T, double* logits, int32_t* topk,
               double* topw, double* gsh, double* margin);
/* union of the top-k lists: ascending unique routed experts; returns U */
int orc_union(const int32_t* topk, int T, int k, int32_t* uniq);
int orc_moe(orc_model* m, int layer, const uint16_t* xn, int T, const int32_t* topk,
            const double* topw, const double* gsh, double* out);
/* attention block: residual x entering the layer -> O-proj output (what is
 * added to the residual); kcache/vcache [KV][ctx][hd] bf16; the T new rows
 * (rotated, bf16) are written to k_new/v_new [KV][T][hd] when non-NULL. */
int orc_attention(orc_model* m, int layer, const float* x, int T, int ctx, const uint16_t* kcache,
                  const uint16_t* vcache, double* out, uint16_t* k_new, uint16_t* v_new);
int orc_lm_head(orc_model* m, const uint16_t* xn, int T, double* logits, int32_t* argmax,
                double* margin);
/* greedy acceptance: leading drafts equal to argmax; writes emitted tokens
 * (accepted drafts + bonus) and returns `accepted` */
int orc_greedy_accept(const int32_t* argmax, const int32_t* drafts, int K, int32_t* emitted);

/* ---- end-to-end (independent of the device) ---- */
orc_session* orc_session_create(orc_model* m, int max_ctx);
void orc_session_destroy(orc_session* s);
int orc_prefill(orc_session* s, const int32_t* prompt, int n);
/* verify the pending token + K drafts; logits [T][V] (optional), argmax [T],
 * margin [T] (top-1 minus top-2 logit) optional; returns accepted (>= 0) */
int orc_verify(orc_session* s, const int32_t* drafts, int K, double* logits, int32_t* argmax,
               double* margin, int32_t* union_sizes);
int orc_cache_len(const orc_session* s);
/* smallest router top-k decision margin (logit units) seen since the last
 * reset: a device/oracle routing disagreement below it is a flagged tie */
double orc_min_router_margin(orc_session* s, int reset);
/* routing of the last forward pass: topk [L][T][k], margins [L][T]; returns T */
int orc_last_routing(const orc_session* s, int32_t* topk, double* margin);

#ifdef __cplusplus
}
#endif

#endif
