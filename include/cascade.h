/* cascade.h — C ABI of the B200-native MoE verification step.
 *
 * This is the drop-in boundary for the hot path named in BASELINE.json
 * (`north_star`): the target-model verification step over K+1 speculative
 * tokens.  In the reference (`/root/reference/proj`, the header-only C++
 * `specsim` library) that step is *priced*, not computed, by two calls in the
 * per-iteration loop of `run_request`:
 *
 *   iteration_cost(iter_cfg, draft, k, rng) -> CostBreakdown
 *       proj/include/specsim/engine.hpp:158   (replay: engine.hpp:227)
 *       defined at proj/include/specsim/expert_model.hpp:145-172
 *   pstate.sample_accepted(k, rng) -> int
 *       proj/include/specsim/engine.hpp:159   (replay: engine.hpp:228)
 *       defined at proj/include/specsim/workload.hpp:80-86, 102-104
 *
 * `cascade_verify` replaces both with one real step on the GPU: it runs the
 * K+1 tokens through every layer (router -> expert union -> grouped expert
 * FFN, attention + KV append), then the LM head, greedy acceptance and the
 * on-device utility, and returns the same quantities the reference returned
 * (a CostBreakdown and an accepted count) plus the emitted tokens.
 *
 * Conventions
 *  - Plain C: opaque handles, caller-owned buffers, int status codes.
 *  - Status codes mirror the reference's exception classes so the C++
 *    wrapper (include/specsim/verifier.hpp) can rethrow the same types:
 *      CASCADE_EINVAL    <-> std::invalid_argument  (expert_model.hpp:38-49, 85-88, 147)
 *      CASCADE_ERUNTIME  <-> std::runtime_error     (trace.hpp:78)
 *      CASCADE_ECUDA     <-> std::runtime_error     (device failure; no reference analogue)
 *      CASCADE_ENOBASE   <-> MissingBaselineError   (utility.hpp:52-55)
 *  - One session per request, one host thread per session.
 *  - `stream` arguments are `cudaStream_t` passed as `void*` (NULL = the
 *    session creates its own non-blocking stream).
 *  - No torch types, no C++ types in any signature.
 */
#ifndef CASCADE_H_
#define CASCADE_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CASCADE_API __attribute__((visibility("default")))
#else
#define CASCADE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define CASCADE_OK 0
#define CASCADE_EINVAL 1
#define CASCADE_ERUNTIME 2
#define CASCADE_ECUDA 3
#define CASCADE_ENOBASE 4

/* Maximum in-flight tokens per verification step (K+1).  The BASELINE
 * configs need K <= 8; the mma n-tiles cover 16 tokens for free. */
#define CASCADE_MAX_TOKENS 16
#define CASCADE_MAX_K (CASCADE_MAX_TOKENS - 1)
#define CASCADE_MAX_LAYERS 128

/* Model geometry.  The first block is the reference's routing geometry,
 * `ExpertConfig` (expert_model.hpp:27-51); the second block is the tensor
 * shape the reference never needed because it only priced the step.  A
 * fixture JSON carrying the extra keys still loads in the reference, whose
 * parsers ignore unknown keys (scenario.hpp:119-133). */
typedef struct cascade_geometry {
    /* --- ExpertConfig (expert_model.hpp:27-35) --- */
    int32_t num_layers;         /* L */
    int32_t experts_per_layer;  /* routed pool E (<= 128, expert_model.hpp:96) */
    int32_t top_k;              /* routed experts per token */
    int32_t shared_experts;     /* always-active expert blocks of width d_ff */
    /* --- tensor shape (public model configs; not in the reference) --- */
    int32_t d_model;            /* hidden size d (multiple of 256) */
    int32_t d_ff;               /* routed expert intermediate f (multiple of 32) */
    int32_t n_heads;            /* query heads H */
    int32_t n_kv_heads;         /* key/value heads (GQA) */
    int32_t head_dim;           /* per-head dim (even, <= 256) */
    int32_t vocab;              /* V (multiple of 64) */
    int32_t renormalize_topk;   /* 1: Mixtral (softmax over the chosen k); 0: OLMoE/Qwen */
    int32_t shared_gate;        /* 1: sigmoid gate on the shared blocks (Qwen1.5-MoE) */
    float rope_theta;
    float norm_eps;
    float router_scale;         /* multiplier on the router init scale (spreads logits) */
    int32_t reserved[5];
} cascade_geometry;

/* Result of one verification step.  `accepted`/`emitted` replace
 * sample_accepted (workload.hpp:80-86: 0 <= accepted <= K, emitted = accepted+1);
 * the *_time fields are the CostBreakdown (expert_model.hpp:54-61) with
 * measured device times in nanoseconds instead of abstract units. */
typedef struct cascade_verify_out {
    int32_t accepted;            /* leading drafts equal to the target argmax */
    int32_t emitted;             /* accepted + 1 */
    int32_t n_tokens;            /* T = K + 1 tokens that were in flight */
    int32_t cache_len;           /* committed KV length after this step */
    int32_t tokens[CASCADE_MAX_TOKENS]; /* emitted: drafts[0..accepted-1] then the bonus */
    int32_t argmax[CASCADE_MAX_TOKENS]; /* target greedy token per in-flight row */
    /* CostBreakdown (expert_model.hpp:54-61), device-measured, ns */
    double attention_time;
    double expert_time;
    double draft_time;           /* host drafter time passed in by the caller */
    double sampling_time;        /* LM head + greedy acceptance */
    double active_experts_per_layer; /* mean over layers of unique routed + shared */
    double total;                /* attention + expert + draft + sampling */
    /* on-device utility of this step: emitted * t_base / total
     * (utility.hpp:59-76 restricted to one iteration); 0 without a baseline */
    double utility;
    double verify_ns;            /* globaltimer: first kernel start -> last kernel end */
} cascade_verify_out;

typedef struct cascade_model cascade_model;
typedef struct cascade_session cascade_session;

/* Last error message of the calling thread (copied, NUL-terminated).
 * Returns the full message length. */
CASCADE_API size_t cascade_last_error(char* buf, size_t n);

/* Validates a geometry; CASCADE_EINVAL with a message when unusable. */
CASCADE_API int cascade_geometry_validate(const cascade_geometry* g);

/* Bytes of device weights the model holds on one rank (expert-parallel
 * shard when ep_size > 1). */
CASCADE_API int cascade_model_bytes(const cascade_geometry* g, int ep_rank, int ep_size, uint64_t* out);

/* Allocates and initialises random weights on `device` from a counter hash
 * of (weight_seed, tensor, row, col): identical on CPU and GPU, so the
 * oracle regenerates any tensor without a host<->device copy. */
CASCADE_API int cascade_model_create(const cascade_geometry* g, uint64_t weight_seed, int device,
                         cascade_model** out);

/* Expert-parallel shard: rank `ep_rank` of `ep_size` holds routed experts
 * [E*r/G, E*(r+1)/G) plus the replicated dense weights; `nccl_unique_id`
 * points to the 128-byte ncclUniqueId created by rank 0 (NCCL is loaded
 * with dlopen at this call only). */
CASCADE_API int cascade_model_create_ep(const cascade_geometry* g, uint64_t weight_seed, int device,
                            int ep_rank, int ep_size, const void* nccl_unique_id,
                            cascade_model** out);
CASCADE_API int cascade_model_destroy(cascade_model* m);

/* Writes a 128-byte ncclUniqueId into `out` (rank 0 only). */
CASCADE_API int cascade_ep_unique_id(void* out, size_t n);

/* One decode request: KV cache for max_ctx positions, CUDA graphs for every
 * in-flight width 1..k_max+1 captured lazily on first use.  The committed KV
 * length never exceeds max_ctx: a committing step whose K+1 rows could take
 * it past max_ctx is refused before launch (CASCADE_ERUNTIME, "full"). */
CASCADE_API int cascade_session_create(cascade_model* m, int max_ctx, int k_max, void* stream,
                           cascade_session** out);
CASCADE_API int cascade_session_destroy(cascade_session* s);

/* Feeds prompt[0..n-2] into the KV cache (chunks of CASCADE_MAX_TOKENS)
 * and keeps prompt[n-1] as the pending token of the next step. */
CASCADE_API int cascade_prefill(cascade_session* s, const int32_t* prompt, int n);

/* Resets the session to an empty cache (weights untouched). */
CASCADE_API int cascade_session_reset(cascade_session* s);

/* No-speculation baseline t_base in ns, used for the on-device utility
 * (utility.hpp:104-117 computes it as the mean of k=0 probe totals). */
CASCADE_API int cascade_set_baseline(cascade_session* s, double t_base_ns);

/* One verification step over the pending token plus `K` drafts (0 <= K <=
 * k_max): host buffers in, host struct out; the H2D of the drafts and the
 * D2H of the result are inside the captured graph.  `draft_ns` is the
 * caller's drafting time, folded into CostBreakdown.draft_time/total.
 * Precondition (checked before launch): cache_len + K + 1 <= max_ctx,
 * else CASCADE_ERUNTIME and the session is unchanged. */
CASCADE_API int cascade_verify(cascade_session* s, const int32_t* draft, int K, double draft_ns,
                   cascade_verify_out* out);

/* Per-layer unique-expert counts (routed, before adding shared blocks) of
 * the last step; `out` holds num_layers ints. */
CASCADE_API int cascade_last_union_sizes(cascade_session* s, int32_t* out, int n);

/* Enqueue-only variant for timing: launches the step graph for width
 * K+1 on the session stream with inputs already resident, no host sync,
 * no result copy.  `commit` = 0 leaves the KV length unchanged so the same
 * context is re-verified every call.  The drafts are the session's current
 * token slots (the last prefill chunk's tokens, or the last verify's
 * drafts).  Step parameters live in one pinned slot per width; a call that
 * changes its width's slot (commit flag, drafts, baseline) first waits for
 * the stream, so an enqueued graph never sees a later call's parameters.
 * A committing enqueue counts K+1 rows against max_ctx until the next
 * cascade_sync, which reads the exact KV length back. */
CASCADE_API int cascade_verify_enqueue(cascade_session* s, int K, int commit);
CASCADE_API int cascade_sync(cascade_session* s);
CASCADE_API void* cascade_session_stream(cascade_session* s);

/* Profiling pass for the roofline: runs one step of width K+1 eagerly
 * (not captured, commit=0) with a CUDA event pair around every kernel on
 * the session stream.  Writes per-launch durations (ns) and a kernel class
 * per launch:  0 embed+norm, 1 QKV GEMV, 2 attention, 3 attention combine,
 * 4 O GEMV, 5 route (norm+router+top-k+union), 6 expert gate/up GEMV,
 * 7 expert down GEMV, 8 combine+norm, 9 LM head GEMV, 10 accept, 11 EP
 * all-reduce.  Returns the number of launches via *n (<= cap). */
CASCADE_API int cascade_profile_step(cascade_session* s, int K, double* ns, int32_t* kind, int cap, int* n);

/* In-graph trace of one step of width K+1 (captured path, commit = 0):
 * every kernel stamps %globaltimer when it starts (after its programmatic
 * dependency wait), so ns[i] = start(i+1) - start(i) is kernel i's share
 * of the step on the real graph timeline; kind[i] uses the classes of
 * cascade_profile_step. */
CASCADE_API int cascade_step_trace(cascade_session* s, int K, double* ns, int32_t* kind, int cap, int* n);

/* Per-CTA timeline of one captured step of width K+1 (diagnostic, commit =
 * 0): out[(i * 512 + cta) * 4 + {0, 1}] = %globaltimer (ns) when CTA `cta`
 * of launch i started (after its dependency wait) and when it exited;
 * {2, 3} = optional phase stamps (expert FFN: gate/up range done, first
 * down-phase readiness wait released); 0 for CTAs / stamps that do not
 * exist (cta >= 496 is not recorded).  kind[i] as in cascade_profile_step;
 * *n_slots = launches (<= cap_slots). */
CASCADE_API int cascade_step_cta_trace(cascade_session* s, int K, uint64_t* out, int32_t* kind, int cap_slots,
                                       int* n_slots);

/* Batch-invariant mode (default off): the expert GEMVs cut every expert
 * block at fixed pieces instead of splitting the active range evenly
 * (stream-K), so a token's logits are bitwise identical whatever the step
 * width and routing of the other tokens, and greedy speculative decoding
 * reproduces the K=0 token sequence exactly.  Costs 5-25% of expert-GEMV
 * time.  Invalidates the captured step graphs. */
CASCADE_API int cascade_set_batch_invariant(cascade_session* s, int on);

/* Number of kernel launches one step of width K+1 performs (graph nodes
 * that are kernels). */
CASCADE_API int cascade_step_kernel_count(cascade_session* s, int K, int* out);

/* Debug taps for the parity tests (teacher forcing).  After the next
 * cascade_verify, copies per-layer tensors of the last step to host:
 *   kind 0: MoE input xn (bf16 bits as uint16)        [L][T][d]
 *   kind 1: router logits (fp32)                      [L][T][E (+1 shared gate)]
 *   kind 2: top-k expert ids (int32)                  [L][T][top_k]
 *   kind 3: top-k weights (fp32)                      [L][T][top_k]
 *   kind 4: MoE output added to the residual (fp32)   [L][T][d]
 *   kind 5: final logits (fp32)                       [T][V]
 *   kind 6: attention input xn (bf16 bits)            [L][T][d]
 *   kind 7: attention block output added to residual (fp32) [L][T][d]
 *   kind 8: residual stream entering each layer (fp32) [L][T][d]
 * Enabling taps switches the session to the un-captured (eager) path. */
CASCADE_API int cascade_enable_taps(cascade_session* s, int enable);
CASCADE_API int cascade_read_tap(cascade_session* s, int kind, void* out, size_t bytes);

/* Copies `n` bf16 weights (as uint16) of a named tensor for tests:
 * tensor kinds follow oracle/cascade_oracle.h (CASCADE_T_*). Logical
 * row-major order, rows [row0, row0+nrows). */
CASCADE_API int cascade_read_weight(cascade_model* m, int kind, int layer, int expert, int row0,
                        int nrows, uint16_t* out);

/* KV cache rows of one layer: [n_kv_heads][len][head_dim] bf16 bits for K
 * (which=0) or V (which=1), positions [0, len). */
CASCADE_API int cascade_read_kv(cascade_session* s, int layer, int which, int len, uint16_t* out);

/* Full speculative decode loop in C++ (host) over the device verifier:
 * n-gram (prompt-lookup) drafter + utility-driven test-and-set controller
 * (controller.hpp:81-321) or a static K.  `policy` = -1: adaptive, k >= 0:
 * static k.  Writes generated tokens to out_tokens (capacity max_new) and,
 * when `telemetry` is non-NULL, one row per iteration (IterationRecord,
 * utility.hpp:32-42, plus the drafts actually offered):
 *   {iter, k_used, tokens_emitted, draft_ns, verify_ns, sampling_ns, total_ns, tag, trial, k_offered}
 * as 10 doubles.  The session is reset first; its max_ctx must hold the
 * prompt plus max_new + 32 tokens.  Returns the number of iterations via *n_iters. */
typedef struct cascade_decode_cfg {
    int32_t policy;            /* -1 adaptive, else static K */
    int32_t max_new;           /* tokens to generate */
    int32_t ngram_n;           /* n-gram match length (prompt lookup) */
    int32_t t_trial, max_trials, s_set, s_cap, k_max, k_start;   /* ControllerConfig */
    double convergence_band;
    int32_t baseline_refresh_interval, baseline_probe_len, backoff_enabled;
    int32_t injected_cost;     /* 1: replace measured time by cost_by_k[k] (K-trace parity) */
    double cost_by_k[CASCADE_MAX_TOKENS];
    /* drafter: 0 = n-gram prompt lookup; 1 = replay of replay_tokens (the
     * model's own greedy continuation of the prompt), each proposal kept
     * with probability replay_p (i.i.d. acceptance as in the reference's
     * workload model, workload.hpp:80-86) */
    int32_t drafter;
    int32_t n_replay;
    const int32_t* replay_tokens;
    double replay_p;
    uint64_t replay_seed;
    /* optional artifacts in the reference's formats (NULL = none):
     *  telemetry_csv: IterationRecord CSV, header kTelemetryCsvHeader
     *                 (report.hpp:123-138), one row per iteration;
     *  trace_path:    acceptance trace "request_id,iter,k_offered,accepted"
     *                 (trace.hpp:36,101-108), rows tagged `request_id`;
     *                 trace_append = 1 adds this request to an existing file. */
    const char* telemetry_csv;
    const char* trace_path;
    int64_t request_id;
    int32_t trace_append;
    int32_t reserved_cfg;
} cascade_decode_cfg;

CASCADE_API int cascade_decode(cascade_session* s, const int32_t* prompt, int n_prompt,
                   const cascade_decode_cfg* cfg, int32_t* out_tokens, int32_t* n_out,
                   double* telemetry, int32_t telemetry_cap, int32_t* n_iters);

/* One cell of the reference scenario sweep (engine.hpp run_cell) on the
 * device: the task's request stream (profile mix with cyclic acceptance
 * phases and output lengths, token budget) decoded under one policy with
 * the profile-driven replay drafter (proposals = the model's own greedy
 * continuation, kept with the current phase's acceptance probability).
 * Sets the session batch-invariant. */
#define CASCADE_CELL_MAX_PROFILES 4
#define CASCADE_CELL_MAX_PHASES 4
typedef struct cascade_cell_cfg {
    int32_t policy;            /* -1 adaptive, 0 none, else static K */
    int32_t t_trial, max_trials, s_set, s_cap, k_max, k_start;   /* ControllerConfig */
    double convergence_band;
    int32_t baseline_refresh_interval, baseline_probe_len, backoff_enabled;
    int32_t n_profiles;
    double share[CASCADE_CELL_MAX_PROFILES];
    int32_t n_phases[CASCADE_CELL_MAX_PROFILES];
    double accept_p[CASCADE_CELL_MAX_PROFILES][CASCADE_CELL_MAX_PHASES];
    double mean_duration[CASCADE_CELL_MAX_PROFILES][CASCADE_CELL_MAX_PHASES];
    int32_t out_len_lo[CASCADE_CELL_MAX_PROFILES], out_len_hi[CASCADE_CELL_MAX_PROFILES];
    int64_t tokens_per_cell;
    int32_t prompt_len;
    uint64_t seed;
} cascade_cell_cfg;

typedef struct cascade_cell_result {
    int64_t requests, iterations, tokens;
    double total_time, t_base, tpot, etr, cost, utility, utility_hmean;  /* device ns; engine.hpp CellResult */
} cascade_cell_result;

CASCADE_API int cascade_run_cell(cascade_session* s, const cascade_cell_cfg* cfg, cascade_cell_result* out);

/* Geometry of the model a session runs (for host code above the ABI). */
CASCADE_API int cascade_session_geometry(cascade_session* s, cascade_geometry* out);

/* Device replay of an acceptance trace (the reference's `replay` command,
 * tools/specsim.cpp:123-160, over engine.hpp replay_request 194-248 with the
 * priced step replaced by real verification steps).  Every request of the
 * trace (first-appearance order) is replayed under the policy of `cfg`
 * (policy and ControllerConfig fields; -1 adaptive, 0 none, k static) on a
 * random prompt of `prompt_len` tokens drawn from `seed`: each iteration's
 * acceptance is the recorded one truncated to the offered k, forced on the
 * real model by its own greedy continuation, and the costs are measured.
 * Writes `out_csv` (NULL = none) in the reference's replay.csv format
 * "request_id,iterations,tokens,total_time,t_base,tpot,etr,cost,utility";
 * `total` receives the aggregate (requests, iterations, tokens, total_time,
 * tpot, utility_hmean); `mismatches` the number of iterations where the
 * device accepted a different count than the trace asked (0 expected). */
CASCADE_API int cascade_replay_trace(cascade_session* s, const char* trace_path, const cascade_decode_cfg* cfg,
                                     int32_t prompt_len, uint64_t seed, const char* out_csv,
                                     cascade_cell_result* total, int64_t* mismatches);

/* Device-backed scenario sweep: the reference's run_scenario (engine.hpp:
 * 418-466) over verifier cells, reading the reference's scenario JSON
 * (scenario.hpp schema; proj/fixtures/*.json load unchanged).  Cells are
 * tasks x policies of the file on the loaded model (`model_name` in the
 * report); `sessions[0..n_sessions)` are worker sessions, one per GPU (each
 * on its own device's copy of the model), each running whole cells.
 * tokens_per_cell > 0 overrides the file.  Writes out_dir/cells.csv and
 * out_dir/summary.json in the reference's report formats (report.hpp).
 * *n_cells = number of cells (failed cells are reported in the files). */
CASCADE_API int cascade_run_scenario(cascade_session* const* sessions, int n_sessions, const char* scenario_json,
                                     const char* out_dir, int64_t tokens_per_cell, int32_t prompt_len,
                                     const char* model_name, int32_t* n_cells);

/* Library build identity: "sm_100a" plus the git hash baked at build. */
CASCADE_API const char* cascade_build_info(void);

#ifdef __cplusplus
}
#endif

#endif /* CASCADE_H_ */
