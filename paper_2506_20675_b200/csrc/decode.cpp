// decode.cpp — cascade_decode: the full speculative decode loop in host C++
// (n-gram drafter -> GPU verify -> utility analyzer -> test-and-set
// controller), i.e. the reference's run_request loop (engine.hpp:115-182)
// with the priced step replaced by the device step.  Errors thrown by the
// specsim host code are mapped back to C status codes.
#include <array>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "cascade.h"
#include "specsim/verifier.hpp"

// cascade.cu owns the thread's error slot; route messages through a tiny
// setter it exports internally.
extern "C" int cascade_internal_set_error(int code, const char* msg);
extern "C" int cascade_internal_vocab(const cascade_session* s);

extern "C" int cascade_decode(cascade_session* s, const int32_t* prompt, int n_prompt, const cascade_decode_cfg* cfg,
                              int32_t* out_tokens, int32_t* n_out, double* telemetry, int32_t telemetry_cap,
                              int32_t* n_iters) {
    using namespace specsim;
    if (!s || !prompt || !cfg || !out_tokens || !n_out || !n_iters)
        return cascade_internal_set_error(CASCADE_EINVAL, "cascade_decode: NULL argument");
    if (n_prompt < 1 || cfg->max_new < 1)
        return cascade_internal_set_error(CASCADE_EINVAL, "cascade_decode: need a prompt and max_new >= 1");
    try {
        int rc = cascade_session_reset(s);
        if (rc) return rc;
        Policy policy;
        if (cfg->policy < 0) {
            ControllerConfig c;
            c.t_trial = cfg->t_trial;
            c.max_trials = cfg->max_trials;
            c.s_set = cfg->s_set;
            c.s_cap = cfg->s_cap;
            c.k_max = cfg->k_max;
            c.k_start = cfg->k_start;
            c.convergence_band = cfg->convergence_band;
            c.baseline_refresh_interval = cfg->baseline_refresh_interval;
            c.baseline_probe_len = cfg->baseline_probe_len;
            c.backoff_enabled = cfg->backoff_enabled != 0;
            policy = Policy::adaptive(c);
        } else if (cfg->policy == 0) {
            policy = Policy::none();
        } else {
            if (cfg->policy > CASCADE_MAX_K) throw std::invalid_argument("static policy: k must be in [0,15]");
            policy.kind = Policy::Kind::static_k;  // the verifier goes past the reference's k<=7
            policy.k = cfg->policy;
        }
        GpuRunOptions opt;
        opt.engine.keep_telemetry = true;
        opt.k_limit = CASCADE_MAX_K;
        if (cfg->injected_cost) {
            std::array<double, CASCADE_MAX_TOKENS> c{};
            for (int i = 0; i < CASCADE_MAX_TOKENS; ++i) c[i] = cfg->cost_by_k[i];
            opt.injected_cost = c;
        }
        std::vector<TraceRecord> trace;
        opt.trace = &trace;
        std::vector<int32_t> toks(prompt, prompt + n_prompt);
        Verifier v(s);
        RequestMetrics m;
        if (cfg->drafter == 1) {
            if (!cfg->replay_tokens || cfg->n_replay < 1)
                throw std::invalid_argument("cascade_decode: replay drafter needs replay_tokens");
            const int vocab = cascade_internal_vocab(s);
            ReplayDrafter drafter(std::vector<int32_t>(cfg->replay_tokens, cfg->replay_tokens + cfg->n_replay), n_prompt,
                                  cfg->replay_p, vocab, cfg->replay_seed);
            m = run_request(v, drafter, policy, toks, cfg->max_new, opt);
        } else if (cfg->drafter == 0) {
            NgramDrafter drafter(cfg->ngram_n);
            m = run_request(v, drafter, policy, toks, cfg->max_new, opt);
        } else {
            throw std::invalid_argument("cascade_decode: drafter must be 0 (n-gram) or 1 (replay)");
        }
        const int gen = static_cast<int>(toks.size()) - n_prompt;
        const int cap = cfg->max_new + CASCADE_MAX_TOKENS;
        const int n = gen < cap ? gen : cap;
        std::memcpy(out_tokens, toks.data() + n_prompt, static_cast<size_t>(n) * sizeof(int32_t));
        *n_out = n;
        *n_iters = static_cast<int32_t>(m.telemetry.size());
        if (telemetry) {
            const int rows = std::min<int>(telemetry_cap, static_cast<int>(m.telemetry.size()));
            for (int i = 0; i < rows; ++i) {
                const IterationRecord& r = m.telemetry[i];
                double* o = telemetry + 10 * i;
                o[0] = static_cast<double>(r.iter_index);
                o[1] = r.k_used;
                o[2] = r.tokens_emitted;
                o[3] = r.draft_time;
                o[4] = r.verify_time;
                o[5] = r.sampling_time;
                o[6] = r.total_time;
                o[7] = static_cast<double>(static_cast<int>(r.tag));
                o[8] = r.trial_no;
                o[9] = trace[i].k_offered;
            }
        }
        return CASCADE_OK;
    } catch (const std::invalid_argument& e) {
        return cascade_internal_set_error(CASCADE_EINVAL, e.what());
    } catch (const MissingBaselineError& e) {
        return cascade_internal_set_error(CASCADE_ENOBASE, e.what());
    } catch (const std::exception& e) {
        return cascade_internal_set_error(CASCADE_ERUNTIME, e.what());
    }
}

extern "C" int cascade_run_cell(cascade_session* s, const cascade_cell_cfg* cfg, cascade_cell_result* out) {
    using namespace specsim;
    if (!s || !cfg || !out) return cascade_internal_set_error(CASCADE_EINVAL, "cascade_run_cell: NULL argument");
    try {
        if (cfg->n_profiles < 1 || cfg->n_profiles > CASCADE_CELL_MAX_PROFILES)
            throw std::invalid_argument("cascade_run_cell: n_profiles must be in [1,4]");
        Policy policy;
        if (cfg->policy < 0) {
            ControllerConfig c;
            c.t_trial = cfg->t_trial;
            c.max_trials = cfg->max_trials;
            c.s_set = cfg->s_set;
            c.s_cap = cfg->s_cap;
            c.k_max = cfg->k_max;
            c.k_start = cfg->k_start;
            c.convergence_band = cfg->convergence_band;
            c.baseline_refresh_interval = cfg->baseline_refresh_interval;
            c.baseline_probe_len = cfg->baseline_probe_len;
            c.backoff_enabled = cfg->backoff_enabled != 0;
            policy = Policy::adaptive(c);
        } else if (cfg->policy == 0) {
            policy = Policy::none();
        } else {
            if (cfg->policy > CASCADE_MAX_K) throw std::invalid_argument("static policy: k must be in [0,15]");
            policy.kind = Policy::Kind::static_k;
            policy.k = cfg->policy;
        }
        RequestStream task;
        for (int i = 0; i < cfg->n_profiles; ++i) {
            if (cfg->n_phases[i] < 1 || cfg->n_phases[i] > CASCADE_CELL_MAX_PHASES)
                throw std::invalid_argument("cascade_run_cell: n_phases must be in [1,4]");
            WorkloadProfile prof;
            prof.name = "profile" + std::to_string(i);
            for (int j = 0; j < cfg->n_phases[i]; ++j) {
                AcceptancePhase ph;
                ph.per_token_accept_prob = cfg->accept_p[i][j];
                ph.mean_duration = cfg->mean_duration[i][j];
                prof.phases.push_back(ph);
            }
            prof.transition = PhaseTransition::cyclic;
            prof.output_len.lo = cfg->out_len_lo[i];
            prof.output_len.hi = cfg->out_len_hi[i];
            task.mix.emplace_back(prof, cfg->share[i]);
        }
        task.max_tokens = cfg->tokens_per_cell;
        int rc = cascade_set_batch_invariant(s, 1);
        if (rc) return rc;
        GpuRunOptions opt;
        opt.k_limit = CASCADE_MAX_K;
        Verifier v(s);
        const CellResult c = run_cell(v, cascade_internal_vocab(s), task, policy, cfg->tokens_per_cell,
                                      cfg->prompt_len, cfg->seed, opt);
        out->requests = c.requests;
        out->iterations = c.iterations;
        out->tokens = c.tokens;
        out->total_time = c.total_time;
        out->t_base = c.t_base;
        out->tpot = c.tpot;
        out->etr = c.etr;
        out->cost = c.cost;
        out->utility = c.utility;
        out->utility_hmean = c.utility_hmean;
        return CASCADE_OK;
    } catch (const std::invalid_argument& e) {
        return cascade_internal_set_error(CASCADE_EINVAL, e.what());
    } catch (const MissingBaselineError& e) {
        return cascade_internal_set_error(CASCADE_ENOBASE, e.what());
    } catch (const std::exception& e) {
        return cascade_internal_set_error(CASCADE_ERUNTIME, e.what());
    }
}
