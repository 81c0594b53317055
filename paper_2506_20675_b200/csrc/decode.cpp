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
#include "specsim/report.hpp"
#include "specsim/scenario.hpp"
#include "specsim/verifier.hpp"

// cascade.cu owns the thread's error slot; route messages through a tiny
// setter it exports internally.
extern "C" int cascade_internal_set_error(int code, const char* msg);
extern "C" int cascade_internal_vocab(const cascade_session* s);

namespace {

// Policy of a decode / cell config (-1 adaptive with its ControllerConfig,
// 0 none, k static; the verifier allows k up to CASCADE_MAX_K, past the
// reference's k <= 7).
template <typename Cfg>
specsim::Policy policy_of(const Cfg& cfg) {
    using namespace specsim;
    if (cfg.policy == 0) return Policy::none();
    if (cfg.policy > 0) {
        if (cfg.policy > CASCADE_MAX_K) throw std::invalid_argument("static policy: k must be in [0,15]");
        Policy p;
        p.kind = Policy::Kind::static_k;
        p.k = cfg.policy;
        return p;
    }
    ControllerConfig c;
    c.t_trial = cfg.t_trial;
    c.max_trials = cfg.max_trials;
    c.s_set = cfg.s_set;
    c.s_cap = cfg.s_cap;
    c.k_max = cfg.k_max;
    c.k_start = cfg.k_start;
    c.convergence_band = cfg.convergence_band;
    c.baseline_refresh_interval = cfg.baseline_refresh_interval;
    c.baseline_probe_len = cfg.baseline_probe_len;
    c.backoff_enabled = cfg.backoff_enabled != 0;
    return Policy::adaptive(c);
}

// Runs `body`, mapping the reference's exception classes to status codes.
template <typename F>
int guarded(F&& body) {
    using namespace specsim;
    try {
        return body();
    } catch (const std::invalid_argument& e) {
        return cascade_internal_set_error(CASCADE_EINVAL, e.what());
    } catch (const MissingBaselineError& e) {
        return cascade_internal_set_error(CASCADE_ENOBASE, e.what());
    } catch (const std::exception& e) {
        return cascade_internal_set_error(CASCADE_ERUNTIME, e.what());
    }
}

// Appends (or writes) the request's acceptance records to a trace file in
// the reference's format (trace.hpp AcceptanceTrace::save / load).
void write_trace(const std::vector<specsim::TraceRecord>& recs, const char* path, bool append) {
    specsim::AcceptanceTrace t;
    if (append && std::filesystem::exists(path)) t = specsim::AcceptanceTrace::load(path);
    for (const specsim::TraceRecord& r : recs) t.add(r);
    t.save(path);
}

}  // namespace

extern "C" int cascade_decode(cascade_session* s, const int32_t* prompt, int n_prompt, const cascade_decode_cfg* cfg,
                              int32_t* out_tokens, int32_t* n_out, double* telemetry, int32_t telemetry_cap,
                              int32_t* n_iters) {
    using namespace specsim;
    if (!s || !prompt || !cfg || !out_tokens || !n_out || !n_iters)
        return cascade_internal_set_error(CASCADE_EINVAL, "cascade_decode: NULL argument");
    if (n_prompt < 1 || cfg->max_new < 1)
        return cascade_internal_set_error(CASCADE_EINVAL, "cascade_decode: need a prompt and max_new >= 1");
    return guarded([&]() -> int {
        int rc = cascade_session_reset(s);
        if (rc) return rc;
        const Policy policy = policy_of(*cfg);
        GpuRunOptions opt;
        opt.engine.keep_telemetry = true;
        opt.k_limit = CASCADE_MAX_K;
        opt.trace_request_id = static_cast<long>(cfg->request_id);
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
        if (cfg->telemetry_csv) write_telemetry_csv(m.telemetry, cfg->telemetry_csv);
        if (cfg->trace_path) write_trace(trace, cfg->trace_path, cfg->trace_append != 0);
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
    });
}

extern "C" int cascade_run_cell(cascade_session* s, const cascade_cell_cfg* cfg, cascade_cell_result* out) {
    using namespace specsim;
    if (!s || !cfg || !out) return cascade_internal_set_error(CASCADE_EINVAL, "cascade_run_cell: NULL argument");
    return guarded([&]() -> int {
        if (cfg->n_profiles < 1 || cfg->n_profiles > CASCADE_CELL_MAX_PROFILES)
            throw std::invalid_argument("cascade_run_cell: n_profiles must be in [1,4]");
        const Policy policy = policy_of(*cfg);
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
    });
}

extern "C" int cascade_replay_trace(cascade_session* s, const char* trace_path, const cascade_decode_cfg* cfg,
                                    int32_t prompt_len, uint64_t seed, const char* out_csv, cascade_cell_result* total,
                                    int64_t* mismatches) {
    using namespace specsim;
    if (!s || !trace_path || !cfg) return cascade_internal_set_error(CASCADE_EINVAL, "cascade_replay_trace: NULL argument");
    return guarded([&]() -> int {
        if (prompt_len < 1) throw std::invalid_argument("cascade_replay_trace: prompt_len must be >= 1");
        const AcceptanceTrace trace = AcceptanceTrace::load(trace_path);
        const Policy policy = policy_of(*cfg);
        GpuRunOptions opt;
        opt.k_limit = CASCADE_MAX_K;
        Verifier v(s);
        const int vocab = v.vocab();
        std::ofstream csv;
        if (out_csv) {
            csv.open(out_csv);
            if (!csv) throw std::runtime_error(std::string("cannot write ") + out_csv);
            csv << "request_id,iterations,tokens,total_time,t_base,tpot,etr,cost,utility\n";
        }
        long tokens = 0, iterations = 0, bad_total = 0;
        double time = 0.0;
        std::vector<double> utils;
        for (long id : trace.request_ids()) {
            Rng prng(splitmix64(seed + static_cast<std::uint64_t>(id)));
            std::uniform_int_distribution<int32_t> tok(0, vocab - 1);
            std::vector<int32_t> prompt(static_cast<std::size_t>(prompt_len));
            for (int32_t& t : prompt) t = tok(prng);
            long bad = 0;
            const RequestMetrics m = replay_request(v, trace, id, policy, prompt, opt, &bad);
            bad_total += bad;
            if (out_csv)
                csv << id << ',' << m.iterations << ',' << m.tokens << ',' << fmt_num(m.total_time) << ','
                    << fmt_num(m.t_base) << ',' << fmt_num(m.tpot) << ',' << fmt_num(m.etr) << ','
                    << fmt_num(m.cost) << ',' << fmt_num(m.utility) << "\n";
            tokens += m.tokens;
            iterations += m.iterations;
            time += m.total_time;
            utils.push_back(m.utility);
        }
        if (total) {
            *total = cascade_cell_result{};
            total->requests = static_cast<int64_t>(utils.size());
            total->iterations = iterations;
            total->tokens = tokens;
            total->total_time = time;
            total->tpot = time / static_cast<double>(tokens);
            total->etr = static_cast<double>(tokens) / static_cast<double>(iterations);
            total->utility_hmean = harmonic_mean(utils);
        }
        if (mismatches) *mismatches = bad_total;
        return CASCADE_OK;
    });
}

extern "C" int cascade_run_scenario(cascade_session* const* sessions, int n_sessions, const char* scenario_json,
                                    const char* out_dir, int64_t tokens_per_cell, int32_t prompt_len,
                                    const char* model_name, int32_t* n_cells) {
    using namespace specsim;
    if (!sessions || n_sessions < 1 || !scenario_json || !out_dir)
        return cascade_internal_set_error(CASCADE_EINVAL, "cascade_run_scenario: NULL argument");
    return guarded([&]() -> int {
        ScenarioConfig cfg = load_scenario(scenario_json);
        if (tokens_per_cell > 0) cfg.tokens_per_cell = static_cast<long>(tokens_per_cell);
        std::vector<Verifier> vs;
        vs.reserve(static_cast<std::size_t>(n_sessions));
        for (int i = 0; i < n_sessions; ++i) {
            if (!sessions[i]) throw std::invalid_argument("cascade_run_scenario: NULL session");
            vs.emplace_back(sessions[i]);
        }
        std::vector<Verifier*> ptrs;
        for (Verifier& v : vs) ptrs.push_back(&v);
        GpuRunOptions opt;
        opt.k_limit = CASCADE_MAX_K;
        const ScenarioReport rep = run_scenario(ptrs, cfg, model_name ? model_name : "device", prompt_len, opt);
        std::filesystem::create_directories(out_dir);
        write_cells_csv(rep, std::filesystem::path(out_dir) / "cells.csv");
        write_summary_json(rep, std::filesystem::path(out_dir) / "summary.json");
        if (n_cells) *n_cells = static_cast<int32_t>(rep.cells.size());
        return CASCADE_OK;
    });
}
