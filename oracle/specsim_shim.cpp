// specsim_shim.cpp — extern "C" shim over a `specsim` header set.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles it twice:
//  * `make ref`  -> oracle/_ref/libspecsim_ref.so against the UNMODIFIED
//    reference headers where they lie (/root/reference/proj/include, plus
//    the reference harness /root/reference/proj/tests/landscape_harness.hpp);
//  * `make ours` -> oracle/libspecsim_ours.so against this repository's
//    include/specsim (plus tests/cpp/landscape_harness.hpp).
// tests/test_specsim_parity.py calls both with identical inputs and
// requires identical outputs; tests/golden/make_golden.py records the
// reference's outputs as committed golden vectors; bench.py times the
// reference build as the reference CPU path.  Nothing here is copied from
// the reference; the shim only calls the API.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include <cstdio>
#include <sstream>
#include <string>

#include "landscape_harness.hpp"
#include "specsim/engine.hpp"
#include "specsim/expert_model.hpp"
#include "specsim/report.hpp"
#include "specsim/scenario.hpp"
#include "specsim/trace.hpp"
#include "specsim/utility.hpp"
#include "specsim/workload.hpp"

using namespace specsim;

extern "C" {

double ref_expected_unique_experts(int E, int k, int T) { return expected_unique_experts(E, k, T); }

// n draws of sample_active_experts for (E, top_k, shared, affinity) at `tokens`
int ref_sample_active_experts(int E, int top_k, int shared, double affinity, int tokens, uint64_t seed, int n,
                              double* out) {
    try {
        ExpertConfig c;
        c.experts_per_layer = E;
        c.top_k = top_k;
        c.shared_experts = shared;
        c.affinity = affinity;
        Rng rng(seed);
        for (int i = 0; i < n; ++i) out[i] = sample_active_experts(c, tokens, rng);
        return 0;
    } catch (...) {
        return -1;
    }
}

// out[6] = attention, expert, draft, sampling, active, total (one call)
int ref_iteration_cost(const char* preset, const char* draft, int k, uint64_t seed, int n, double* out) {
    try {
        const ExpertConfig c = expert_preset(preset);
        const DraftCostModel d = draft_preset(draft);
        Rng rng(seed);
        for (int i = 0; i < n; ++i) {
            const CostBreakdown b = iteration_cost(c, d, k, rng);
            double* o = out + 6 * i;
            o[0] = b.attention_time;
            o[1] = b.expert_time;
            o[2] = b.draft_time;
            o[3] = b.sampling_time;
            o[4] = b.active_experts_per_layer;
            o[5] = b.total;
        }
        return 0;
    } catch (...) {
        return -1;
    }
}

// Times the reference verify step (iteration_cost + sample_accepted) on
// `threads` host threads, `calls_per_thread` calls each.  Returns the
// aggregate wall time in ns.
double ref_time_verify(const char* preset, int k, double p_accept, int threads, long calls_per_thread) {
    const ExpertConfig c = expert_preset(preset);
    const DraftCostModel d = draft_preset("ngram");
    std::vector<std::thread> pool;
    std::vector<long> sink(threads, 0);
    const auto t0 = std::chrono::steady_clock::now();
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t]() {
            Rng rng(1234 + t);
            long acc = 0;
            for (long i = 0; i < calls_per_thread; ++i) {
                const CostBreakdown b = iteration_cost(c, d, k, rng);
                acc += sample_accepted(p_accept, k, rng) + (b.total > 0 ? 1 : 0);
            }
            sink[t] = acc;
        });
    for (auto& th : pool) th.join();
    const auto t1 = std::chrono::steady_clock::now();
    volatile long keep = 0;
    for (long v : sink) keep += v;
    (void)keep;
    return std::chrono::duration<double, std::nano>(t1 - t0).count();
}

int ref_sample_accepted(double p, int k, uint64_t seed, int n, int32_t* out) {
    try {
        Rng rng(seed);
        for (int i = 0; i < n; ++i) out[i] = sample_accepted(p, k, rng);
        return 0;
    } catch (...) {
        return -1;
    }
}

int ref_trace_replay(int k_offered, int accepted, int k) {
    AcceptanceTrace tr;
    tr.add({0, 0, k_offered, accepted});
    return tr.replay(0, 0, k);
}

// Drives the reference controller with the reference harness.
// cfg_i[9] = t_trial, max_trials, s_set, s_cap, k_max, k_start, refresh, probe_len, backoff
// util[k] for k=0..15 (U(k), k>=1), optionally switching at iter `switch_iter` to util2.
int ref_drive_controller(const int32_t* cfg_i, double band, const double* util, long switch_iter,
                         const double* util2, long max_iters, int stop_after_sets, double noise,
                         uint64_t noise_seed, int32_t* k_seq, int32_t* tags, long* n_iters, long* test_iters,
                         double* total_time, int32_t* set_k, int32_t* set_len, int* n_sets) {
    try {
        ControllerConfig cfg;
        cfg.t_trial = cfg_i[0];
        cfg.max_trials = cfg_i[1];
        cfg.s_set = cfg_i[2];
        cfg.s_cap = cfg_i[3];
        cfg.k_max = cfg_i[4];
        cfg.k_start = cfg_i[5];
        cfg.baseline_refresh_interval = cfg_i[6];
        cfg.baseline_probe_len = cfg_i[7];
        cfg.backoff_enabled = cfg_i[8] != 0;
        cfg.convergence_band = band;
        auto fn = [&](int k, long iter) {
            if (switch_iter >= 0 && iter >= switch_iter) return util2[k];
            return util[k];
        };
        const auto res = harness::drive_controller(cfg, fn, max_iters, (std::size_t)stop_after_sets, noise,
                                                   noise_seed);
        for (std::size_t i = 0; i < res.k_sequence.size(); ++i) {
            k_seq[i] = res.k_sequence[i];
            tags[i] = (int32_t)res.tags[i];
        }
        *n_iters = (long)res.k_sequence.size();
        *test_iters = res.test_iterations;
        *total_time = res.total_time;
        *n_sets = (int)res.sets.size();
        for (std::size_t i = 0; i < res.sets.size(); ++i) {
            set_k[i] = res.sets[i].k;
            set_len[i] = res.sets[i].length;
        }
        return 0;
    } catch (...) {
        return -1;
    }
}

// run_request on a one-phase profile; out[8] = tokens, iterations, total_time,
// t_base, tpot, etr, cost, utility
int ref_run_request(double p, double affinity, int out_len, int policy, const char* preset, const char* draft,
                    uint64_t seed, double* out) {
    try {
        WorkloadProfile prof;
        prof.name = "flat";
        prof.phases = {{p, 1.0, std::nullopt}};
        prof.expert_affinity = affinity;
        prof.output_len = {out_len, out_len};
        Policy pol = policy < 0 ? Policy::adaptive({}) : (policy == 0 ? Policy::none() : Policy::static_k(policy));
        const RequestMetrics m = run_request(prof, pol, expert_preset(preset), draft_preset(draft), seed);
        out[0] = (double)m.tokens;
        out[1] = (double)m.iterations;
        out[2] = m.total_time;
        out[3] = m.t_base;
        out[4] = m.tpot;
        out[5] = m.etr;
        out[6] = m.cost;
        out[7] = m.utility;
        return 0;
    } catch (...) {
        return -1;
    }
}

// Replays recorded iterations (tokens, total time) through a fresh
// controller; writes the k the controller chose before each record and its
// tag.  Used to check the GPU decode loop's K trace (cascade_decode with an
// injected cost) against this controller.
int ref_controller_replay(const int32_t* cfg_i, double band, int n, const int32_t* tokens, const double* total,
                          int32_t* k_out, int32_t* tag_out) {
    try {
        ControllerConfig cfg;
        cfg.t_trial = cfg_i[0];
        cfg.max_trials = cfg_i[1];
        cfg.s_set = cfg_i[2];
        cfg.s_cap = cfg_i[3];
        cfg.k_max = cfg_i[4];
        cfg.k_start = cfg_i[5];
        cfg.baseline_refresh_interval = cfg_i[6];
        cfg.baseline_probe_len = cfg_i[7];
        cfg.backoff_enabled = cfg_i[8] != 0;
        cfg.convergence_band = band;
        SpeculationController ctl(cfg);
        UtilityAnalyzer an(16);
        for (int i = 0; i < n; ++i) {
            IterationRecord r;
            r.iter_index = i;
            r.k_used = ctl.current_k();
            r.tag = ctl.current_tag();
            r.trial_no = ctl.current_trial();
            r.tokens_emitted = tokens[i];
            if (r.tokens_emitted > r.k_used + 1) r.tokens_emitted = r.k_used + 1;
            r.total_time = total[i];
            r.verify_time = total[i];
            k_out[i] = r.k_used;
            tag_out[i] = (int32_t)r.tag;
            ctl.next_k(r, an);
        }
        return 0;
    } catch (...) {
        return -1;
    }
}

// UtilityAnalyzer window arithmetic on given records; out[3] = etr, cost, utility
int ref_window_utility(int window, double t_base, int n, const int32_t* k, const int32_t* tokens,
                       const double* total, const int32_t* tag, double* out) {
    try {
        UtilityAnalyzer an(window);
        an.set_baseline(t_base);
        for (int i = 0; i < n; ++i) {
            IterationRecord r;
            r.iter_index = i;
            r.k_used = k[i];
            r.tokens_emitted = tokens[i];
            r.total_time = total[i];
            r.verify_time = total[i];
            r.tag = (PhaseTag)tag[i];
            an.record(r);
        }
        out[0] = an.window_etr();
        out[1] = an.window_cost();
        out[2] = an.window_utility();
        return 0;
    } catch (...) {
        return -1;
    }
}

// ---- report / trace / scenario interop (f3, f4) --------------------------

// AcceptanceTrace::load; out[4*i..] = request_id, iter, k_offered, accepted.
// Returns the record count (<= cap), -1 on error.
long ref_trace_load(const char* path, int64_t* out, long cap) {
    try {
        const AcceptanceTrace t = AcceptanceTrace::load(path);
        long n = 0;
        for (const TraceRecord& r : t.records()) {
            if (n >= cap) break;
            out[4 * n] = r.request_id;
            out[4 * n + 1] = r.iter;
            out[4 * n + 2] = r.k_offered;
            out[4 * n + 3] = r.accepted;
            ++n;
        }
        return n;
    } catch (...) {
        return -1;
    }
}

// replay_request of one request of a trace file (mixtral preset, ngram
// draft, policy -1 adaptive / 0 none / k static, rng seed); out[8] as
// ref_run_request; emitted[i] = tokens_emitted of iteration i.  Returns the
// iteration count, -1 on error.
long ref_trace_replay_request(const char* path, long request_id, int policy, uint64_t seed, double* out,
                              int32_t* emitted, long cap) {
    try {
        const AcceptanceTrace t = AcceptanceTrace::load(path);
        Policy pol = policy < 0 ? Policy::adaptive({}) : (policy == 0 ? Policy::none() : Policy::static_k(policy));
        Rng rng(seed);
        EngineOptions opts;
        opts.keep_telemetry = true;
        const RequestMetrics m =
            replay_request(t, request_id, pol, expert_preset("mixtral"), draft_preset("ngram"), rng, opts);
        out[0] = (double)m.tokens;
        out[1] = (double)m.iterations;
        out[2] = m.total_time;
        out[3] = m.t_base;
        out[4] = m.tpot;
        out[5] = m.etr;
        out[6] = m.cost;
        out[7] = m.utility;
        long n = 0;
        for (const IterationRecord& r : m.telemetry)
            if (n < cap) emitted[n++] = r.tokens_emitted;
        return (long)m.telemetry.size();
    } catch (...) {
        return -1;
    }
}

// write_telemetry_csv of n records given as rows of 9 doubles
// (iter, k, tokens, draft, verify, sampling, total, tag, trial).
int ref_write_telemetry(const char* path, int n, const double* rows) {
    try {
        std::vector<IterationRecord> recs(n);
        for (int i = 0; i < n; ++i) {
            const double* r = rows + 9 * i;
            recs[i].iter_index = (long)r[0];
            recs[i].k_used = (int)r[1];
            recs[i].tokens_emitted = (int)r[2];
            recs[i].draft_time = r[3];
            recs[i].verify_time = r[4];
            recs[i].sampling_time = r[5];
            recs[i].total_time = r[6];
            recs[i].tag = (PhaseTag)(int)r[7];
            recs[i].trial_no = (int)r[8];
        }
        write_telemetry_csv(recs, path);
        return 0;
    } catch (...) {
        return -1;
    }
}

// Runs the simulated scenario sweep of a scenario file (tokens override >0)
// and writes cells.csv + summary.json (without the timestamp line) to dir.
int ref_scenario_report(const char* scenario, long tokens, const char* dir) {
    try {
        ScenarioConfig cfg = load_scenario(scenario);
        if (tokens > 0) cfg.tokens_per_cell = tokens;
        const ScenarioReport rep = run_scenario(cfg);
        write_cells_csv(rep, std::string(dir) + "/cells.csv");
        std::ofstream out(std::string(dir) + "/summary.json");
        out << summary_json(rep, false).dump(2) << "\n";
        return 0;
    } catch (...) {
        return -1;
    }
}

// load_cells_csv; out[3*i..] = requests, tokens, utility; returns the row
// count (<= cap) or -1.
long ref_load_cells(const char* path, double* out, long cap) {
    try {
        const std::vector<CellResult> cells = load_cells_csv(path);
        long n = 0;
        for (const CellResult& c : cells) {
            if (n >= cap) break;
            out[3 * n] = (double)c.requests;
            out[3 * n + 1] = (double)c.tokens;
            out[3 * n + 2] = c.utility;
            ++n;
        }
        return (long)cells.size();
    } catch (...) {
        return -1;
    }
}

// A canonical text digest of a parsed scenario (for parser parity).
// Returns the digest length (copied into buf, NUL-terminated) or -1.
long ref_scenario_digest(const char* path, char* buf, long n) {
    try {
        const ScenarioConfig c = load_scenario(path);
        std::ostringstream o;
        o.precision(17);
        o << c.name << '|' << c.seed << '|' << c.seed_in_file << '|' << c.tokens_per_cell << '|' << c.jobs << '|'
          << (int)c.draft.kind << ',' << c.draft.per_k_overhead << ',' << c.draft.sampling_overhead << ','
          << c.draft.always_on_overhead << "\n";
        for (const ExpertConfig& m : c.models)
            o << "M " << m.name << ',' << m.num_layers << ',' << m.experts_per_layer << ',' << m.top_k << ','
              << m.shared_experts << ',' << m.affinity << ',' << m.baseline_iter_time << ',' << m.attention_fraction
              << "\n";
        for (const TaskSpec& t : c.tasks) {
            o << "T " << t.name << "\n";
            for (const auto& [p, share] : t.stream.mix) {
                o << "  P " << p.name << ',' << share << ',' << (int)p.transition << ',' << p.output_len.lo << ','
                  << p.output_len.hi << ',' << (p.expert_affinity ? *p.expert_affinity : -1.0) << "\n";
                for (const AcceptancePhase& ph : p.phases)
                    o << "    " << ph.per_token_accept_prob << ',' << ph.mean_duration << ','
                      << (ph.affinity_override ? *ph.affinity_override : -1.0) << "\n";
                for (const auto& row : p.transition_matrix) {
                    o << "    R";
                    for (double v : row) o << ' ' << v;
                    o << "\n";
                }
            }
        }
        for (const Policy& p : c.policies) {
            const ControllerConfig& k = p.controller;
            o << "P " << p.label() << ',' << k.t_trial << ',' << k.max_trials << ',' << k.s_set << ',' << k.s_cap
              << ',' << k.k_max << ',' << k.k_start << ',' << k.convergence_band << ',' << k.baseline_refresh_interval
              << ',' << k.baseline_probe_len << ',' << k.backoff_enabled << "\n";
        }
        const std::string d = o.str();
        if (buf && n > 0) {
            const long c2 = (long)d.size() < n - 1 ? (long)d.size() : n - 1;
            std::memcpy(buf, d.data(), (size_t)c2);
            buf[c2] = 0;
        }
        return (long)d.size();
    } catch (...) {
        return -1;
    }
}

}  // extern "C"
