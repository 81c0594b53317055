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

#include "landscape_harness.hpp"
#include "specsim/engine.hpp"
#include "specsim/expert_model.hpp"
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

}  // extern "C"
