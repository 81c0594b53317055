// specsim/verifier.hpp — the GPU-backed side of the drop-in seam.
//
// The reference request loop prices a verification step and draws an
// acceptance outcome (proj/include/specsim/engine.hpp:158-159):
//     cost     = iteration_cost(iter_cfg, draft, k, rng);
//     accepted = pstate.sample_accepted(k, rng);
// Here both become one real step on the B200 through the C ABI
// (include/cascade.h): `Verifier::verify` runs the K+1 tokens through the
// model and returns the device-measured CostBreakdown (ns) and the greedy
// accepted prefix.  `run_request(Verifier&, ...)` is the engine.hpp:140-179
// loop with that seam swapped and an n-gram (prompt-lookup) drafter in
// front; everything above the seam (IterationRecord -> SpeculationController
// -> UtilityAnalyzer) is the unchanged host logic of specsim/*.hpp.
#pragma once

#include <array>
#include <atomic>
#include <chrono>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "cascade.h"
#include "specsim/engine.hpp"

namespace specsim {

struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Rethrows a C status code as the reference's exception classes.
inline void check_status(int rc) {
    if (rc == CASCADE_OK) return;
    char msg[1024];
    cascade_last_error(msg, sizeof(msg));
    switch (rc) {
    case CASCADE_EINVAL: throw std::invalid_argument(msg);
    case CASCADE_ENOBASE: throw MissingBaselineError{};
    default: throw DeviceError(msg);
    }
}

struct VerifyResult {
    CostBreakdown cost;          // ns, device-measured (draft_time from the host)
    int accepted = 0;            // 0..K
    std::vector<int32_t> emitted;  // accepted drafts + bonus token
    cascade_verify_out raw{};
};

class Verifier {
public:
    explicit Verifier(cascade_session* s) : s_(s) {}

    void prefill(const std::vector<int32_t>& prompt) {
        check_status(cascade_prefill(s_, prompt.data(), static_cast<int>(prompt.size())));
    }

    void set_baseline(double t_base_ns) { check_status(cascade_set_baseline(s_, t_base_ns)); }

    VerifyResult verify(const std::vector<int32_t>& drafts, double draft_ns) {
        VerifyResult r;
        check_status(cascade_verify(s_, drafts.empty() ? nullptr : drafts.data(), static_cast<int>(drafts.size()),
                                    draft_ns, &r.raw));
        r.cost.attention_time = r.raw.attention_time;
        r.cost.expert_time = r.raw.expert_time;
        r.cost.draft_time = r.raw.draft_time;
        r.cost.sampling_time = r.raw.sampling_time;
        r.cost.active_experts_per_layer = r.raw.active_experts_per_layer;
        r.cost.total = r.raw.total;
        r.accepted = r.raw.accepted;
        r.emitted.assign(r.raw.tokens, r.raw.tokens + r.raw.emitted);
        return r;
    }

    // Drops the KV cache (the next prefill starts a new request).
    void reset() { check_status(cascade_session_reset(s_)); }

    void set_batch_invariant(bool on) { check_status(cascade_set_batch_invariant(s_, on ? 1 : 0)); }

    int vocab() const {
        cascade_geometry g{};
        check_status(cascade_session_geometry(s_, &g));
        return g.vocab;
    }

    cascade_session* session() const { return s_; }

private:
    cascade_session* s_;
};

// Prompt-lookup drafter: find the most recent earlier
// occurrence of the longest suffix n-gram (n = max_n .. 1) and propose the
// tokens that followed it, at most k.  Fewer than k proposals (or none)
// shrink the step; the acceptance is still a causal prefix.
class NgramDrafter {
public:
    explicit NgramDrafter(int max_n = 3) : max_n_(max_n < 1 ? 1 : max_n) {}

    std::vector<int32_t> propose(const std::vector<int32_t>& ctx, int k) const {
        std::vector<int32_t> out;
        const long len = static_cast<long>(ctx.size());
        if (k <= 0 || len < 2) return out;
        for (int n = static_cast<int>(std::min<long>(max_n_, len - 1)); n >= 1; --n) {
            const long tail = len - n;
            for (long start = tail - 1; start >= 0; --start) {
                bool match = true;
                for (int i = 0; i < n && match; ++i) match = ctx[start + i] == ctx[tail + i];
                if (!match) continue;
                for (long j = start + n; j < len && static_cast<int>(out.size()) < k; ++j) out.push_back(ctx[j]);
                return out;
            }
        }
        return out;
    }

private:
    int max_n_;
};

// Replay drafter: proposes the target model's own greedy continuation
// (recorded by a K=0 run), each proposal independently corrupted with
// probability 1 - p.  The accepted prefix then follows the reference's
// acceptance model exactly (i.i.d. Bernoulli(p) until the first rejection,
// workload.hpp:80-86), but measured through the real verifier, so the
// utility controller sees real device costs at a controlled acceptance rate.
class ReplayDrafter {
public:
    ReplayDrafter(std::vector<int32_t> truth, int n_prompt, double p, int vocab, uint64_t seed)
        : truth_(std::move(truth)), n_prompt_(n_prompt), p_(p), vocab_(vocab), rng_(seed) {
        if (p < 0.0 || p > 1.0) throw std::invalid_argument("ReplayDrafter: p must be in [0,1]");
        if (vocab < 2) throw std::invalid_argument("ReplayDrafter: vocab must be >= 2");
    }

    std::vector<int32_t> propose(const std::vector<int32_t>& ctx, int k) {
        std::vector<int32_t> out;
        const long pos = static_cast<long>(ctx.size()) - n_prompt_;
        std::uniform_real_distribution<double> u(0.0, 1.0);
        for (int i = 0; i < k; ++i) {
            const long j = pos + i;
            if (j < 0 || j >= static_cast<long>(truth_.size())) break;
            int32_t t = truth_[j];
            if (u(rng_) >= p_) t = static_cast<int32_t>((t + 1) % vocab_);
            out.push_back(t);
        }
        return out;
    }

private:
    std::vector<int32_t> truth_;
    int n_prompt_;
    double p_;
    int vocab_;
    Rng rng_;
};

struct GpuRunOptions {
    EngineOptions engine;
    int k_limit = 8;                       // verifier K cap (session k_max)
    int baseline_probes = 4;               // K=0 steps that measure t_base for static/none policies
    std::optional<std::array<double, CASCADE_MAX_TOKENS>> injected_cost;  // k -> total_time
    std::vector<TraceRecord>* trace = nullptr;  // records (trace_request_id, iter, k_offered, accepted)
    long trace_request_id = 0;
};

// The reference request loop (engine.hpp:115-182) over the real verifier.
// `tokens` holds the prompt and receives the generated tokens.
template <typename Drafter>
inline RequestMetrics run_request(Verifier& verifier, Drafter& drafter, const Policy& policy,
                                  std::vector<int32_t>& tokens, int output_len, const GpuRunOptions& opt = {}) {
    if (tokens.empty()) throw std::invalid_argument("run_request: empty prompt");
    if (output_len < 1) throw std::invalid_argument("run_request: output_len must be >= 1");
    verifier.prefill(tokens);

    UtilityAnalyzer analyzer(16);
    std::optional<SpeculationController> ctl;
    if (policy.kind == Policy::Kind::adaptive) ctl.emplace(policy.controller);

    std::vector<IterationRecord> telemetry;
    long emitted = 0;
    long iter = 0;
    std::vector<double> probe_times;
    using clock = std::chrono::steady_clock;
    while (emitted < output_len) {
        detail::Decision d = detail::decide(policy, ctl);
        const bool probing = !ctl && iter < opt.baseline_probes;  // static/none: measure t_base first
        if (probing) d = {0, PhaseTag::baseline_probe, 0};
        d.k = std::min(d.k, opt.k_limit);

        const auto t0 = clock::now();
        const std::vector<int32_t> drafts = drafter.propose(tokens, d.k);
        const double draft_ns = std::chrono::duration<double, std::nano>(clock::now() - t0).count();

        VerifyResult v = verifier.verify(drafts, policy.kind == Policy::Kind::none ? 0.0 : draft_ns);
        CostBreakdown cost = v.cost;
        if (opt.injected_cost) {
            // K-trace parity mode: deterministic k -> time, real acceptance
            cost = CostBreakdown{};
            cost.total = (*opt.injected_cost)[static_cast<std::size_t>(d.k)];
            cost.expert_time = cost.total;
        }
        const IterationRecord rec = detail::make_record(iter, d, v.accepted, cost);
        if (opt.trace) opt.trace->push_back({opt.trace_request_id, iter, static_cast<int>(drafts.size()), v.accepted});

        if (ctl) {
            ctl->next_k(rec, analyzer);
            if (analyzer.baseline().valid()) verifier.set_baseline(analyzer.baseline().t_base);
        } else {
            analyzer.record(rec);
            if (probing) {
                probe_times.push_back(rec.total_time);
                if (static_cast<int>(probe_times.size()) == opt.baseline_probes) {
                    analyzer.refresh_from_pending();
                    verifier.set_baseline(analyzer.baseline().t_base);
                }
            }
        }
        if (opt.engine.keep_telemetry) telemetry.push_back(rec);
        tokens.insert(tokens.end(), v.emitted.begin(), v.emitted.end());
        emitted += rec.tokens_emitted;
        ++iter;
    }
    if (!analyzer.baseline().valid()) {
        if (analyzer.pending_probe_count() > 0) analyzer.refresh_from_pending();
        else throw MissingBaselineError{};
    }
    return detail::finalize_metrics(analyzer, std::move(telemetry));
}

// Replay drafter driven by a reference WorkloadProfile: the keep
// probability of each iteration's proposals is the current phase's
// per_token_accept_prob, and the phase walker advances once per iteration,
// exactly as the reference request loop does with ProfileState
// (engine.hpp:122,159,176).
class ProfileReplayDrafter {
public:
    ProfileReplayDrafter(std::vector<int32_t> truth, int n_prompt, const WorkloadProfile& profile, int vocab,
                         uint64_t seed)
        : truth_(std::move(truth)), n_prompt_(n_prompt), vocab_(vocab), rng_(seed), state_(profile, rng_) {
        if (vocab < 2) throw std::invalid_argument("ProfileReplayDrafter: vocab must be >= 2");
    }

    std::vector<int32_t> propose(const std::vector<int32_t>& ctx, int k) {
        std::vector<int32_t> out;
        const double p = state_.phase().per_token_accept_prob;
        const long pos = static_cast<long>(ctx.size()) - n_prompt_;
        std::uniform_real_distribution<double> u(0.0, 1.0);
        for (int i = 0; i < k; ++i) {
            const long j = pos + i;
            if (j < 0 || j >= static_cast<long>(truth_.size())) break;
            int32_t t = truth_[j];
            if (u(rng_) >= p) t = static_cast<int32_t>((t + 1) % vocab_);
            out.push_back(t);
        }
        state_.advance(rng_);
        return out;
    }

private:
    std::vector<int32_t> truth_;
    int n_prompt_;
    int vocab_;
    Rng rng_;
    ProfileState state_;
};

// K=0 stand-in drafter (proposes nothing).
struct NoDrafter {
    std::vector<int32_t> propose(const std::vector<int32_t>&, int) const { return {}; }
};

// The target's greedy continuation of `prompt` (n tokens, K=0 steps).  When
// `t_base` is given it receives the mean device time of the first `probes`
// of those K=0 steps: the no-speculation baseline of this request.
inline std::vector<int32_t> greedy_continuation(Verifier& verifier, const std::vector<int32_t>& prompt, long n,
                                                double* t_base = nullptr, int probes = 4) {
    verifier.reset();
    verifier.prefill(prompt);
    std::vector<int32_t> out;
    out.reserve(static_cast<std::size_t>(n));
    double sum = 0.0;
    int cnt = 0;
    for (long i = 0; i < n; ++i) {
        const VerifyResult r = verifier.verify({}, 0.0);
        if (cnt < probes) {
            sum += r.cost.total;
            ++cnt;
        }
        out.push_back(r.emitted.at(0));
    }
    if (t_base) *t_base = cnt ? sum / cnt : 0.0;
    verifier.reset();
    return out;
}

// One cell of the reference scenario sweep (engine.hpp run_cell, 339-376) on
// the device: the task's request stream (profile mix, output lengths, token
// budget) is drawn from the workload seed `wseed` exactly as the reference
// draws it, every request gets a random prompt, its greedy continuation is
// recorded with K=0 steps, and the request is then decoded under the
// policy with the profile-driven replay drafter.  Costs are the device's;
// the aggregation is the reference's (tpot, ETR, cost, utility, harmonic
// mean).  The session is made batch-invariant so replayed drafts stay
// aligned with the recorded continuation.
inline CellResult run_cell_seeded(Verifier& verifier, int vocab, const RequestStream& task, const Policy& policy,
                                  long tokens_per_cell, int prompt_len, std::uint64_t wseed,
                                  const GpuRunOptions& opt = {}) {
    if (prompt_len < 1) throw std::invalid_argument("run_cell: prompt_len must be >= 1");
    verifier.set_batch_invariant(true);
    CellResult cell;
    cell.policy = policy.label();
    Rng stream_rng(wseed);
    RequestStream stream = task;
    stream.max_tokens = tokens_per_cell;
    StreamSampler sampler(stream);
    std::vector<double> utils;
    double t_base_sum = 0.0;
    while (!sampler.exhausted()) {
        const auto [profile, len] = sampler.next_request(stream_rng);
        Rng prng(splitmix64(wseed + 0x9E3779B97F4A7C15ull * static_cast<std::uint64_t>(cell.requests + 1)));
        std::vector<int32_t> prompt(static_cast<std::size_t>(prompt_len));
        std::uniform_int_distribution<int32_t> tok(0, vocab - 1);
        for (int32_t& t : prompt) t = tok(prng);
        std::vector<int32_t> truth = greedy_continuation(verifier, prompt, len + CASCADE_MAX_TOKENS);
        ProfileReplayDrafter drafter(std::move(truth), prompt_len, *profile, vocab, prng());
        std::vector<int32_t> toks = prompt;
        verifier.reset();
        RequestMetrics m = run_request(verifier, drafter, policy, toks, len, opt);
        ++cell.requests;
        cell.iterations += m.iterations;
        cell.tokens += m.tokens;
        cell.total_time += m.total_time;
        t_base_sum += m.t_base;
        utils.push_back(m.utility);
    }
    cell.t_base = t_base_sum / static_cast<double>(cell.requests);
    cell.tpot = cell.total_time / static_cast<double>(cell.tokens);
    cell.etr = static_cast<double>(cell.tokens) / static_cast<double>(cell.iterations);
    cell.cost = (cell.total_time / static_cast<double>(cell.iterations)) / cell.t_base;
    cell.utility = cell.etr / cell.cost;
    cell.utility_hmean = harmonic_mean(utils);
    return cell;
}

inline CellResult run_cell(Verifier& verifier, int vocab, const RequestStream& task, const Policy& policy,
                           long tokens_per_cell, int prompt_len, uint64_t seed, const GpuRunOptions& opt = {}) {
    return run_cell_seeded(verifier, vocab, task, policy, tokens_per_cell, prompt_len, splitmix64(seed), opt);
}

// The reference sweep (engine.hpp run_scenario, 418-466) over verifier-backed
// cells.  The reference's cell thread pool (427-459) becomes one worker per
// verifier session: sessions live on different GPUs (one per device, each
// with its own weights), so cells run device-parallel; every worker pulls
// the next cell index from a shared cursor and a failing cell is recorded
// without stopping the sweep.  The models axis is the loaded device model
// (`model_name`); tasks x policies are crossed as in the reference, with the
// reference's policy-independent workload seeds (engine.hpp:355-357), so
// every policy of a task faces the same requests.
inline ScenarioReport run_scenario(const std::vector<Verifier*>& devices, const ScenarioConfig& cfg,
                                   const std::string& model_name, int prompt_len, const GpuRunOptions& opt = {}) {
    if (devices.empty()) throw std::invalid_argument("run_scenario: need at least one verifier session");
    if (cfg.tasks.empty() || cfg.policies.empty())
        throw std::invalid_argument("scenario needs at least one model, task, and policy");
    for (const TaskSpec& t : cfg.tasks) t.stream.validate();
    if (cfg.tokens_per_cell < 1) throw std::invalid_argument("tokens_per_cell must be >= 1");
    ScenarioReport rep;
    rep.name = cfg.name;
    rep.seed = cfg.seed;
    const std::size_t np = cfg.policies.size(), nt = cfg.tasks.size(), n = nt * np;
    rep.cells.resize(n);
    std::vector<int> vocab(devices.size());
    for (std::size_t i = 0; i < devices.size(); ++i) vocab[i] = devices[i]->vocab();
    std::atomic<std::size_t> cursor{0};
    auto work = [&](std::size_t dev) {
        for (std::size_t idx; (idx = cursor.fetch_add(1)) < n;) {
            const std::size_t pi = idx % np, ti = idx / np;
            CellResult& c = rep.cells[idx];
            try {
                const std::uint64_t wseed = splitmix64(cfg.seed ^ splitmix64(1 * 0x10001ull + (ti + 1) * 0x101ull));
                c = run_cell_seeded(*devices[dev], vocab[dev], cfg.tasks[ti].stream, cfg.policies[pi],
                                    cfg.tokens_per_cell, prompt_len, wseed, opt);
            } catch (const std::exception& e) {
                c = CellResult{};
                c.failed = true;
                c.error = e.what();
            }
            c.model_idx = 0;
            c.task_idx = ti;
            c.policy_idx = pi;
            c.model = model_name;
            c.task = cfg.tasks[ti].name;
            c.policy = cfg.policies[pi].label();
        }
    };
    if (devices.size() == 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (std::size_t d = 0; d < devices.size(); ++d) pool.emplace_back(work, d);
        for (std::thread& t : pool) t.join();
    }
    for (const Policy& p : cfg.policies)
        if (p.kind == Policy::Kind::none) {
            // a failed device cell is a runtime failure, not a missing
            // baseline policy: name it instead of the reference's message
            for (const CellResult& c : rep.cells)
                if (c.failed && c.policy == "none")
                    throw std::runtime_error("run_scenario: baseline cell " + c.task + "/none failed: " + c.error);
            compare_policies(rep);
            break;
        }
    return rep;
}

// Replays a recorded request on the device: the reference's replay loop
// (engine.hpp replay_request, 194-248) with the priced step (227) swapped for
// a real verification step.  The request spans exactly its recorded
// iterations; each iteration's acceptance is the recorded one truncated to
// the offered k (trace.hpp:69-74), and the costs are measured.  The drafts
// force that acceptance on the real model: the first a = min(recorded, k)
// drafts are the target's own greedy continuation and the next one is a
// token the target does not pick, so the device's greedy check accepts
// exactly a (the session is batch-invariant, so the continuation recorded
// at K=0 is what every wider step computes).  Static and none policies run
// the offered k on every recorded iteration, as the reference does; their
// baseline is measured on the same request's K=0 continuation steps (the
// reference takes an analytic one, engine.hpp:212).  `mismatches` counts
// iterations where the device accepted something else (0 unless the model
// or numerics changed under the trace).
inline RequestMetrics replay_request(Verifier& verifier, const AcceptanceTrace& trace, long request_id,
                                     const Policy& policy, const std::vector<int32_t>& prompt,
                                     const GpuRunOptions& opt = {}, long* mismatches = nullptr) {
    if (prompt.empty()) throw std::invalid_argument("replay_request: empty prompt");
    const std::vector<const TraceRecord*> recorded = trace.iterations_of(request_id);
    if (recorded.empty()) throw MissingRecordError(request_id, 0);
    const int vocab = verifier.vocab();
    verifier.set_batch_invariant(true);
    long need = CASCADE_MAX_TOKENS;
    for (const TraceRecord* r : recorded) need += r->accepted + 1;
    double t_base = 0.0;
    const std::vector<int32_t> truth = greedy_continuation(verifier, prompt, need, &t_base, opt.baseline_probes);
    verifier.prefill(prompt);

    UtilityAnalyzer analyzer(16);
    std::optional<SpeculationController> ctl;
    if (policy.kind == Policy::Kind::adaptive) {
        ctl.emplace(policy.controller);
    } else {
        analyzer.set_baseline(t_base);
        verifier.set_baseline(t_base);
    }
    std::vector<IterationRecord> telemetry;
    long pos = 0, iter = 0, bad = 0;
    using clock = std::chrono::steady_clock;
    for (const TraceRecord* src : recorded) {
        detail::Decision d = detail::decide(policy, ctl);
        d.k = std::min(d.k, opt.k_limit);
        const int want = std::min(src->accepted, d.k);
        const auto t0 = clock::now();
        std::vector<int32_t> drafts(truth.begin() + pos, truth.begin() + pos + d.k);
        if (want < d.k) drafts[static_cast<std::size_t>(want)] = (drafts[static_cast<std::size_t>(want)] + 1) % vocab;
        const double draft_ns = std::chrono::duration<double, std::nano>(clock::now() - t0).count();
        const VerifyResult v = verifier.verify(drafts, policy.kind == Policy::Kind::none ? 0.0 : draft_ns);
        if (v.accepted != want) ++bad;
        CostBreakdown cost = v.cost;
        if (opt.injected_cost) {
            cost = CostBreakdown{};
            cost.total = (*opt.injected_cost)[static_cast<std::size_t>(d.k)];
            cost.expert_time = cost.total;
        }
        const IterationRecord rec = detail::make_record(iter, d, v.accepted, cost);
        if (opt.trace) opt.trace->push_back({request_id, iter, static_cast<int>(drafts.size()), v.accepted});
        if (ctl) {
            ctl->next_k(rec, analyzer);
            if (analyzer.baseline().valid()) verifier.set_baseline(analyzer.baseline().t_base);
        } else {
            analyzer.record(rec);
        }
        if (opt.engine.keep_telemetry) telemetry.push_back(rec);
        pos += v.accepted + 1;
        if (pos + CASCADE_MAX_TOKENS > static_cast<long>(truth.size())) break;  // device diverged past the record
        ++iter;
    }
    if (mismatches) *mismatches = bad;
    if (!analyzer.baseline().valid()) {
        if (analyzer.pending_probe_count() > 0) analyzer.refresh_from_pending();
        else throw MissingBaselineError{};
    }
    return detail::finalize_metrics(analyzer, std::move(telemetry));
}

}  // namespace specsim
