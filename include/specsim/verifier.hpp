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
    std::vector<TraceRecord>* trace = nullptr;  // records (0, iter, k_offered, accepted)
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
        if (opt.trace) opt.trace->push_back({0, iter, static_cast<int>(drafts.size()), v.accepted});

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

// One cell of the reference scenario sweep (engine.hpp run_cell / run_scenario,
// 300-466) on the device: the task's request stream (profile mix, output
// lengths, token budget) is drawn with the reference's policy-independent
// seeds, every request gets a random prompt, its greedy continuation is
// recorded with a K=0 decode, and the request is then decoded under the
// policy with the profile-driven replay drafter.  Costs are the device's;
// the aggregation is the reference's (tpot, ETR, cost, utility, harmonic mean).
// The session must be batch-invariant so replayed drafts stay aligned.
inline CellResult run_cell(Verifier& verifier, int vocab, const RequestStream& task, const Policy& policy,
                           long tokens_per_cell, int prompt_len, uint64_t seed, const GpuRunOptions& opt = {}) {
    if (prompt_len < 1) throw std::invalid_argument("run_cell: prompt_len must be >= 1");
    CellResult cell;
    cell.policy = policy.label();
    const std::uint64_t wseed = splitmix64(seed);
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
        std::vector<int32_t> truth_toks = prompt;
        NoDrafter none_drafter;
        check_status(cascade_session_reset(verifier.session()));
        run_request(verifier, none_drafter, Policy::none(), truth_toks, len + CASCADE_MAX_TOKENS, opt);
        std::vector<int32_t> truth(truth_toks.begin() + prompt_len, truth_toks.end());
        ProfileReplayDrafter drafter(std::move(truth), prompt_len, *profile, vocab, prng());
        std::vector<int32_t> toks = prompt;
        check_status(cascade_session_reset(verifier.session()));
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

}  // namespace specsim
