// CPU unit test of the host-side drafters in include/specsim/verifier.hpp
// (no GPU: only header-inline classes that do not call the C ABI).
#include <cassert>
#include <cmath>
#include <cstdio>
#include <vector>

#include "specsim/verifier.hpp"

using namespace specsim;

static int accepted_prefix(const std::vector<int32_t>& drafts, const std::vector<int32_t>& truth, long pos) {
    int n = 0;
    while (n < (int)drafts.size() && drafts[n] == truth[pos + n]) ++n;
    return n;
}

int main() {
    std::vector<int32_t> truth(4096);
    for (size_t i = 0; i < truth.size(); ++i) truth[i] = (int32_t)((i * 7919) % 1000);
    const int n_prompt = 16;
    std::vector<int32_t> ctx(n_prompt, 5);
    // 1. keep probability 1 / 0
    {
        ReplayDrafter d1(truth, n_prompt, 1.0, 1000, 1);
        auto a = d1.propose(ctx, 6);
        assert(a.size() == 6);
        for (int i = 0; i < 6; ++i) assert(a[i] == truth[i]);
        ReplayDrafter d0(truth, n_prompt, 0.0, 1000, 1);
        auto b = d0.propose(ctx, 6);
        for (int i = 0; i < 6; ++i) assert(b[i] != truth[i]);
    }
    // 2. acceptance statistics follow the reference model: E[accepted] = sum_{j=1..K} p^j
    for (double p : {0.5, 0.8}) {
        ReplayDrafter d(truth, n_prompt, p, 1000, 7);
        const int K = 4, N = 200000;
        double sum = 0.0;
        std::vector<int32_t> c = ctx;
        for (int it = 0; it < N; ++it) {
            c.resize(n_prompt + (it % 3000));
            const long pos = (long)c.size() - n_prompt;
            sum += accepted_prefix(d.propose(c, K), truth, pos);
        }
        double expect = 0.0;
        for (int j = 1; j <= K; ++j) expect += std::pow(p, j);
        std::printf("p=%.1f mean accepted %.4f expected %.4f\n", p, sum / N, expect);
        assert(std::fabs(sum / N - expect) < 0.02);
    }
    // 3. profile-driven keep probability: cyclic phases p = 1 then 0, one iteration each
    {
        WorkloadProfile prof;
        prof.phases = {AcceptancePhase{1.0, 1.0, {}}, AcceptancePhase{0.0, 1.0, {}}};
        prof.transition = PhaseTransition::cyclic;
        ProfileReplayDrafter d(truth, n_prompt, prof, 1000, 3);
        for (int it = 0; it < 8; ++it) {
            auto a = d.propose(ctx, 3);
            const int acc = accepted_prefix(a, truth, 0);
            assert(acc == (it % 2 == 0 ? 3 : 0));
        }
    }
    // 4. n-gram prompt lookup proposes the continuation of the last match
    {
        NgramDrafter ng(3);
        std::vector<int32_t> c = {1, 2, 3, 4, 5, 9, 1, 2, 3};
        auto a = ng.propose(c, 3);
        assert((a == std::vector<int32_t>{4, 5, 9}));
    }
    std::printf("drafters ok\n");
    return 0;
}
