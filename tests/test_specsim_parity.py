"""Host-side parity of this repository's specsim headers (include/specsim)
with the reference's (CPU only).

* every scenario of tests/golden/make_golden.py is replayed against our
  headers and must reproduce the committed reference outputs bit for bit
  (expected_unique_experts, sample_active_experts / iteration_cost RNG
  streams, sample_accepted, trace truncation, controller K-decision traces
  under the injected-cost harness, run_request metrics, window utility,
  controller replay of recorded iterations);
* when the reference build is present (this container), a fresh randomized
  set of controller landscapes is compared live as well.
"""

import json
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(HERE, "golden"))

import specsim_shim as sh  # noqa: E402
from make_golden import scenarios, unimodal  # noqa: E402

GOLDEN = json.load(open(os.path.join(HERE, "golden", "specsim_reference.json")))


@pytest.fixture(scope="module")
def ours():
    if not sh.available("ours"):
        import subprocess

        subprocess.check_call(["make", "-s", "-C", os.path.join(sh.ROOT, "oracle"), "libspecsim_ours.so"])
    return sh.Shim("ours")


SCEN = scenarios()


@pytest.mark.parametrize("idx", range(len(SCEN)), ids=[n for n, _ in SCEN])
def test_matches_reference_golden(ours, idx):
    name, fn = SCEN[idx]
    got = json.loads(json.dumps(fn(ours)))
    assert got == GOLDEN[name]


def test_golden_covers_the_appendix_traces():
    """SURVEY.md Appendix A, measured from the reference harness."""
    a1 = GOLDEN["drive/appendixA-1"]
    assert a1["test_iters"] == 12 and a1["sets"][0] == [2, 16]
    assert abs(a1["total_time"] - 24.854701) < 1e-6
    flat = GOLDEN["drive/flat-0.5"]
    assert flat["test_iters"] == 24 and flat["total_time"] == 424.0
    rising = GOLDEN["drive/rising"]
    assert rising["test_iters"] == 60 and abs(rising["total_time"] - 204.0) < 1e-9


@pytest.mark.skipif(not sh.available("ref"), reason="reference build not present")
def test_live_random_landscapes_match_reference(ours):
    ref = sh.Shim("ref")
    rng = np.random.default_rng(int.from_bytes(os.urandom(4), "little"))
    for _ in range(40):
        k_max = int(rng.integers(1, 8))
        peak = int(rng.integers(1, k_max + 1))
        u = unimodal(k_max, peak, (1.02 + rng.random(7)).tolist(), float(0.5 + rng.random()))
        c = sh.cfg(k_max=k_max, k_start=int(rng.integers(1, k_max + 1)), t_trial=int(rng.integers(1, 6)),
                   max_trials=int(rng.integers(1, 6)), band=float(0.02 + 0.3 * rng.random()),
                   backoff=int(rng.integers(0, 2)))
        c["s_set"] = max(c["t_trial"], int(rng.integers(4, 32)))
        c["s_cap"] = c["s_set"] * int(rng.integers(1, 16))
        noise = float(rng.choice([0.0, 0.03, 0.1]))
        seed = int(rng.integers(0, 2**31))
        a = ours.drive(c, u, 600, 0, noise, seed)
        b = ref.drive(c, u, 600, 0, noise, seed)
        assert a == b, (c, u, noise, seed)


@pytest.mark.skipif(not sh.available("ref"), reason="reference build not present")
def test_live_cost_and_acceptance_streams_match_reference(ours):
    ref = sh.Shim("ref")
    for seed in (3, 99, 12345):
        for preset in ("mixtral", "olmoe", "qwen15", "deepseekv1"):
            for k in (0, 3, 8, 12):
                assert np.array_equal(ours.iteration_cost(preset, "eagle", k, seed, 16),
                                      ref.iteration_cost(preset, "eagle", k, seed, 16))
        assert np.array_equal(ours.sample_accepted(0.63, 7, seed, 500), ref.sample_accepted(0.63, 7, seed, 500))
