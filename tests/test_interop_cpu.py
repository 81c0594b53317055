"""Telemetry / trace / scenario interoperability with the reference (§8 f3, f4).

Every check runs the same inputs through this repository's headers
(oracle/libspecsim_ours.so) and the UNMODIFIED reference headers
(oracle/_ref/libspecsim_ref.so) and requires identical results:

* the IterationRecord telemetry CSV is byte-identical (report.hpp:123-138);
* the reference's scenario fixtures parse to the same configuration
  (scenario.hpp:205-251), and the simulated sweep over them writes
  byte-identical cells.csv / summary.json (report.hpp:31-121);
* cells.csv written here is read by the reference's load_cells_csv
  (report.hpp:141-177);
* acceptance traces (trace.hpp:36,77-108): the reference fixture and the
  trace recorded on a B200 by cascade_decode (tests/golden/device_trace_tiny
  .trace, made by scripts/make_device_trace.py) load in the reference, and
  the reference's replay_request reproduces the recorded accepted counts.
"""

import csv
import json
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import specsim_shim as sh  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
FIX = os.path.join(HERE, "golden", "reference_fixtures")
DEVICE_TRACE = os.path.join(HERE, "golden", "device_trace_tiny.trace")
DEVICE_TELEMETRY = os.path.join(HERE, "golden", "device_telemetry_tiny.csv")

need_both = pytest.mark.skipif(not (sh.available("ref") and sh.available("ours")), reason="shim builds missing")


@pytest.fixture(scope="module")
def shims():
    return sh.Shim("ours"), sh.Shim("ref")


@need_both
def test_telemetry_csv_is_byte_identical(shims, tmp_path):
    ours, ref = shims
    rng = np.random.default_rng(3)
    n = 200
    rows = np.zeros((n, 9))
    rows[:, 0] = np.arange(n)
    rows[:, 1] = rng.integers(0, 8, n)
    rows[:, 2] = [rng.integers(1, k + 2) for k in rows[:, 1].astype(int)]
    rows[:, 3:7] = rng.random((n, 4)) * 1e6
    rows[:, 7] = rng.integers(0, 3, n)
    rows[:, 8] = rng.integers(0, 5, n)
    a, b = tmp_path / "ours.csv", tmp_path / "ref.csv"
    ours.write_telemetry(a, rows)
    ref.write_telemetry(b, rows)
    assert a.read_bytes() == b.read_bytes()
    assert a.read_text().splitlines()[0] == (
        "iter_index,k_used,tokens_emitted,draft_time,verify_time,sampling_time,total_time,phase_tag,trial_no")


SCENARIO_ROUNDTRIP = {
    "name": "t", "seed": 99,
    "models": ["mixtral", {"name": "tiny", "num_layers": 4, "experts_per_layer": 4, "top_k": 1, "affinity": 0.2,
                           "attention_fraction": 0.1}],
    "tasks": ["code", {"name": "bursty", "mix": [{"share": 1.0, "profile": {
        "name": "bursty", "phases": [{"accept_prob": 0.9, "mean_duration": 20.0},
                                     {"accept_prob": 0.1, "mean_duration": 30.0, "affinity": 0.8}],
        "output_len": [100, 200], "expert_affinity": 0.4}}]},
              {"name": "markov", "mix": [{"share": 0.5, "profile": {"preset": "extract", "transition": "markov",
                                                                     "transition_matrix": [[0.9, 0.1], [0.2, 0.8]]}},
                                         {"share": 0.5, "profile": "math"}]}],
    "policies": ["none", "static:1..2", "adaptive"],
    "draft": {"kind": "per_token_linear", "per_k_overhead": 0.05, "always_on_overhead": 0.02},
    "controller": {"k_max": 5, "k_start": 2, "backoff": False},
    "tokens_per_cell": 1234, "jobs": 2,
}


@need_both
def test_scenario_files_parse_identically(shims, tmp_path):
    ours, ref = shims
    custom = tmp_path / "custom.json"
    custom.write_text(json.dumps(SCENARIO_ROUNDTRIP))
    files = [os.path.join(FIX, f) for f in sorted(os.listdir(FIX)) if f.endswith(".json")] + [str(custom)]
    assert len(files) == 4
    for f in files:
        d_ours, d_ref = ours.scenario_digest(f), ref.scenario_digest(f)
        assert d_ref is not None and d_ours == d_ref, f
    bad = tmp_path / "bad.json"
    bad.write_text('{"models": ["mixtral"], "tasks": ["code"]}')  # policies missing
    assert ours.scenario_digest(bad) is None and ref.scenario_digest(bad) is None


@need_both
@pytest.mark.parametrize("fixture,tokens", [("mixtral_all3.json", 1500), ("dominance.json", 800)])
def test_simulated_sweep_reports_are_byte_identical(shims, tmp_path, fixture, tokens):
    ours, ref = shims
    a, b = tmp_path / "ours", tmp_path / "ref"
    a.mkdir()
    b.mkdir()
    ours.scenario_report(os.path.join(FIX, fixture), tokens, a)
    ref.scenario_report(os.path.join(FIX, fixture), tokens, b)
    assert (a / "cells.csv").read_bytes() == (b / "cells.csv").read_bytes()
    assert (a / "summary.json").read_bytes() == (b / "summary.json").read_bytes()
    # the reference's `report` reader consumes the cells.csv written here
    rows = ref.load_cells(a / "cells.csv")
    with open(a / "cells.csv") as fh:
        assert len(rows) == sum(1 for _ in csv.DictReader(fh))


@need_both
def test_reference_trace_fixture_loads_identically(shims):
    ours, ref = shims
    path = os.path.join(FIX, "example.trace")
    a, b = ours.trace_load(path), ref.trace_load(path)
    assert len(a) > 0 and np.array_equal(a, b)


@need_both
@pytest.mark.skipif(not os.path.exists(DEVICE_TRACE), reason="device trace fixture not generated")
def test_device_recorded_trace_replays_in_the_reference(shims):
    """The trace cascade_decode recorded on a B200 loads with the reference's
    AcceptanceTrace::load, agrees with the device telemetry written beside
    it, and the reference's replay_request at the recorded k reproduces every
    recorded accepted count (tokens_emitted = accepted + 1)."""
    ours, ref = shims
    recs = ref.trace_load(DEVICE_TRACE)
    assert len(recs) > 0 and np.array_equal(recs, ours.trace_load(DEVICE_TRACE))
    with open(DEVICE_TELEMETRY) as fh:
        tel = list(csv.DictReader(fh))
    ids = sorted(set(recs[:, 0].tolist()))
    first = recs[recs[:, 0] == ids[0]]
    assert len(first) == len(tel)
    for r, t in zip(first, tel):
        assert int(t["iter_index"]) == r[1]
        assert int(t["tokens_emitted"]) == r[3] + 1
        assert r[2] <= int(t["k_used"])
    for rid in ids:
        mine = recs[recs[:, 0] == rid]
        k = int(max(1, mine[:, 2].max()))
        if k > 7:
            continue  # the reference's static policy caps k at 7
        _, emitted = ref.trace_replay_request(DEVICE_TRACE, rid, k)
        assert np.array_equal(emitted, mine[:, 3] + 1), rid
