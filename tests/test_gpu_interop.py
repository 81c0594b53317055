"""Device-side telemetry, trace and scenario interop (§8 f3, f4) on a B200.

* cascade_decode writes the IterationRecord telemetry CSV (report.hpp:
  123-138) and the acceptance trace (trace.hpp:36,101-108) of real device
  decodes; the reference's AcceptanceTrace::load (oracle/_ref, the
  unmodified headers) reads the trace, its records agree with the
  telemetry, and the reference's replay_request at the recorded k
  reproduces every accepted count.
* cascade_replay_trace replays the reference's fixture trace
  (proj/fixtures/example.trace) on the device: the replay spans exactly the
  recorded iterations, the device accepts exactly min(recorded, k) every
  iteration (forced through the model's own greedy continuation), and the
  per-request tokens / iterations equal the reference replay's; costs are
  measured (Theorem 1 holds per request).
* cascade_run_scenario runs a reference-format scenario file over two
  worker sessions: cells.csv / summary.json are read by the reference's
  loader, `none` normalises speedups, and utility * TPOT == t_base per cell.
"""

import csv
import json
import os
import sys

import numpy as np
import pytest

import paper_2506_20675_b200 as cb

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import specsim_shim as sh  # noqa: E402

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
EXAMPLE_TRACE = os.path.join(HERE, "golden", "reference_fixtures", "example.trace")
TEL_HEADER = "iter_index,k_used,tokens_emitted,draft_time,verify_time,sampling_time,total_time,phase_tag,trial_no"
TAGS = {0: "probe", 1: "test", 2: "set"}


@pytest.fixture(scope="module")
def tiny():
    shape = cb.preset("tiny")
    m = cb.Model(shape, cb.TINY_SEED)
    s = cb.Session(m, max_ctx=1024, k_max=15)
    yield shape, m, s
    s.close()
    m.close()


@pytest.fixture(scope="module")
def ref():
    if not sh.available("ref"):
        pytest.skip("oracle/_ref build missing")
    return sh.Shim("ref")


def motif_prompt(shape, seed, n=64):
    rng = np.random.default_rng(seed)
    motif = rng.integers(0, shape.vocab, 9)
    return np.concatenate([np.tile(motif, n // 9 + 1)[:n - 7], rng.integers(0, shape.vocab, 7)]).astype(np.int32)


def test_decode_writes_reference_telemetry_and_trace(tiny, ref, tmp_path):
    shape, m, s = tiny
    tel_csv, trace = str(tmp_path / "tel.csv"), str(tmp_path / "req.trace")
    tels = []
    for rid in range(3):
        cfg = cb.decode_cfg(policy=-1, max_new=150, ngram_n=3, k_max=5)
        toks, tel, n = s.decode(motif_prompt(shape, rid + 1), cfg, telemetry_cap=4096,
                                telemetry_csv=tel_csv if rid == 0 else None, trace_path=trace, request_id=rid,
                                trace_append=rid > 0)
        assert n == len(tel)
        tels.append(tel)
    recs = ref.trace_load(trace)
    assert sorted(set(recs[:, 0].tolist())) == [0, 1, 2]
    for rid, tel in enumerate(tels):
        mine = recs[recs[:, 0] == rid]
        assert np.array_equal(mine[:, 1], np.arange(len(tel)))
        assert np.array_equal(mine[:, 2], tel[:, 9].astype(np.int64))          # k_offered
        assert np.array_equal(mine[:, 3], tel[:, 2].astype(np.int64) - 1)      # accepted
        assert (mine[:, 3] > 0).any()                                          # the drafter got accepted
        k = int(max(1, mine[:, 2].max()))
        _, emitted = ref.trace_replay_request(trace, rid, k)
        assert np.array_equal(emitted, mine[:, 3] + 1)
    lines = open(tel_csv).read().splitlines()
    assert lines[0] == TEL_HEADER
    rows = list(csv.reader(lines[1:]))
    tel = tels[0]
    assert len(rows) == len(tel)
    for r, t in zip(rows, tel):
        assert [int(r[0]), int(r[1]), int(r[2]), int(r[8])] == [int(t[0]), int(t[1]), int(t[2]), int(t[8])]
        assert np.allclose([float(x) for x in r[3:7]], t[3:7], rtol=1e-11, atol=0)
        assert r[7] == TAGS[int(t[7])]


@pytest.mark.parametrize("policy", [3, 1, -1])
def test_device_replay_of_reference_trace(tiny, ref, tmp_path, policy):
    shape, m, s = tiny
    out_csv = str(tmp_path / "replay.csv")
    r = cb.replay_trace(s, EXAMPLE_TRACE, policy=policy, prompt_len=24, seed=5, out_csv=out_csv, k_max=3)
    assert r["mismatches"] == 0
    recs = ref.trace_load(EXAMPLE_TRACE)
    ids = list(dict.fromkeys(recs[:, 0].tolist()))
    with open(out_csv) as fh:
        rows = list(csv.DictReader(fh))
    assert open(out_csv).readline().strip() == "request_id,iterations,tokens,total_time,t_base,tpot,etr,cost,utility"
    assert [int(x["request_id"]) for x in rows] == ids and r["requests"] == len(ids)
    for row in rows:
        rid = int(row["request_id"])
        mine = recs[recs[:, 0] == rid]
        assert int(row["iterations"]) == len(mine)
        if policy > 0:
            assert int(row["tokens"]) == int((np.minimum(mine[:, 3], policy) + 1).sum())
            ref_m, _ = ref.trace_replay_request(EXAMPLE_TRACE, rid, policy)
            assert (int(row["tokens"]), int(row["iterations"])) == (int(ref_m[0]), int(ref_m[1]))
        u, tpot, tb = float(row["utility"]), float(row["tpot"]), float(row["t_base"])
        assert abs(u * tpot - tb) <= 1e-9 * tb
    assert r["tokens"] == sum(int(x["tokens"]) for x in rows)


def test_device_scenario_sweep_two_sessions(tiny, ref, tmp_path):
    shape, m, s = tiny
    scen = {"name": "device", "seed": 7, "models": ["mixtral"], "tasks": ["code", "math+extract"],
            "policies": ["none", "static:2", "adaptive"], "controller": {"k_max": 4}, "tokens_per_cell": 150}
    path = tmp_path / "scenario.json"
    path.write_text(json.dumps(scen))
    workers = [cb.Session(m, max_ctx=1024, k_max=15) for _ in range(2)]
    out = tmp_path / "report"
    n = cb.run_scenario_device(workers, str(path), str(out), prompt_len=24, model_name="tiny")
    for w in workers:
        w.close()
    assert n == 6
    cells = ref.load_cells(str(out / "cells.csv"))
    assert len(cells) == 6 and (cells[:, 1] >= 150).all()
    with open(out / "cells.csv") as fh:
        rows = list(csv.DictReader(fh))
    assert [(r["task"], r["policy"]) for r in rows] == [(t, p) for t in ("code", "math+extract")
                                                        for p in ("none", "static:2", "adaptive")]
    for r in rows:
        assert r["failed"] == "0" and r["model"] == "tiny"
        assert abs(float(r["utility"]) * float(r["tpot"]) - float(r["t_base"])) <= 1e-9 * float(r["t_base"])
        if r["policy"] == "none":
            assert float(r["speedup"]) == 1.0 and float(r["etr"]) == 1.0
    summ = json.loads((out / "summary.json").read_text())
    assert summ["cells"] == 6 and summ["failed_cells"] == [] and summ["regression"]["points"] == 6
    # the request stream is the reference's (policy-independent seeds): every
    # policy of a task serves the same requests and tokens budget
    for t in ("code", "math+extract"):
        req = {r["requests"] for r in rows if r["task"] == t}
        assert len(req) == 1
