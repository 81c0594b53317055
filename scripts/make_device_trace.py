"""Records an acceptance trace and IterationRecord telemetry on the B200
(cascade_decode, tiny model, utility controller, n-gram drafter) in the
reference's file formats, for the CPU interop test
(tests/test_interop_cpu.py::test_device_recorded_trace_replays_in_the_reference).

    python scripts/make_device_trace.py gpurun_out/golden
then copy the two files into tests/golden/.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_20675_b200 as cb  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/golden"
os.makedirs(out, exist_ok=True)
shape = cb.preset("tiny")
m = cb.Model(shape, cb.TINY_SEED)
s = cb.Session(m, max_ctx=1024, k_max=15)
trace = os.path.join(out, "device_trace_tiny.trace")
for rid, seed in enumerate((1, 2, 3)):
    rng = np.random.default_rng(seed)
    motif = rng.integers(0, shape.vocab, 9)
    prompt = np.concatenate([np.tile(motif, 7)[:57], rng.integers(0, shape.vocab, 7)]).astype(np.int32)
    cfg = cb.decode_cfg(policy=-1, max_new=200, ngram_n=3, k_max=5)
    toks, tel, n = s.decode(prompt, cfg, telemetry_cap=4096,
                            telemetry_csv=os.path.join(out, "device_telemetry_tiny.csv") if rid == 0 else None,
                            trace_path=trace, request_id=rid, trace_append=rid > 0)
    print(f"request {rid}: {len(toks)} tokens in {n} iterations, accepted {int(tel[:, 2].sum() - n)}")
s.close()
m.close()
