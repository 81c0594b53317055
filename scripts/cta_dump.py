"""Dumps the raw per-CTA (start, exit) stamps of one captured step
(cascade_step_cta_trace) to an .npz for offline analysis.
usage: python scripts/cta_dump.py config K out.npz [layers]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_20675_b200 as cb  # noqa: E402

cfg, K, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
shape = cb.preset(cfg)
if len(sys.argv) > 4:
    shape = shape.with_layers(int(sys.argv[4]))
m = cb.Model(shape, 1)
ctx = 1024
s = cb.Session(m, max_ctx=ctx + 64, k_max=max(K, 1))
s.prefill(np.random.default_rng(1).integers(0, shape.vocab, ctx + 1).astype(np.int32))
for _ in range(3):
    s.enqueue(K)
s.sync()
tr, kind = s.cta_trace(K)
np.savez_compressed(out, tr=tr, kind=kind, union=s.union_sizes())
print("saved", out, tr.shape)
