"""Small FFN driver for compute-sanitizer runs: one layer of a preset, a prefill
(T = 16: register engine) and verify steps at K = 0 and 4 (ring engine) and 8
(register engine).  usage: python scripts/ring_dbg.py [preset] [prompt_len]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_20675_b200 as cb  # noqa: E402

shape = cb.preset(sys.argv[1] if len(sys.argv) > 1 else "mixtral").with_layers(1)
m = cb.Model(shape, 5)
s = cb.Session(m, max_ctx=256, k_max=8)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
s.prefill(np.random.default_rng(5).integers(0, shape.vocab, n + 1).astype(np.int32))
print("prefill ok")
for K in (0, 4, 8):
    o = s.verify(np.random.default_rng(6 + K).integers(0, shape.vocab, K).astype(np.int32))
    print("verify ok K", K, "accepted", o.accepted)
