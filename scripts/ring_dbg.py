import numpy as np, sys, os
sys.path.insert(0, os.getcwd())
import paper_2506_20675_b200 as cb
shape = cb.preset(sys.argv[1] if len(sys.argv) > 1 else "mixtral").with_layers(1)
m = cb.Model(shape, 5)
s = cb.Session(m, max_ctx=256, k_max=8)
T = int(sys.argv[2]) if len(sys.argv) > 2 else 16
s.prefill(np.random.default_rng(5).integers(0, shape.vocab, T + 1).astype(np.int32))
print("prefill ok")
o = s.verify(np.random.default_rng(6).integers(0, shape.vocab, 8).astype(np.int32))
print("verify ok", o.accepted)
