"""Profiling driver (run under ncu on the GPU box): builds the Mixtral-shape
model, prefills --ctx tokens, captures the step graphs, then replays
--reps steps for each K inside cudaProfilerStart/Stop so that
`ncu --profile-from-start off` sees only the verify-step kernels."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_20675_b200 as cb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mixtral")
ap.add_argument("--ctx", type=int, default=1024)
ap.add_argument("--ks", default="0,8")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--layers", type=int, default=0)
a = ap.parse_args()
shape = cb.preset(a.config)
if a.layers:
    shape = shape.with_layers(a.layers)
m = cb.Model(shape, 1)
s = cb.Session(m, max_ctx=a.ctx + 64, k_max=15)
s.prefill(np.random.default_rng(1).integers(0, shape.vocab, a.ctx + 1).astype(np.int32))
ks = [int(k) for k in a.ks.split(",")]
for K in ks:
    s.enqueue(K)
s.sync()
torch.cuda.cudart().cudaProfilerStart()
for K in ks:
    for _ in range(a.reps):
        s.enqueue(K)
    s.sync()
torch.cuda.cudart().cudaProfilerStop()
print("union sizes (last K):", list(s.union_sizes()))
