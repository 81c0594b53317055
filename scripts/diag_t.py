"""Diagnostic: GPU self-consistency across in-flight widths.  A K=0 decode
gives per-token taps; a K=3 verify of the same (accepted) tokens must give
the same per-layer residuals for every row."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_20675_b200 as cb

shape = cb.preset(sys.argv[1] if len(sys.argv) > 1 else "tiny")
m = cb.Model(shape, cb.TINY_SEED)
rng = np.random.default_rng(5)
prompt = rng.integers(0, shape.vocab, 24).astype(np.int32)
K = int(sys.argv[2]) if len(sys.argv) > 2 else 3
# K=0 reference: T+... steps one at a time with taps
a = cb.Session(m, max_ctx=256, k_max=8); a.enable_taps(True); a.prefill(prompt)
rows = []
toks = []
for i in range(K + 1):
    o = a.verify([])
    rows.append({k: a.tap(k)[:, 0].copy() for k in ("x_in", "x_mid", "moe_out", "xn_moe", "topk_id")} | {"logits": a.tap("final_logits")[0].copy()})
    toks.append(o.argmax[0])
b = cb.Session(m, max_ctx=256, k_max=8); b.enable_taps(True); b.prefill(prompt)
o = b.verify(np.array(toks[:K], np.int32))
print("K=0 tokens", toks, "K-step argmax", list(o.argmax[:K+1]), "accepted", o.accepted)
tb = {k: b.tap(k) for k in ("x_in", "x_mid", "moe_out", "xn_moe", "topk_id")}
lb = b.tap("final_logits")
for t in range(K + 1):
    for l in range(shape.num_layers):
        r = rows[t]
        def rel(x, y): return float(np.abs(x - y).max() / (np.abs(y).max() + 1e-30))
        print(f"t={t} l={l} x_in {rel(tb['x_in'][l,t], r['x_in'][l]):.2e} x_mid {rel(tb['x_mid'][l,t], r['x_mid'][l]):.2e} "
              f"moe {rel(tb['moe_out'][l,t], r['moe_out'][l]):.2e} topk {list(tb['topk_id'][l,t])} vs {list(r['topk_id'][l])}")
    print(f"t={t} logits rel {float(np.abs(lb[t]-rows[t]['logits']).max()):.3e}")
