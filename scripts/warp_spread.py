"""Per-warp end of the gate/up and down ranges in the fused expert FFN
(CTAs 0 and 1, warp_stamp records), relative to the launch's first CTA
start: the intra-CTA spread the piece-level reduction waits for.
usage: python scripts/warp_spread.py [config] [K,K,...]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_20675_b200 as cb  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
ks = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,8").split(",")]
shape = cb.preset(cfg)
m = cb.Model(shape, 1)
s = cb.Session(m, max_ctx=1088, k_max=max(ks))
rng = np.random.default_rng(1)
s.prefill(rng.integers(0, shape.vocab, 1025).astype(np.int32))
for K in ks:
    for _ in range(3):
        s.enqueue(K)
    s.sync()
    tr, kind = s.cta_trace(K)
    gu, dn = [], []
    for i in range(len(tr)):
        if cb.KERNEL_CLASSES[kind[i]] != "expert_gate_up":
            continue
        st = tr[i, :496, 0].astype(np.float64)
        t0 = st[st > 0].min()
        ph = tr[i, 496:, :].reshape(-1).astype(np.float64)
        w = ph[16:48].reshape(2, 8, 2)  # [cta][warp][gate/up, down]
        gu.append(np.where(w[..., 0] > 0, (w[..., 0] - t0) / 1e3, np.nan))
        dn.append(np.where(w[..., 1] > 0, (w[..., 1] - t0) / 1e3, np.nan))
    gu, dn = np.array(gu[1:]), np.array(dn[1:])
    print(f"== {cfg} K={K}: fused FFN, per-warp range end (us from launch start), mean over {len(gu)} layers")
    for c in range(2):
        print(f"  CTA {c} gate/up: " + " ".join(f"{x:7.2f}" for x in np.nanmean(gu[:, c], 0)) +
              f" | spread {np.nanmean(np.nanmax(gu[:, c], 1) - np.nanmin(gu[:, c], 1)):.2f}")
        print(f"  CTA {c} down:    " + " ".join(f"{x:7.2f}" for x in np.nanmean(dn[:, c], 0)) +
              f" | spread {np.nanmean(np.nanmax(dn[:, c], 1) - np.nanmin(dn[:, c], 1)):.2f}")
s.close()
m.close()
