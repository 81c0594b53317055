"""Per-CTA phases of the fused expert FFN from a cta_dump .npz: gate/up end,
first down-phase readiness release, exit (us from the launch's first CTA
start), by CTA-index group.  usage: python scripts/ffn_phases.py dump.npz"""
import sys

import numpy as np

for f in sys.argv[1:]:
    d = np.load(f)
    tr, kind = d["tr"].astype(np.float64), d["kind"]
    idx = [i for i, k in enumerate(kind) if k == 6]
    print(f, "FFN launches", len(idx), "union", d["union"][:4])
    acc = {"gu_end": [], "first_ready": [], "exit": []}
    for i in idx[1:]:
        st = tr[i, :296, 0]
        t0 = st[st > 0].min()
        for j, n in ((2, "gu_end"), (3, "first_ready"), (1, "exit")):
            v = tr[i, :296, j]
            acc[n].append(np.where(v > 0, (v - t0) / 1e3, np.nan))
    for n, v in acc.items():
        a = np.nanmean(np.array(v), axis=0)
        g = np.array_split(np.arange(296), 8)
        print(f"  {n:12s} groups " + " ".join(f"{np.nanmedian(a[x]):6.2f}" for x in g) +
              f" | min {np.nanmin(a):6.2f} med {np.nanmedian(a):6.2f} max {np.nanmax(a):6.2f}")
