"""Per-CTA timeline of captured verify steps (diagnostic for the roofline gap).

For every launch of one graph replay it reads each CTA's start (after the
dependency wait) and exit %globaltimer stamps (cascade_step_cta_trace) and
reports, per kernel class (mean over layers):
  busy   = last CTA exit - first CTA start
  skew   = last CTA start - first CTA start
  tail   = last CTA exit - median CTA exit   (stragglers)
  gap    = next launch's first CTA start - this launch's last CTA exit
usage: python scripts/cta_timeline.py [config] [K,K,...] [tag]
"""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_20675_b200 as cb  # noqa: E402


def analyse(tr, kind):
    rows = []
    for i in range(len(tr)):
        st, en = tr[i, :496, 0].astype(np.float64), tr[i, :496, 1].astype(np.float64)
        ok = (st > 0) & (en > 0)
        if not ok.any():
            rows.append(None)
            continue
        st, en = st[ok], en[ok]
        rows.append({"kind": cb.KERNEL_CLASSES[kind[i]], "n": int(ok.sum()), "first": st.min(), "last_start": st.max(),
                     "med_end": float(np.median(en)), "last_end": en.max()})
    out = []
    for i, r in enumerate(rows):
        if r is None:
            continue
        nxt = next((x for x in rows[i + 1:] if x is not None), None)
        out.append({"kind": r["kind"], "n": r["n"], "busy": r["last_end"] - r["first"],
                    "skew": r["last_start"] - r["first"], "tail": r["last_end"] - r["med_end"],
                    "gap": (nxt["first"] - r["last_end"]) if nxt else 0.0})
    return out, rows


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
    ks = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,8").split(",")]
    tag = sys.argv[3] if len(sys.argv) > 3 else "r"
    shape = cb.preset(cfg)
    m = cb.Model(shape, 1)
    ctx = 1024
    s = cb.Session(m, max_ctx=ctx + 64, k_max=max(ks))
    rng = np.random.default_rng(1)
    s.prefill(rng.integers(0, shape.vocab, ctx + 1).astype(np.int32))
    report = {}
    for K in ks:
        for _ in range(3):
            s.enqueue(K)
        s.sync()
        tr, kind = s.cta_trace(K)
        per, rows = analyse(tr, kind)
        t0 = min(r["first"] for r in rows if r is not None)
        t1 = max(r["last_end"] for r in rows if r is not None)
        cls = {}
        for p in per:
            c = cls.setdefault(p["kind"], {"launches": 0, "busy": 0.0, "skew": 0.0, "tail": 0.0, "gap": 0.0, "n": 0})
            c["launches"] += 1
            for k in ("busy", "skew", "tail", "gap"):
                c[k] += p[k]
            c["n"] = p["n"]
        print(f"\n== {cfg} K={K}: step span {(t1 - t0) / 1e3:.1f} us, {len(per)} launches")
        print(f"{'class':16s} {'CTAs':>5s} {'busy':>8s} {'skew':>7s} {'tail':>7s} {'gap':>7s}  (us, mean per launch)")
        for k, c in cls.items():
            n = c["launches"]
            print(f"{k:16s} {c['n']:5d} {c['busy'] / n / 1e3:8.2f} {c['skew'] / n / 1e3:7.2f} "
                  f"{c['tail'] / n / 1e3:7.2f} {c['gap'] / n / 1e3:7.2f}")
        # CTA-0 phase stamps (records 496..): mean delta of each phase from the CTA start
        ph = {}
        for i in range(len(tr)):
            k = cb.KERNEL_CLASSES[kind[i]]
            stamps = tr[i, 496:, :].reshape(-1).astype(np.float64)
            if not (stamps > 0).any() or tr[i, 0, 0] == 0:
                continue
            rel = [(x - tr[i, 0, 0]) / 1e3 if x > 0 else np.nan for x in stamps[:12]]
            rel.append((tr[i, 0, 1] - tr[i, 0, 0]) / 1e3)
            ph.setdefault(k, []).append(rel)
        for k, v in ph.items():
            a = np.nanmean(np.array(v, dtype=np.float64), axis=0)
            print(f"  phases {k}: " + " ".join("-" if np.isnan(x) else f"{x:.2f}" for x in a[:-1]) + f" | exit {a[-1]:.2f}")
        tot_busy = sum(p["busy"] for p in per) / 1e3
        tot_gap = sum(p["gap"] for p in per) / 1e3
        print(f"sum busy {tot_busy:.1f} us, sum gaps {tot_gap:.1f} us")
        # per-CTA exit spread of the layer-1 GEMVs (relative to the launch's first start)
        detail = {}
        for i in range(len(tr)):
            k = cb.KERNEL_CLASSES[kind[i]]
            if k in ("qkv", "o_proj", "expert_gate_up", "expert_down") and k not in detail and i > 12:
                st, en = tr[i, :, 0].astype(np.float64), tr[i, :, 1].astype(np.float64)
                ok = (st > 0) & (en > 0)
                f = st[ok].min()
                detail[k] = {"start_us": np.round((st[ok] - f) / 1e3, 2).tolist(),
                             "end_us": np.round((en[ok] - f) / 1e3, 2).tolist()}
                e = np.sort((en[ok] - f) / 1e3)
                print(f"  {k}: CTA exit quantiles (us from first start) p0 {e[0]:.2f} p10 {e[len(e) // 10]:.2f} "
                      f"p50 {e[len(e) // 2]:.2f} p90 {e[9 * len(e) // 10]:.2f} p100 {e[-1]:.2f}")
        report[K] = {"classes": {k: {kk: (vv / c["launches"] / 1e3 if kk in ("busy", "skew", "tail", "gap") else vv)
                                     for kk, vv in c.items()} for k, c in cls.items()},
                     "span_us": (t1 - t0) / 1e3, "detail": detail}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(report, open(os.path.join(ROOT, "gpurun_out", f"cta_timeline_{cfg}_{tag}.json"), "w"))
    s.close()
    m.close()


if __name__ == "__main__":
    main()
