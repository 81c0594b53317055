"""Diagnostic: per-SM streaming rate of the expert GEMV CTAs (from the per-CTA
timeline), used to test the SM-rate-weighted split (rejected)."""
import sys, os, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2506_20675_b200 as cb
shape = cb.preset('mixtral')
m = cb.Model(shape, 1)
s = cb.Session(m, max_ctx=1100, k_max=8)
s.prefill(np.random.default_rng(1).integers(0, shape.vocab, 1025).astype(np.int32))
res = {}
for K in (0, 8):
    for _ in range(3): s.enqueue(K)
    s.sync()
    durs = {}
    for rep in range(3):
        tr, kind = s.cta_trace(K)
        for i in range(len(tr)):
            k = cb.KERNEL_CLASSES[kind[i]]
            if k not in ('expert_gate_up', 'expert_down', 'qkv', 'o_proj'): continue
            st = tr[i, :496, 0].astype(np.int64); en = tr[i, :496, 1].astype(np.int64)
            ok = (st > 0) & (en > 0)
            sm = (st & 0xFF)[ok]; d = (en[ok] - (st[ok] & ~0xFF)) / 1e3
            d = d / np.median(d)
            for smid, dd in zip(sm, d):
                durs.setdefault(k, {}).setdefault(int(smid), []).append(dd)
    for k, per in durs.items():
        sms = sorted(per)
        means = np.array([np.mean(per[x]) for x in sms])
        # split-half consistency: even vs odd samples
        a = np.array([np.mean(per[x][0::2]) for x in sms]); b = np.array([np.mean(per[x][1::2]) for x in sms])
        order = np.argsort(means)
        print(f"K={K} {k}: SMs {len(sms)} rel-duration spread p5 {np.percentile(means,5):.3f} p95 {np.percentile(means,95):.3f} "
              f"split-half corr {np.corrcoef(a,b)[0,1]:.2f}; slowest SMs {[sms[j] for j in order[-10:]]}")
        res[(K,k)] = dict(zip(sms, means.tolist()))
import json
json.dump({f"{a}_{b}": v for (a,b), v in res.items()}, open('/root/repo/gpurun_out/sm_speed.json','w'))
