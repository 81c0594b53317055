"""Summarises an ncu launch list (gpu__time_duration.sum CSV) per kernel class,
one block per verify step (a step starts at embed_norm_kernel).
Usage: python scripts/launch_summary.py launches.csv [label,label,...]"""
import collections
import csv
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = [r for r in csv.DictReader(lines[start:]) if r["Metric Name"] == "gpu__time_duration.sum"]
EPI = {"0": "qkv(STORE)", "1": "o_proj(ADD)", "2": "expert_gate_up", "3": "expert_down", "4": "lm_head(ARGMAX)"}


def cls(n):
    m = re.search(r"stream_gemv_umma_kernel<\(?[a-z]*\)?(\d)", n)
    if m:
        return f"tcgen05 gemv {EPI[m.group(1)]}"
    m = re.search(r"dense_gemv_cluster_kernel<\(?[a-z]*\)?(\d)", n)
    if m:
        return f"tcgen05 cluster split-K {EPI[m.group(1)]}"
    m = re.search(r"expert_ffn_kernel<\(?[a-z]*\)?(\d)>", n)
    if m:
        return f"mma.sync fused expert FFN NT={m.group(1)} (gate/up + down)"
    m = re.search(r"stream_gemv_kernel<\(?[a-z]*\)?(\d), \(?[a-z]*\)?(\d)>", n)
    if m:
        return f"mma.sync gemv NT={m.group(1)} {EPI[m.group(2)]}"
    m = re.search(r"(attn_partial_kernel|attn_combine_kernel|moe_route_kernel|moe_combine_kernel|embed_norm_kernel|accept_kernel)", n)
    return m.group(1) if m else n[:40]


steps, cur = [], []
for r in rows:
    if "embed_norm_kernel" in r["Kernel Name"] and cur:
        steps.append(cur)
        cur = []
    cur.append(r)
if cur:
    steps.append(cur)
labels = sys.argv[2].split(",") if len(sys.argv) > 2 else [str(i) for i in range(len(steps))]
for lab, chunk in zip(labels, steps):
    agg, cnt, tot = collections.OrderedDict(), collections.Counter(), 0.0
    for r in chunk:
        c = cls(r["Kernel Name"])
        v = float(r["Metric Value"]) / 1000
        agg[c] = agg.get(c, 0) + v
        cnt[c] += 1
        tot += v
    print(f"step {lab}: {len(chunk)} launches, sum of kernel time {tot:.1f} us (ncu: serialised, caches flushed)")
    for c in agg:
        print(f"  {c:36s} n={cnt[c]:3d} total={agg[c]:9.1f} us  mean={agg[c] / cnt[c]:8.2f} us  share={agg[c] / tot:6.1%}")
