"""Summarises an ncu launch list (gpu__time_duration.sum CSV) per kernel class."""
import collections
import csv
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.DictReader(lines[start:]))
EPI = {"0": "qkv(STORE)", "1": "o_proj(ADD)", "2": "expert_gate_up", "3": "expert_down", "4": "lm_head(ARGMAX)"}


def cls(n):
    m = re.search(r"stream_gemv_kernel<(\d), (\d)>", n)
    if m:
        return f"gemv NT={m.group(1)} {EPI[m.group(2)]}"
    m = re.search(r"(attn_partial_kernel|attn_combine_kernel|moe_route_kernel|moe_combine_kernel|embed_norm_kernel|accept_kernel)", n)
    return m.group(1) if m else n[:40]


per_step = int(sys.argv[2]) if len(sys.argv) > 2 else len(rows)
labels = sys.argv[3].split(",") if len(sys.argv) > 3 else None
for s in range(0, len(rows), per_step):
    chunk = rows[s:s + per_step]
    agg = collections.OrderedDict()
    cnt = collections.Counter()
    tot = 0.0
    for r in chunk:
        c = cls(r["Kernel Name"])
        v = float(r["Metric Value"]) / 1000
        agg[c] = agg.get(c, 0) + v
        cnt[c] += 1
        tot += v
    lab = labels[s // per_step] if labels else s // per_step
    print(f"step {lab}: {len(chunk)} launches, sum of kernel time {tot:.1f} us")
    for c in agg:
        print(f"  {c:34s} n={cnt[c]:3d} total={agg[c]:9.1f} us  mean={agg[c] / cnt[c]:8.2f} us  share={agg[c] / tot:6.1%}")
