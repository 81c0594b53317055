"""Prints the headline and per-K class breakdown of bench JSON lines."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable:", e)
        continue
    r = d.get("roofline", {})
    print(f"{f}: value {d.get('value')} us  e2e {d.get('e2e', {}).get('value')}  frac {r.get('frac')}  step_frac {r.get('step_frac')}")
    for k, v in d.get("per_k", {}).items():
        cls = " ".join(f"{n}={t:.0f}" for n, t in v["class_us"].items())
        print(f"  K={k} {v['latency_us']:9.1f} us  U={v['unique_experts_per_layer']:.2f}  {cls}")
