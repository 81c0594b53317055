"""Generates tests/golden/specsim_reference.json from the UNMODIFIED
reference (oracle/_ref/libspecsim_ref.so, built by `make -C oracle ref`
from /root/reference/proj/include).  Run in the build container:

    python tests/golden/make_golden.py

The same scenario list is replayed against this repository's headers by
tests/test_specsim_parity.py, which requires bit-identical results.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from specsim_shim import Shim, cfg  # noqa: E402

OUT = os.path.join(HERE, "specsim_reference.json")


def unimodal(k_max, peak, gaps, min_value):
    u = [0.0] * (k_max + 1)
    u[peak] = 1.0
    for k in range(peak + 1, k_max + 1):
        u[k] = u[k - 1] / gaps[k - 2]
    for k in range(peak - 1, 0, -1):
        u[k] = u[k + 1] / gaps[k - 1]
    mn = min(u[1:])
    return [0.0] + [v * min_value / mn for v in u[1:]]


def scenarios():
    """(name, callable(shim) -> JSON-able) pairs."""
    S = []
    S.append(("expected_unique_experts", lambda s: [
        [E, k, T, s.expected_unique_experts(E, k, T)]
        for E in (4, 8, 16, 60, 64, 128) for k in (1, 2, 4, 6, 8) if k <= E for T in range(1, 17)]))
    for (E, k, Sh, aff) in [(8, 2, 0, 0.0), (8, 2, 0, 0.1), (64, 8, 0, 0.6), (60, 4, 4, 0.35), (64, 6, 2, 0.35),
                            (128, 8, 0, 0.2)]:
        S.append((f"sample_active_experts/{E}-{k}-{Sh}-{aff}", lambda s, E=E, k=k, Sh=Sh, aff=aff: [
            s.sample_active_experts(E, k, Sh, aff, T, seed, 64).tolist() for T in range(1, 10) for seed in (1, 2)]))
    for preset in ("mixtral", "phi35", "olmoe", "deepseekv1", "qwen15", "dense"):
        for draft in ("ngram", "eagle", "free"):
            S.append((f"iteration_cost/{preset}/{draft}", lambda s, p=preset, d=draft: [
                s.iteration_cost(p, d, k, 100 + k, 8).tolist() for k in range(0, 9)]))
    S.append(("sample_accepted", lambda s: [
        s.sample_accepted(p, k, 7 + k, 64).tolist() for p in (0.0, 0.2, 0.6, 0.9, 1.0) for k in range(0, 9)]))
    S.append(("trace_replay", lambda s: [
        [ko, a, k, s.trace_replay(ko, a, k)] for ko in range(0, 9) for a in range(0, ko + 1) for k in range(0, 9)]))
    # controller: Appendix A of SURVEY.md plus landscapes
    S.append(("drive/appendixA-1", lambda s: s.drive(cfg(max_trials=3), [0, 1.3, 1.5, 0.9], 400, 1)))
    S.append(("drive/flat-0.5", lambda s: s.drive(cfg(), [0, 0.5, 0.5, 0.5], 400)))
    S.append(("drive/rising", lambda s: s.drive(cfg(), [0, 1.3, 1.4, 1.5], 300)))
    S.append(("drive/kmax7-peak5", lambda s: s.drive(
        cfg(k_max=7), unimodal(7, 5, [1.3] * 6, 1.0), 200)))
    S.append(("drive/kmax7-peak5-noise", lambda s: s.drive(
        cfg(k_max=7), unimodal(7, 5, [1.3] * 6, 1.0), 300, 0, 0.05, 5000)))
    S.append(("drive/k1-loss", lambda s: s.drive(cfg(k_start=1), [0, 0.8, 0.8, 0.8], 40, 1)))
    S.append(("drive/backoff-cap", lambda s: s.drive(cfg(k_start=1, s_cap=64), [0, 0.5, 0.5, 0.5], 800, 5)))
    S.append(("drive/no-backoff", lambda s: s.drive(cfg(backoff=0), [0, 0.5, 0.5, 0.5], 800)))
    S.append(("drive/switch", lambda s: s.drive(cfg(), [0, 0.5, 0.5, 0.5], 500, 8, 0.0, 0, 120,
                                                  [0, 1.3, 1.4, 1.5])))
    rng = np.random.default_rng(2024)
    for i in range(24):
        k_max = int(rng.integers(1, 8))
        peak = int(rng.integers(1, k_max + 1))
        gaps = (1.05 + rng.random(7)).tolist()
        minv = float(0.6 + rng.random())
        u = unimodal(k_max, peak, gaps, minv)
        k_start = int(rng.integers(1, k_max + 1))
        noise = float(rng.choice([0.0, 0.05]))
        band = float(rng.choice([0.05, 0.1, 0.2]))
        S.append((f"drive/random-{i}", lambda s, c=cfg(k_max=k_max, k_start=k_start, band=band), u=u, n=noise, i=i:
                  s.drive(c, u, 300, 0, n, 77 + i)))
    for pol in (-1, 0, 1, 2, 3, 7):
        for (p, aff, preset) in [(0.0, 0.0, "mixtral"), (0.7, 0.3, "olmoe"), (1.0, 1.0, "mixtral"),
                                 (0.5, 0.35, "qwen15")]:
            S.append((f"run_request/{pol}/{p}/{aff}/{preset}", lambda s, pol=pol, p=p, aff=aff, pr=preset:
                      s.run_request(p, aff, 300, pol, pr, "ngram", 11 + pol).tolist()))
    rr = np.random.default_rng(5)
    for i in range(8):
        n = int(rr.integers(1, 40))
        k = rr.integers(0, 8, n)
        tok = np.array([1 + int(rr.integers(0, kk + 1)) for kk in k])
        tot = 0.5 + 3 * rr.random(n)
        tag = rr.integers(0, 3, n)
        S.append((f"window_utility/{i}", lambda s, k=k, tok=tok, tot=tot, tag=tag:
                  s.window_utility(int(4 + (len(k) % 5)), 1.3, k, tok, tot, tag).tolist()
                  if (tag != 0).any() else None))
    for i in range(8):
        n = 400
        tok = rr.integers(1, 9, n)
        tot = 1.0 + 2.0 * rr.random(n)
        c = cfg(k_max=int(rr.integers(1, 8)))
        c["k_start"] = int(rr.integers(1, c["k_max"] + 1))
        S.append((f"controller_replay/{i}", lambda s, c=c, tok=tok, tot=tot:
                  [a.tolist() for a in s.controller_replay(c, tok, tot)]))
    return S


def main():
    ref = Shim("ref")
    out = {name: fn(ref) for name, fn in scenarios()}
    json.dump(out, open(OUT, "w"))
    print(f"wrote {OUT}: {len(out)} scenarios, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
