#!/usr/bin/env python
"""Benchmark of the MoE verification step (BASELINE.json metric).

One bench "step" = one sweep of verification steps K = 0..8 (T = K+1 tokens
in flight) of the Mixtral-8x7B-shape model (BASELINE config 2: 8 experts
top-2, d=4096, ffn=14336, 32 layers, random-init bf16) at a committed
context of --ctx tokens.  `value` = mean device latency of one verify step
over K = 0..8 (us, lower is better), inputs resident in HBM, each graph
replay re-verifying the same context (commit=0).  The weights (93 GB) are
far larger than L2 (126 MB), so every step streams from HBM.

`e2e` = the same metric through the public C ABI call `cascade_verify`
with host drafts in and the host result struct out (H2D/D2H inside the
timed call), committing like a real decode.

`--impl reference` times the CPU implementation of the same step (the
oracle port, fp64, all host threads); the reference's own code on this
seam only prices the step (oracle/_ref iteration_cost + sample_accepted)
and is reported beside it as `reference_pricing`.

N > 1 (torchrun): experts are sharded expert-parallel across ranks (NCCL
all-reduce of the per-token expert outputs inside the step graph); the
latency is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "verify-step latency, mean over K=0..8 (us)"
KS = list(range(0, 9))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--ctx", type=int, default=1024)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-layers", type=int, default=4)
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.device = device
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in open(self.path):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- shared config
def bench_config(args, world):
    """The workload both arms report (identical dict: same_config)."""
    return {"workload": f"{args.config} verify step K=0..8 (one bench step = one K sweep)",
            "ctx": args.ctx, "parallelism": f"ep{world}" if world > 1 else "single-device",
            "l2": "inputs larger than L2 (93 GB of weights streamed per sweep)"}


# ----------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """The reference arm: a CPU implementation of the same verify step.

    The reference (specsim) compiles here (oracle/_ref), but on this seam it
    *prices* the step (iteration_cost + sample_accepted, expert_model.hpp:
    145-172, workload.hpp:80-86) instead of computing it: it has no weights,
    router, FFN, attention or LM head.  The CPU implementation of the step
    itself is the oracle port (oracle/, fp64, all host threads), so that is
    the timed arm (kind "port").  Each bench step is one K = 0..8 sweep of
    REAL verify steps through a bounded slice of the model (--cpu-layers
    chained layers + final norm + LM head + greedy acceptance); `value` and
    `ms_per_step` are exactly that timed work.  The full-depth figure
    (slice layers scaled to num_layers, LM head once) is reported apart, in
    `extrapolated_full_depth`.  The reference's own pricing call is timed
    beside it under `reference_pricing` (it computes a cost, not the step)."""
    import ctypes

    if rank != 0:
        return 0
    import paper_2506_20675_b200 as cb

    shape = cb.preset(args.config)
    n_layers = args.cpu_layers
    line = {"impl": "reference", "metric": METRIC, "unit": "us", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (random-init counter-hash weights, random prompt/drafts)",
            "config": bench_config(args, world)}
    cpu = CpuSlice(shape, args.seed, args.ctx, n_layers)
    per_step, per_k, full = [], {K: [] for K in KS}, []
    for i in range(args.warmup + args.steps):
        lat, lat_full = cpu.sweep()
        if i >= args.warmup:
            per_step.append(float(np.sum(lat)))
            full.append(float(np.mean(lat_full)))
            for K, v in zip(KS, lat):
                per_k[K].append(v)
    v = float(np.mean(per_step)) / len(KS)
    sample = cpu.describe()
    line.update({"value": round(v, 1), "ms_per_step": round(float(np.mean(per_step)) / 1e3, 3),
                 "cpu_baseline": {"value": round(v, 1), "unit": "us", "cores": cpu.cores, "kind": "port",
                                  "sample": sample},
                 "e2e": {"value": round(v, 1), "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                 "per_k_us": {K: round(float(np.mean(per_k[K])), 1) for K in KS},
                 "extrapolated_full_depth": {
                     "value": round(float(np.mean(full)), 1), "unit": "us",
                     "how": f"measured per-layer time of the {n_layers}-layer slice x {shape.num_layers} layers "
                            "+ the measured LM head/accept time (not timed end to end)"}})
    path = os.path.join(ROOT, "oracle", "_ref", "libspecsim_ref.so")
    if os.path.exists(path) and args.config in ("mixtral", "olmoe", "qwen15"):
        L = ctypes.CDLL(path)
        L.ref_time_verify.restype = ctypes.c_double
        L.ref_time_verify.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_long]
        calls = 20000
        tot = 0.0
        for K in KS:
            ns = L.ref_time_verify(args.config.encode(), K, 0.5, 1, calls)
            tot += ns / calls / 1e3
        line["reference_pricing"] = {
            "value": round(tot / len(KS), 4), "unit": "us", "cores": 1,
            "what": f"unmodified reference iteration_cost({args.config} preset)+sample_accepted per K=0..8 "
                    "(oracle/_ref): prices the verify step, computes no model numerics"}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------- CPU oracle slice
class CpuSlice:
    """Real-numerics CPU verify steps (fp64 oracle, all host threads) on a
    bounded slice of the model: the pending token + K drafts are embedded,
    run through layers 0..n_layers-1 (RMSNorm, RoPE attention over a ctx-row
    KV cache, router top-k, union, SwiGLU experts, residuals) chained on the
    real activations, then the final norm, LM head, argmax and greedy
    acceptance.  Weights of the slice are generated before timing; the ctx
    KV rows are synthetic bf16 (their values do not change the work)."""

    def __init__(self, shape, seed, ctx, n_layers):
        from oracle.oracle import OracleModel

        import paper_2506_20675_b200 as cb

        self.cb = cb
        self.shape, self.ctx, self.n_layers = shape, ctx, n_layers
        self.om = OracleModel(shape, seed)
        self.cores = self.om.nthreads
        rng = np.random.default_rng(seed)
        kvs = (shape.n_kv_heads, ctx, shape.head_dim)
        self.kv = [(rng.integers(0x3c00, 0x3f00, kvs).astype(np.uint16),
                    rng.integers(0x3c00, 0x3f00, kvs).astype(np.uint16)) for _ in range(n_layers)]
        self.tokens = rng.integers(0, shape.vocab, 64).astype(np.int32)
        for l in range(n_layers):
            self.om.prepare_layer(l, list(range(shape.experts_per_layer + shape.shared_experts)))
        self.om.tensor(cb.T_LM_HEAD, 0, 0, 0, 1, shape.d_model)
        self.emb = {}

    def _embed(self, toks):
        rows = []
        for t in toks:
            t = int(t)
            if t not in self.emb:
                self.emb[t] = (self.om.tensor(self.cb.T_EMBED, 0, 0, t, 1, self.shape.d_model).astype(np.uint32)
                               << 16).view(np.float32)[0]
            rows.append(self.emb[t])
        return np.stack(rows).astype(np.float32)

    def step(self, K, it):
        """One verify step of width K+1; returns (slice us, layer-only us, head us)."""
        from oracle.oracle import greedy_accept

        cb, om = self.cb, self.om
        toks = np.roll(self.tokens, -it)[: K + 1]
        t0 = time.perf_counter()
        x = self._embed(toks)
        for l in range(self.n_layers):
            a, _, _ = om.attention(l, x, self.ctx, self.kv[l][0], self.kv[l][1])
            xm = (x + a).astype(np.float32)
            xn = om.rmsnorm(cb.T_FFN_NORM, l, xm)
            _, topk, topw, gsh, _ = om.router(l, xn)
            x = (xm + om.moe(l, xn, topk, topw, gsh)).astype(np.float32)
        t1 = time.perf_counter()
        _, am, _ = om.lm_head(om.rmsnorm(cb.T_FINAL_NORM, 0, x))
        greedy_accept(am, toks[1:])
        t2 = time.perf_counter()
        return (t2 - t0) * 1e6, (t1 - t0) * 1e6, (t2 - t1) * 1e6

    def sweep(self, it=0):
        lat, full = [], []
        for K in KS:
            tot, layers, head = self.step(K, it + K)
            lat.append(tot)
            full.append(layers / self.n_layers * self.shape.num_layers + head)
        return lat, full

    def describe(self):
        return (f"CPU oracle port (fp64, {self.cores} threads): real verify steps K=0..8 through layers "
                f"0..{self.n_layers - 1} of {self.shape.name} (embedding, attention over {self.ctx} synthetic "
                f"KV rows, router, union, experts, chained on the real activations) + final norm + LM head + "
                f"greedy accept; weights pre-generated; value = that {self.n_layers}-layer slice, not scaled")


# ----------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import ctypes

    import torch

    import paper_2506_20675_b200 as cb

    dist = None
    if world > 1:
        import torch.distributed as dist_

        dist = dist_
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    shape = cb.preset(args.config)
    if world > 1:
        uid = cb.ep_unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8, device="cuda")
        dist.broadcast(t, 0)
        uid = bytes(t.cpu().tolist())
        model = cb.Model(shape, args.seed, device=local_rank, ep_rank=rank, ep_size=world, nccl_id=uid)
    else:
        model = cb.Model(shape, args.seed, device=local_rank)
    ctx = args.ctx
    n_commit = (args.warmup + args.steps + 2) * len(KS) + 64
    sess = cb.Session(model, max_ctx=ctx + n_commit, k_max=max(KS))
    rng = np.random.default_rng(args.seed)
    prompt = rng.integers(0, shape.vocab, ctx + 1).astype(np.int32)
    sess.prefill(prompt)  # cache_len = ctx
    stream = ctypes.c_void_p(sess.stream())
    torch_stream = torch.cuda.ExternalStream(stream.value, device=f"cuda:{local_rank}")

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warmup (graphs captured on first use)
    kernels = {K: sess.kernel_count(K) for K in KS}
    for _ in range(args.warmup):
        for K in KS:
            sess.enqueue(K, commit=False)
    sess.sync()

    # ---- timed region: `steps` sweeps of K = 0..8, CUDA events on the session stream
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    ev = {K: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)] for K in KS}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(torch_stream)
    for s in range(args.steps):
        for K in KS:
            ev[K][s][0].record(torch_stream)
            sess.enqueue(K, commit=False)
            ev[K][s][1].record(torch_stream)
    e1.record(torch_stream)
    sess.sync()
    barrier()
    clk = clocks.stop()
    total_ms = e0.elapsed_time(e1)
    per_k_us = {K: float(np.mean([a.elapsed_time(b) for a, b in ev[K]]) * 1e3) for K in KS}
    if dist is not None:
        t = torch.tensor([total_ms] + [per_k_us[K] for K in KS], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t[0])
        per_k_us = {K: float(t[1 + i]) for i, K in enumerate(KS)}
    ms_per_step = total_ms / args.steps
    value = float(np.mean([per_k_us[K] for K in KS]))

    # ---- roofline: in-graph per-kernel durations of one captured step per K
    #      (globaltimer start stamps of consecutive kernels on the graph timeline)
    peak, peak_kind = measured_peaks()
    per_k = {}
    exp_bytes = exp_ns = 0.0
    for K in KS:
        ns, kind = sess.trace(K)
        us = sess.union_sizes()
        T = K + 1
        b = shape.step_bytes(us, ctx, T)
        cls = {}
        for n_, k_ in zip(ns, kind):
            cls[cb.KERNEL_CLASSES[k_]] = cls.get(cb.KERNEL_CLASSES[k_], 0.0) + float(n_)
        d, f = shape.d_model, shape.d_ff
        eb = sum((int(u) + shape.shared_experts) for u in us) * 3 * d * f * 2
        et = cls.get("expert_gate_up", 0.0) + cls.get("expert_down", 0.0)
        exp_bytes += eb
        exp_ns += et
        # effective tokens/s = E[emitted] / latency under the reference's i.i.d.
        # acceptance model (workload.hpp:80-86): E[emitted] = sum_{j=0..K} p^j
        eff = {f"p={pa}": round(sum(pa ** j for j in range(K + 1)) / (per_k_us[K] * 1e-6), 1) for pa in (0.6, 0.8)}
        per_k[K] = {"latency_us": round(per_k_us[K], 2),
                    "effective_tokens_per_s": eff,
                    "bytes_gb": round(b["total"] / 1e9, 3),
                    "hbm_gbs": round(b["total"] / (per_k_us[K] * 1e3), 1),
                    "roofline_frac": round(b["total"] / (per_k_us[K] * 1e3) / peak, 4),
                    "unique_experts_per_layer": round(float(np.mean(us)), 3),
                    "expert_gbs": round(eb / et, 1) if et else None,
                    "class_us": {k: round(v / 1e3, 1) for k, v in cls.items()}}
    achieved = exp_bytes / exp_ns  # GB/s (bytes per ns)
    prof_path = os.path.join(ROOT, "profiles", "ncu_expert_traffic.json")
    traffic = traffic_alg = traffic_src = None
    if os.path.exists(prof_path):
        try:
            pj = json.load(open(prof_path))
            traffic, traffic_alg = pj.get("traffic_bytes_per_launch"), pj.get("algorithmic_bytes_per_launch")
            traffic_src = {k: pj.get(k) for k in ("launch", "source", "commit", "command")}
        except Exception:
            traffic = None
    # the sweep runs the ring engine at K <= 7 and the register engine at K = 8:
    # the ring engine's capture (K=4) is reported beside the K=8 one
    ring_traffic = None
    ring_path = os.path.join(ROOT, "profiles", "ncu_expert_ring_traffic.json")
    if os.path.exists(ring_path):
        try:
            rj = json.load(open(ring_path))
            ring_traffic = {k: rj.get(k) for k in ("traffic_bytes_per_launch", "algorithmic_bytes_per_launch",
                                                   "ratio_traffic_over_algorithmic", "launch", "commit", "command")}
        except Exception:
            ring_traffic = None
    mean_bytes = float(np.mean([per_k[K]["bytes_gb"] for K in KS])) * 1e9

    # ---- e2e through the public call (host drafts in, host struct out, committing)
    import ctypes as _c

    e2e = {}
    for _ in range(1):
        for K in KS:
            sess.verify(rng.integers(0, shape.vocab, K).astype(np.int32))
    lat_e2e = {K: [] for K in KS}
    barrier()
    for s in range(args.steps):
        for K in KS:
            drafts = rng.integers(0, shape.vocab, K).astype(np.int32)
            t0 = time.perf_counter()
            sess.verify(drafts)
            lat_e2e[K].append((time.perf_counter() - t0) * 1e6)
    barrier()
    e2e_v = float(np.mean([np.mean(lat_e2e[K]) for K in KS]))
    if dist is not None:
        t = torch.tensor([e2e_v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_v = float(t[0])
    h2d = 96  # StepParams (mode, commit, T, tokens[16], t_base, draft_ns)
    d2h = _c.sizeof(cb.VerifyOut)

    if rank != 0:
        return 0
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cs = CpuSlice(shape, args.seed, ctx, args.cpu_layers)
            lat, full = cs.sweep()
            cpu = {"value": round(float(np.mean(lat)), 1), "unit": "us", "cores": cs.cores, "kind": "port",
                   "sample": cs.describe(),
                   "extrapolated_full_depth_us": round(float(np.mean(full)), 1)}
            del cs
        except Exception as e:  # the baseline must not kill the GPU line
            cpu = {"value": None, "unit": "us", "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {e}"}
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "us",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 3),
        "higher_is_better": False,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (random-init counter-hash weights, random prompt/drafts)",
        "config": bench_config(args, world),
        "e2e": {"value": round(e2e_v, 2), "unit": "us", "h2d_bytes_per_step": h2d * len(KS),
                "d2h_bytes_per_step": d2h * len(KS)},
        "gpu_launches": int(sum(kernels.values()) * args.steps),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "traffic_algorithmic_bytes": traffic_alg,
                     "traffic_provenance": traffic_src,
                     "traffic_ring_engine": ring_traffic,
                     "kernel": "expert GEMV (gate/up+SiLU and down), bytes = sum_l (U_l+S)*3*d*f*2",
                     "peak_kind": peak_kind,
                     "step_frac": round(mean_bytes / (value * 1e3) / peak, 4)},
        "per_k": per_k,
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line))
    sess.close()
    model.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
