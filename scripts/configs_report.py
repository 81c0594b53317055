"""BASELINE configs 3-5 on one B200 (writes profiles/configs_<tag>.json).

config 3  OLMoE-1B-7B shape: verify latency and measured expert-union
          growth U(K) vs the bucket-and-balls closed form
          E*(1-(1-k/E)^(K+1)) (expert_model.hpp:84-92), K = 0..8.
config 4  Qwen1.5-MoE-A2.7B shape: greedy decode through cascade_decode
          with the utility-driven test-and-set controller choosing K
          (device-measured costs), vs static K and no speculation, with the
          replay drafter at acceptance p = 0.6 / 0.8 / 0.95 (the random-init
          model never repeats the prompt, so n-gram drafts are never
          accepted); the same effective tokens/s sweep for Mixtral-8x7B.
config 5  Mixtral-8x22B shape: 281 GB does not fit one GPU; a 24-layer
          slice (121 GB) gives the per-layer verify cost K = 0..8 (the
          expert-parallel run across 2/4/8 GPUs needs a multi-GPU box).
"""

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_20675_b200 as cb  # noqa: E402

KS = list(range(9))
TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def closed_form(E, k, T):
    return E * (1 - (1 - k / E) ** T)


def latency_sweep(shape, ctx=1024, reps=5, prompts=4, seed=1, invariant=False):
    m = cb.Model(shape, seed)
    out = {}
    rng = np.random.default_rng(seed)
    u_acc = {K: [] for K in KS}
    lat = {K: [] for K in KS}
    for pi in range(prompts):
        s = cb.Session(m, max_ctx=ctx + 64, k_max=15)
        s.set_batch_invariant(invariant)
        s.prefill(rng.integers(0, shape.vocab, ctx + 1).astype(np.int32))
        for K in KS:
            s.enqueue(K)
        s.sync()
        for K in KS:
            ns, kind = s.trace(K)  # one captured step; union sizes of this step
            u_acc[K].append(float(np.mean(s.union_sizes())))
            st = torch.cuda.ExternalStream(s.stream(), device="cuda:0")
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(reps):
                s.enqueue(K, commit=False)
            e1.record(st)
            s.sync()
            lat[K].append(e0.elapsed_time(e1) / reps * 1e3)  # device time on the session stream
        s.close()
    for K in KS:
        U = float(np.mean(u_acc[K]))
        us = [U] * shape.num_layers
        b = shape.step_bytes(us, ctx, K + 1)["total"]
        t = float(np.median(lat[K]))
        out[K] = {"latency_us": round(t, 1), "unique_experts_per_layer": round(U, 3),
                  "closed_form_uniform": round(closed_form(shape.experts_per_layer, shape.top_k, K + 1), 3),
                  "bytes_gb": round(b / 1e9, 3), "hbm_gbs": round(b / (t * 1e3), 1),
                  "roofline_frac": round(b / (t * 1e3) / PEAK, 4)}
    m.close()
    return out


def spec_decode(shape, seed=3, max_new=256, ps=(0.6, 0.8, 0.95), statics=(1, 2, 3, 4, 6), k_max=7):
    """Speculative greedy decode on the device with the replay drafter: the
    model's own K=0 greedy continuation, each proposal kept with
    probability p (i.i.d. acceptance, the reference's workload model).
    Reports effective tokens/s (device time) for no speculation, static K
    and the utility-driven test-and-set controller."""
    m = cb.Model(shape, seed)
    s = cb.Session(m, max_ctx=2048, k_max=15)
    s.set_batch_invariant(True)  # bitwise-lossless speculation: replay drafts stay aligned with the K=0 sequence
    rng = np.random.default_rng(seed)
    prompt = rng.integers(0, shape.vocab, 64).astype(np.int32)
    truth, _, _ = s.decode(prompt, cb.decode_cfg(policy=0, max_new=max_new + 16), telemetry_cap=0)
    res = {}

    def run(label, pol, p):
        cfg = cb.decode_cfg(policy=pol, max_new=max_new, k_max=k_max, replay=(truth, p, 1234))
        t0 = time.perf_counter()
        toks, tel, n_it = s.decode(prompt, cfg, telemetry_cap=4096)
        wall = time.perf_counter() - t0
        assert list(toks[:max_new]) == list(truth[:max_new]), "speculative decode must be lossless"
        dev_ns = float(tel[:, 6].sum())
        ks, cnt = np.unique(tel[:, 1].astype(int), return_counts=True)
        return {"tokens": int(len(toks)), "iterations": int(n_it), "etr": round(len(toks) / n_it, 3),
                "device_ms": round(dev_ns / 1e6, 2), "tokens_per_s_device": round(len(toks) / (dev_ns / 1e9), 1),
                "tokens_per_s_wall": round(len(toks) / wall, 1),
                "k_histogram": {int(a): int(b) for a, b in zip(ks, cnt)}}

    base = run("none", 0, 1.0)
    res["none"] = base
    for p in ps:
        r = {}
        for k in statics:
            r[f"static:{k}"] = run(f"static:{k}", k, p)
        r["adaptive"] = run("adaptive", -1, p)
        for v in r.values():
            v["speedup_vs_none"] = round(v["tokens_per_s_device"] / base["tokens_per_s_device"], 3)
        res[f"p={p}"] = r
    s.close()
    m.close()
    return res


def ep_shard_sweep(shape, G=2, ctx=1024, ks=(0, 2, 4, 8), seed=1):
    """Expert-parallel shards measured one at a time on this one GPU
    (CASCADE_EP_NOCOMM=1: no all-reduce).  The EP step on G GPUs costs the
    max over ranks of these plus one all-reduce of T*(k+S)*d fp32 per layer,
    which is reported as a byte count (not measured here)."""
    os.environ["CASCADE_EP_NOCOMM"] = "1"
    out = {}
    try:
        for r in range(G):
            m = cb.Model(shape, seed, device=0, ep_rank=r, ep_size=G, nccl_id=bytes(128))
            s = cb.Session(m, max_ctx=ctx + 64, k_max=15)
            rng = np.random.default_rng(seed)
            s.prefill(rng.integers(0, shape.vocab, ctx + 1).astype(np.int32))
            st = torch.cuda.ExternalStream(s.stream(), device="cuda:0")
            res = {}
            for K in ks:
                for _ in range(2):
                    s.enqueue(K, commit=False)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(3):
                    s.enqueue(K, commit=False)
                e1.record(st)
                s.sync()
                U = float(np.mean(s.union_sizes()))
                res[K] = {"latency_us": round(e0.elapsed_time(e1) / 3 * 1e3, 1), "unique_experts_per_layer": round(U, 3),
                          "allreduce_bytes_per_layer": (K + 1) * (shape.top_k + shape.shared_experts) * shape.d_model * 4,
                          "shard_bytes_gb": round(cb.model_bytes(shape, r, G) / 1e9, 1)}
            out[f"rank{r}"] = res
            s.close()
            m.close()
    finally:
        os.environ.pop("CASCADE_EP_NOCOMM", None)
    return out


def scenario_sweep(shape, seed=5):
    """Reference scenario sweep (engine.hpp run_scenario) with verifier-backed cells:
    two tasks (a phased high/low-acceptance profile and a low-acceptance mix) x
    {none, static 2, static 4, adaptive}; speedup vs none and utility->speedup OLS."""
    m = cb.Model(shape, seed)
    s = cb.Session(m, max_ctx=1024, k_max=15)
    tasks = {"phased_0.9_0.5": [(1.0, [(0.9, 16.0), (0.5, 16.0)], (96, 128))],
             "mix_0.3_0.6": [(0.5, [(0.3, 1.0)], (96, 96)), (0.5, [(0.6, 1.0)], (128, 128))]}
    rep = cb.run_scenario(s, tasks, [0, 2, 4, -1], tokens_per_cell=512, prompt_len=64, seed=seed, k_max=7)
    s.close()
    m.close()
    for c in rep["cells"]:
        for k in ("total_time", "t_base", "tpot"):
            c[k] = round(c[k], 1)
        for k in ("etr", "cost", "utility", "utility_hmean", "speedup"):
            c[k] = round(c[k], 4) if c[k] is not None else None
    return rep


def main():
    report = {"peak_hbm_gbs": PEAK}
    report["config3_olmoe"] = latency_sweep(cb.preset("olmoe"))
    report["config4_qwen15_controller"] = spec_decode(cb.preset("qwen15"))
    report["config2_mixtral_effective_tokens"] = spec_decode(cb.preset("mixtral"), max_new=128, statics=(1, 2, 4, 6, 8),
                                                              ps=(0.6, 0.8))
    report["config4_qwen15_latency"] = latency_sweep(cb.preset("qwen15"), prompts=2)
    report["config2_mixtral_latency_batch_invariant"] = latency_sweep(cb.preset("mixtral"), prompts=1,
                                                                       invariant=True)
    report["config4_qwen15_scenario"] = scenario_sweep(cb.preset("qwen15"))
    report["config2_mixtral_ctx4096"] = latency_sweep(cb.preset("mixtral"), ctx=4096, prompts=1)
    report["config5_mixtral8x22b_ep2_shards"] = ep_shard_sweep(cb.preset("mixtral8x22b"), G=2)
    report["config5_mixtral8x22b_24layer_slice"] = latency_sweep(cb.preset("mixtral8x22b").with_layers(24), prompts=1)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out", f"configs_{TAG}.json")
    json.dump(report, open(path, "w"), indent=1)
    print(json.dumps(report))


if __name__ == "__main__":
    main()
