"""Expert-parallel shards of the Mixtral-8x22B shape (BASELINE config 5),
each measured on this one GPU without the per-layer combine
(CASCADE_EP_NOCOMM=1): rank r of G holds routed experts [E r/G, E(r+1)/G)
of all 56 layers plus the replicated dense weights, and runs the full
verify step.  Routing after layer 0 follows the shard's own partial
activations, so the bytes per rank are representative and the values are
not; the EP step on G GPUs costs about the max over ranks of these plus one
combine per layer (T*(k+S)*d fp32, reported as bytes).
usage: python scripts/ep_shards.py G[,G...] out.json"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_20675_b200 as cb  # noqa: E402

KS = (0, 2, 4, 8)


def shard_sweep(shape, G, ctx=1024, seed=1):
    os.environ["CASCADE_EP_NOCOMM"] = "1"
    out = {}
    for r in range(G):
        m = cb.Model(shape, seed, device=0, ep_rank=r, ep_size=G, nccl_id=bytes(128))
        s = cb.Session(m, max_ctx=ctx + 64, k_max=15)
        s.prefill(np.random.default_rng(seed).integers(0, shape.vocab, ctx + 1).astype(np.int32))
        st = torch.cuda.ExternalStream(s.stream(), device="cuda:0")
        res = {}
        for K in KS:
            for _ in range(2):
                s.enqueue(K, commit=False)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(3):
                s.enqueue(K, commit=False)
            e1.record(st)
            s.sync()
            us = s.union_sizes()
            res[K] = {"latency_us": round(e0.elapsed_time(e1) / 3 * 1e3, 1),
                      "unique_experts_per_layer": round(float(np.mean(us)), 3),
                      "combine_bytes_per_layer": (K + 1) * (shape.top_k + shape.shared_experts) * shape.d_model * 4}
        out[f"rank{r}"] = {"shard_bytes_gb": round(cb.model_bytes(shape, r, G) / 1e9, 1), "per_k": res}
        s.close()
        m.close()
    out["max_over_ranks_us"] = {K: max(out[f"rank{r}"]["per_k"][K]["latency_us"] for r in range(G)) for K in KS}
    return out


if __name__ == "__main__":
    Gs = [int(g) for g in sys.argv[1].split(",")]
    path = sys.argv[2]
    shape = cb.preset("mixtral8x22b")
    rep = {f"G={G}": shard_sweep(shape, G) for G in Gs}
    json.dump(rep, open(path, "w"), indent=1)
    print(json.dumps({k: v["max_over_ranks_us"] for k, v in rep.items()}))
