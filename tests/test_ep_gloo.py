"""Expert-parallel host logic on CPU with world_size-2 gloo.

The device EP path (cascade_model_create_ep) shards routed experts
[E*r/G, E*(r+1)/G) and shared blocks b % G == r, writes each rank's
per-(token, top-k rank) expert outputs into ycontrib[T][k+S][d] with exact
zeros elsewhere, and sums the buffer with one all-reduce per layer before
the fixed-order combine.  This test runs the same algebra with the CPU
oracle's expert outputs and a real gloo all-reduce, and requires the
combined MoE output to be bit-identical to the single-rank combine
(adding exact zeros is exact), for Mixtral-like and OLMoE-like routing.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def local_range(E, r, G):
    return E * r // G, E * (r + 1) // G


def expert_outputs(shape, seed, T, rank, world, xn, topk):
    """ycontrib for this rank: rows of local experts filled, exact zeros elsewhere."""
    import sys

    sys.path.insert(0, ROOT)
    from oracle.oracle import OracleModel

    k, d, E = shape.top_k, shape.d_model, shape.experts_per_layer
    assert shape.shared_experts == 0
    om = OracleModel(shape, seed, nthreads=2)
    lo, hi = local_range(E, rank, world)
    y = np.zeros((T, k, d), np.float32)
    for t in range(T):
        for r in range(k):
            e = int(topk[t, r])
            if not lo <= e < hi:
                continue
            # this expert alone: weight 1 on slot 0, zero-weight distinct fillers
            tk = np.array([[e] + [(e + j + 1) % E for j in range(k - 1)]], np.int32)
            w = np.zeros((1, k))
            w[0, 0] = 1.0
            y[t, r] = om.moe(0, xn[t:t + 1], tk, w, np.zeros(1)).astype(np.float32)[0]
    return y


def combine(y, topw, gsh, k, S):
    T, _, d = y.shape
    out = np.zeros((T, d), np.float32)
    for t in range(T):
        acc = np.zeros(d, np.float32)
        for r in range(k):
            acc = (acc + np.float32(topw[t, r]) * y[t, r]).astype(np.float32)
        if S:
            sh = np.zeros(d, np.float32)
            for b in range(S):
                sh = (sh + y[t, k + b]).astype(np.float32)
            acc = (acc + np.float32(gsh[t]) * sh).astype(np.float32)
        out[t] = acc
    return out


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, ROOT)
        import paper_2506_20675_b200 as cb

        shape = cb.ModelShape(**case)
        rng = np.random.default_rng(0)
        T = 5
        xn = rng.integers(0x3c00, 0x3f80, (T, shape.d_model)).astype(np.uint16)
        E, k = shape.experts_per_layer, shape.top_k
        topk = np.array([rng.permutation(E)[:k] for _ in range(T)], np.int32)
        topw = rng.random((T, k))
        gsh = rng.random(T)
        y_local = expert_outputs(shape, 3, T, rank, world, xn, topk)
        y_full = expert_outputs(shape, 3, T, 0, 1, xn, topk)
        buf = torch.from_numpy(y_local.copy())
        dist.all_reduce(buf, op=dist.ReduceOp.SUM)
        y_red = buf.numpy()
        ok_buf = np.array_equal(y_red, y_full)
        ok_out = np.array_equal(combine(y_red, topw, gsh, k, shape.shared_experts),
                                combine(y_full, topw, gsh, k, shape.shared_experts))
        # each rank owns a disjoint expert slice and the slices cover E
        lo, hi = local_range(E, rank, world)
        owned = torch.tensor([hi - lo], dtype=torch.int64)
        dist.all_reduce(owned)
        q.put((rank, ok_buf, ok_out, int(owned.item()) == E))
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = {
    "mixtral_like": dict(name="m", num_layers=1, experts_per_layer=8, top_k=2, shared_experts=0, d_model=128,
                         d_ff=64, n_heads=2, n_kv_heads=1, head_dim=64, vocab=128),
    "olmoe_like": dict(name="o", num_layers=1, experts_per_layer=16, top_k=4, shared_experts=0, d_model=128,
                       d_ff=64, n_heads=2, n_kv_heads=2, head_dim=64, vocab=128, renormalize_topk=0),
}


@pytest.mark.parametrize("case", list(CASES))
def test_ep_combine_bit_identical_world2(case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, CASES[case], q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_buf, ok_out, covers in res:
        assert ok_buf, rank
        assert ok_out, rank
        assert covers, rank


def test_ep_shard_bytes_partition(cascade):
    """Per-rank weight bytes: experts partitioned, dense replicated."""
    s = cascade.preset("mixtral8x22b")
    full = cascade.model_bytes(s)
    for G in (2, 4, 8):
        parts = [cascade.model_bytes(s, r, G) for r in range(G)]
        expert = 3 * s.d_model * s.d_ff * 2 * s.num_layers * s.experts_per_layer
        assert sum(parts) == full + (G - 1) * (full - expert)
        assert max(parts) < 180e9  # every 8x22B shard fits one B200 from G=2
