"""GPU parity of the full verification step on the tiny config (BASELINE
config 1: 8 experts top-2, 4 layers), through the C ABI, against the CPU
oracle on identical counter-hash weights.

Bars:
  * weights: bit-exact (same hash, device layout undone by read-back)
  * router top-k, expert union, greedy argmax and accepted counts: exact,
    except where the oracle's own decision margin is below MARGIN (flagged)
  * logits / layer outputs: |gpu - oracle| <= ATOL + RTOL * max|oracle|
"""

import numpy as np
import pytest

import paper_2506_20675_b200 as cb
from oracle.oracle import OracleModel, OracleSession, greedy_accept, union

pytestmark = pytest.mark.gpu

SEED = cb.TINY_SEED
MARGIN = 2e-3      # decision margins below this are flagged, not failed
LOGIT_RTOL = 1e-2  # of max |logit|
LOGIT_ATOL = 2e-3


def bf2f(a):
    return (np.asarray(a, np.uint32) << 16).view(np.float32)


@pytest.fixture(scope="module")
def tiny():
    shape = cb.preset("tiny")
    m = cb.Model(shape, SEED)
    om = OracleModel(shape, SEED)
    yield shape, m, om
    m.close()


def prompt(n=48, seed=3):
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 1024, 12)
    return np.concatenate([base, base[:5], rng.integers(0, 1024, n - 17)]).astype(np.int32)


def test_device_weights_bit_exact(tiny):
    shape, m, om = tiny
    d, f, hq, kvd = shape.d_model, shape.d_ff, shape.n_heads * shape.head_dim, shape.n_kv_heads * shape.head_dim
    cases = [
        (cb.T_EMBED, 0, 0, 0, 50, d),
        (cb.T_ATTN_NORM, 1, 0, 0, 1, d),
        (cb.T_FFN_NORM, 3, 0, 0, 1, d),
        (cb.T_WQ, 0, 0, 0, hq, d),
        (cb.T_WK, 2, 0, 0, kvd, d),
        (cb.T_WV, 3, 0, 0, kvd, d),
        (cb.T_WO, 1, 0, 0, d, hq),
        (cb.T_ROUTER, 2, 0, 0, shape.experts_per_layer, d),
        (cb.T_W_GATE, 1, 5, 0, f, d),
        (cb.T_W_UP, 1, 5, 0, f, d),
        (cb.T_W_DOWN, 3, 7, 0, d, f),
        (cb.T_LM_HEAD, 0, 0, 100, 64, d),
        (cb.T_FINAL_NORM, 0, 0, 0, 1, d),
    ]
    for kind, layer, expert, row0, n, cols in cases:
        g = m.read_weight(kind, layer, expert, row0, n, cols)
        o = om.tensor(kind, layer, expert, row0, n, cols)
        assert np.array_equal(g, o), (kind, layer, expert)


def test_teacher_forced_stages(tiny):
    """One verify step with debug taps; every stage checked against the oracle
    fed the device's own stage inputs (so errors do not compound)."""
    shape, m, om = tiny
    s = cb.Session(m, max_ctx=256, k_max=8)
    p = prompt()
    s.prefill(p)
    ctx = len(p) - 1
    s.enable_taps(True)
    drafts = np.array([11, 22, 33, 44, 55, 66, 77, 88], np.int32)
    out = s.verify(drafts)
    T = len(drafts) + 1
    x_in, x_mid = s.tap("x_in"), s.tap("x_mid")
    xn_attn, xn_moe = s.tap("xn_attn"), s.tap("xn_moe")
    rl, tid, tw, moe = s.tap("router_logits"), s.tap("topk_id"), s.tap("topk_w"), s.tap("moe_out")
    flagged = 0
    for l in range(shape.num_layers):
        kc = s.read_kv(l, 0, ctx + T)
        vc = s.read_kv(l, 1, ctx + T)
        # attention input norm: bf16 outputs may differ by one ulp at rounding ties
        ox = om.rmsnorm(cb.T_ATTN_NORM, l, x_in[l, :T])
        diff = np.abs(ox.astype(np.int32) - xn_attn[l, :T].astype(np.int32))
        assert diff.max() <= 1 and (diff > 0).mean() < 0.01
        # attention block (RoPE, KV append, causal GQA, O-proj)
        oa, kn, vn = om.attention(l, x_in[l, :T], ctx, kc[:, :ctx], vc[:, :ctx])
        ga = x_mid[l, :T].astype(np.float64) - x_in[l, :T]
        assert np.abs(ga - oa).max() <= 1e-3 + 1e-2 * np.abs(oa).max()
        # appended KV rows (bf16, may differ by one ulp)
        dk = np.abs(bf2f(kc[:, ctx:ctx + T]) - bf2f(kn))
        assert dk.max() <= 1e-2 * max(1.0, np.abs(bf2f(kn)).max())
        # router on the device's MoE input
        ox2 = om.rmsnorm(cb.T_FFN_NORM, l, x_mid[l, :T])
        assert np.abs(ox2.astype(np.int32) - xn_moe[l, :T].astype(np.int32)).max() <= 1
        logits, topk, topw, gsh, margin = om.router(l, xn_moe[l, :T])
        E = shape.experts_per_layer
        assert np.abs(rl[l, :T, :E] - logits[:, :E]).max() <= 1e-4 * max(1, np.abs(logits).max())
        for t in range(T):
            if margin[t] < MARGIN:
                flagged += 1
                continue
            assert list(tid[l, t]) == list(topk[t]), (l, t)
            assert np.allclose(tw[l, t], topw[t], rtol=1e-5, atol=1e-6)
        # expert union of the step equals the oracle's union
        assert sorted(set(tid[l, :T].ravel())) == list(union(tid[l, :T]))
        # MoE block on the device routing
        om_out = om.moe(l, xn_moe[l, :T], tid[l, :T], tw[l, :T].astype(np.float64), gsh)
        assert np.abs(moe[l, :T] - om_out).max() <= 1e-3 + 1e-2 * np.abs(om_out).max()
    # LM head on the device's final norm input (x after last layer = x_mid + moe)
    x_last = x_mid[-1, :T].astype(np.float64) + moe[-1, :T]
    xf = om.rmsnorm(cb.T_FINAL_NORM, 0, x_last.astype(np.float32))
    lg, am, mg = om.lm_head(xf)
    glog = s.tap("final_logits")[:T]
    assert np.abs(glog - lg).max() <= LOGIT_ATOL + LOGIT_RTOL * np.abs(lg).max()
    for t in range(T):
        if mg[t] >= MARGIN:
            assert out.argmax[t] == am[t]
    acc, _ = greedy_accept(np.array(out.argmax[:T]), drafts)
    assert out.accepted == acc
    assert flagged <= T  # near-ties are rare with router_scale 4
    s.close()


def greedy_sequence(om, p, n):
    os_ = OracleSession(om, 512)
    os_.prefill(p)
    seq = []
    for _ in range(n):
        acc, am, lg, mg, us = os_.verify([])
        seq.append(int(am[0]))
    return seq


# End to end (no teacher forcing) the random-init tiny model amplifies the
# bf16 rounding-flip noise of each stage (~1e-4, see the teacher-forced
# test) to ~1.5% of the logit range after 4 layers; the bounds below state
# that.  Teacher-forced stage bars are 100x tighter.
E2E_LOGIT_RTOL = 3e-2
ROUTER_FLIP_BOUND = 0.25   # a device/oracle routing disagreement needs an oracle gap below this


def assert_first_flip_is_near_tie(gtk, otk, omg):
    """Routing disagreement [L, T, k]: only the first layer that disagrees
    is an independent event (a flipped token's MoE output, hence its next-
    layer routing and every later KV row, legitimately differs after it);
    every disagreeing row there must be an oracle near-tie."""
    bad = np.any(gtk != otk, axis=2)
    l0 = int(np.argmax(bad.any(axis=1)))
    assert np.all(omg[l0][bad[l0]] < ROUTER_FLIP_BOUND), (l0, omg[l0][bad[l0]])


def lockstep_prefill(s, os_, p):
    """Prefill device and oracle in the same <=16-token chunks (both sides
    chunk at 16; consecutive chunks overlap by the pending token) and compare
    every chunk's per-layer routing.  A disagreement is legal only where the
    oracle's own decision gap is below ROUTER_FLIP_BOUND; it is flagged and
    the prompt is skipped (its decodes legitimately diverge)."""
    pos = 0
    while pos < len(p) - 1:
        end = min(pos + 17, len(p))
        s.prefill(p[pos:end])
        os_.prefill(p[pos:end])
        otk, omg = os_.last_routing()
        T = otk.shape[1]
        gtk = s.tap("topk_id")[:, :T]
        if not np.array_equal(gtk, otk):
            assert_first_flip_is_near_tie(gtk, otk, omg)
            return False
        pos = end - 1
    return True


@pytest.mark.parametrize("K", [0, 1, 2, 3, 4])
def test_end_to_end_greedy_decode(tiny, K):
    """Lock-step decode, device vs independent oracle (no teacher forcing):
    drafts are the true greedy continuation with random corruptions, so
    every accepted count 0..K occurs.  Logits must agree within the stated
    tolerance; argmax rows, accepted counts, KV length, per-layer routing
    and union sizes must agree exactly.  Near-ties are handled explicitly:
    a routing disagreement is legal only where the oracle's decision gap is
    below ROUTER_FLIP_BOUND (then the decodes legitimately diverge and the
    comparison of that prompt stops), likewise an argmax disagreement only
    inside the observed logit error."""
    shape, m, om = tiny
    clean_steps = 0
    worst = 0.0
    for trial in range(32):  # prompts until enough clean lock-step verifies (near-tie flips end a prompt early)
        if clean_steps >= 40:
            break
        p = prompt(24, seed=100 * K + trial)
        truth = greedy_sequence(om, p, 60)
        s = cb.Session(m, max_ctx=512, k_max=8)
        s.enable_taps(True)  # eager path + routing / logits taps
        os_ = OracleSession(om, 512)
        if not lockstep_prefill(s, os_, p):
            s.close()
            continue  # flagged near-tie flip inside the prompt
        rng = np.random.default_rng(K + trial)
        pos = 0
        while pos + K < len(truth):
            drafts = np.array(truth[pos: pos + K], np.int32)
            for i in range(K):
                if rng.random() < 0.3:
                    drafts[i] = rng.integers(0, shape.vocab)
            g = s.verify(drafts)
            acc, am, lg, mg, us = os_.verify(drafts)
            T = K + 1
            otk, omg = os_.last_routing()
            gtk = s.tap("topk_id")[:, :T]
            if not np.array_equal(gtk, otk):
                assert_first_flip_is_near_tie(gtk, otk, omg)
                break  # flagged near-tie flip
            glog = s.tap("final_logits")[:T]
            err = float(np.abs(glog - lg).max())
            worst = max(worst, err)
            assert err <= LOGIT_ATOL + E2E_LOGIT_RTOL * np.abs(lg).max(), (trial, pos, err)
            if list(g.argmax[:T]) != list(am):
                assert np.all(mg[np.array(g.argmax[:T]) != am] <= 2 * err + MARGIN), (trial, pos)
                break  # flagged LM near-tie
            assert g.accepted == acc
            assert g.emitted == acc + 1
            assert g.cache_len == os_.cache_len
            assert list(s.union_sizes()) == list(us)
            assert list(g.tokens[: acc + 1]) == list(truth[pos: pos + acc + 1])
            pos += acc + 1
            clean_steps += 1
        s.close()
    print(f"K={K}: {clean_steps} clean lock-step verifies, worst |dlogit| = {worst:.2e}")
    assert clean_steps >= 12


def test_graph_replay_matches_eager(tiny):
    shape, m, om = tiny
    p = prompt(33, seed=5)
    res = []
    for taps in (False, True):
        s = cb.Session(m, max_ctx=256, k_max=8)
        if taps:
            s.enable_taps(True)
        s.prefill(p)
        outs = []
        for K in (3, 0, 8, 2):
            o = s.verify(np.arange(1, K + 1, dtype=np.int32) * 7)
            outs.append((o.accepted, list(o.argmax[: K + 1]), o.cache_len, list(s.union_sizes())))
        res.append(outs)
        s.close()
    assert res[0] == res[1]


def test_rejects_bad_requests(tiny):
    shape, m, om = tiny
    s = cb.Session(m, max_ctx=64, k_max=4)
    with pytest.raises(ValueError):
        s.verify(np.arange(5, dtype=np.int32))  # K > k_max
    with pytest.raises(ValueError):
        s.prefill(np.array([5000], np.int32))  # token out of range
    with pytest.raises(ValueError):
        s.set_baseline(0.0)
    s.close()


def test_kv_cache_bounds(tiny):
    """The session's KV capacity is a precondition, checked before anything
    is launched: a prefill beyond max_ctx is rejected (EINVAL); a committing
    verify or enqueue whose K+1 in-flight rows could take the committed
    length past max_ctx is refused (ERUNTIME, "full") and leaves the session
    unchanged, so no step ever appends past the KV slab."""
    shape, m, om = tiny
    s = cb.Session(m, max_ctx=48, k_max=4)
    with pytest.raises(ValueError):
        s.prefill(prompt(60, seed=2))
    s.prefill(prompt(40, seed=2))
    last = None
    with pytest.raises(cb.CascadeError, match="full"):
        for _ in range(64):
            last = s.verify(np.array([1, 2, 3, 4], np.int32))
            assert last.cache_len <= 48
    assert last is not None and last.cache_len > 40
    # the refused step changed nothing; a narrower step that fits still runs
    if last.cache_len + 1 <= 48:
        o = s.verify(np.array([], np.int32))
        assert o.cache_len == last.cache_len + 1
    # enqueue-only committing steps are bounded the same way (upper bound
    # T rows each until the next sync reads the exact length)
    s2 = cb.Session(m, max_ctx=64, k_max=4)
    s2.prefill(prompt(40, seed=2))
    n_ok = 0
    with pytest.raises(cb.CascadeError, match="full"):
        for _ in range(64):
            s2.enqueue(4, commit=True)
            n_ok += 1
    s2.sync()
    assert n_ok == (64 - 39) // 5
    try:
        o = s2.verify(np.array([], np.int32))
        assert 39 + n_ok < o.cache_len <= 64
    except cb.CascadeError as e:  # every enqueued draft accepted: exactly full
        assert "full" in str(e)
    s.close()
    s2.close()


def test_sessions_are_independent(tiny):
    """One session per request, each owning its state (the reference runs
    scenario cells in parallel, engine.hpp:427-459): two sessions on one
    model, interleaved on one thread and run concurrently from two host
    threads (each on its own stream), give exactly the results of running
    each alone."""
    import threading

    shape, m, om = tiny
    prompts = [prompt(30, seed=11), prompt(26, seed=12)]
    ks = [3, 0, 8, 2, 5, 1]

    def step(s, K):
        o = s.verify(np.arange(1, K + 1, dtype=np.int32) * 5)
        return (o.accepted, list(o.argmax[: K + 1]), o.cache_len, list(s.union_sizes()))

    def alone(p):
        s = cb.Session(m, max_ctx=256, k_max=8)
        s.prefill(p)
        out = [step(s, K) for K in ks]
        s.close()
        return out

    ref = [alone(p) for p in prompts]
    ss = [cb.Session(m, max_ctx=256, k_max=8) for _ in prompts]
    for s, p in zip(ss, prompts):
        s.prefill(p)
    inter = [[], []]
    for K in ks:
        for i, s in enumerate(ss):
            inter[i].append(step(s, K))
    for s in ss:
        s.close()
    assert inter == ref

    conc = [None, None]

    def worker(i):
        conc[i] = alone(prompts[i])

    th = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert conc == ref


def test_utility_and_cost_breakdown(tiny):
    """CostBreakdown parts sum to total (expert_model_test.cpp:120-133) and
    the on-device utility equals emitted * t_base / total."""
    shape, m, om = tiny
    s = cb.Session(m, max_ctx=256, k_max=8)
    s.prefill(prompt(20, seed=9))
    s.set_baseline(1.0e6)
    o = s.verify(np.array([1, 2, 3], np.int32), draft_ns=1234.0)
    assert o.total == pytest.approx(o.attention_time + o.expert_time + o.draft_time + o.sampling_time, rel=1e-12)
    assert o.draft_time == 1234.0
    assert o.attention_time > 0 and o.expert_time > 0 and o.sampling_time > 0
    assert o.utility == pytest.approx(o.emitted * 1.0e6 / o.total, rel=1e-12)
    assert shape.top_k <= o.active_experts_per_layer <= shape.experts_per_layer
    s.close()


def test_expert_parallel_single_rank_nccl_in_graph(tiny):
    """The expert-parallel build (cascade_model_create_ep) on one rank: the
    captured step graph carries the per-layer ncclAllReduce of the expert
    outputs; with one rank it must reproduce the non-EP logits bitwise
    (adding exact zeros / a single contribution is exact)."""
    shape, m, _ = tiny
    uid = cb.ep_unique_id()
    mep = cb.Model(shape, cb.TINY_SEED, device=0, ep_rank=0, ep_size=1, nccl_id=uid)
    rng = np.random.default_rng(3)
    prompt = rng.integers(0, shape.vocab, 40).astype(np.int32)
    drafts = rng.integers(0, shape.vocab, 5).astype(np.int32)
    outs = []
    for model in (m, mep):
        s = cb.Session(model, max_ctx=256, k_max=8)
        s.prefill(prompt)
        o = s.verify(drafts)
        outs.append((list(o.argmax[:6]), o.accepted, list(s.union_sizes())))
        s.close()
    mep.close()
    assert outs[0] == outs[1]


def test_expert_shards_partition_the_moe_output(tiny, monkeypatch):
    """Expert parallelism on one GPU: with CASCADE_EP_NOCOMM=1 each shard
    model (rank r of G) runs without the all-reduce, so its layer-0 MoE
    output is the sum over its own experts only (the others contribute exact
    zeros).  The shards' outputs must add up to the full model's, and their
    union sizes (the global distinct-expert count) must agree with it."""
    shape, m, _ = tiny
    monkeypatch.setenv("CASCADE_EP_NOCOMM", "1")
    rng = np.random.default_rng(11)
    prompt = rng.integers(0, shape.vocab, 30).astype(np.int32)
    drafts = rng.integers(0, shape.vocab, 4).astype(np.int32)

    def layer0_moe(model):
        s = cb.Session(model, max_ctx=128, k_max=8)
        s.enable_taps(True)
        s.prefill(prompt)
        s.verify(drafts)
        out = s.tap("moe_out")[0, :5].copy()
        us = list(s.union_sizes())
        s.close()
        return out, us

    full, us_full = layer0_moe(m)
    for G in (2, 4):
        parts = []
        for r in range(G):
            mr = cb.Model(shape, cb.TINY_SEED, device=0, ep_rank=r, ep_size=G, nccl_id=bytes(128))
            out, us = layer0_moe(mr)
            mr.close()
            assert us[0] == us_full[0]
            parts.append(out)
        total = np.sum(parts, axis=0)
        assert np.allclose(total, full, rtol=1e-5, atol=1e-6), float(np.abs(total - full).max())
        assert sum(np.abs(p).max() > 0 for p in parts) >= 2  # the work really is split across shards
