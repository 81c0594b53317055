"""Concurrent sessions on one GPU with the fused expert FFN.

The fused FFN (expert_ffn_kernel) spin-waits on gate/up tiles produced by
other CTAs of its grid, so its whole grid must be co-resident.  It is
launched cooperatively (co-residency guaranteed by the driver) and only
used when 2 CTAs per SM fit (otherwise the two-launch path runs).  Two
sessions on their own streams, driven from two host threads (ctypes drops
the GIL), replay Mixtral-width step graphs concurrently many times: no
trap, no hang, and every session's results equal running it alone
(engine.hpp:427-459 runs scenario cells concurrently, each owning its
state).
"""

import threading

import numpy as np
import pytest

import paper_2506_20675_b200 as cb

pytestmark = pytest.mark.gpu


def test_fused_ffn_concurrent_sessions():
    shape = cb.preset("mixtral").with_layers(2)
    m = cb.Model(shape, 5)
    rng = np.random.default_rng(5)
    prompts = [rng.integers(0, shape.vocab, 80).astype(np.int32) for _ in range(2)]
    drafts = [rng.integers(0, shape.vocab, 8).astype(np.int32) for _ in range(2)]
    Ks = [0, 8, 3, 5, 1]

    def make(i):
        s = cb.Session(m, max_ctx=256, k_max=8)
        s.prefill(prompts[i])
        return s

    def finish(s, i):
        o = s.verify(drafts[i])
        return (o.accepted, list(o.argmax[:9]), o.cache_len, list(s.union_sizes()))

    alone = []
    for i in range(2):
        s = make(i)
        # the fused single-launch FFN is the path under test: 1 + 7 L + 2 kernels
        assert s.kernel_count(8) == 1 + 7 * shape.num_layers + 2
        alone.append(finish(s, i))
        s.close()

    errors = []
    results = [None, None]
    ss = [make(i) for i in range(2)]
    start = threading.Barrier(2)

    def worker(i):
        try:
            s = ss[i]
            start.wait()
            for _ in range(40):
                for K in Ks:
                    s.enqueue(K, commit=False)
            s.sync()
            results[i] = finish(s, i)
        except Exception as e:  # surfaced below
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), "concurrent sessions hung"
    assert not errors, errors
    assert results == alone
    for s in ss:
        s.close()
    m.close()
