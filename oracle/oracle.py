"""ctypes wrapper of the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs, as the checker.  The product path
(paper_2506_20675_b200/libcascade.so) never loads it.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            import subprocess

            subprocess.check_call(["make", "-s", "-C", _HERE, "liboracle.so"])
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        I32P = ctypes.POINTER(ctypes.c_int32)
        U16P = ctypes.POINTER(ctypes.c_uint16)
        DP = ctypes.POINTER(ctypes.c_double)
        FP = ctypes.POINTER(ctypes.c_float)
        c = ctypes.c_int
        sig = {
            "orc_model_create": (P, [P, ctypes.c_uint64, c]),
            "orc_model_destroy": (None, [P]),
            "orc_model_drop_cache": (None, [P]),
            "orc_cached_bytes": (ctypes.c_uint64, [P]),
            "orc_tensor": (c, [P, c, c, c, c, c, U16P]),
            "orc_prepare_layer": (c, [P, c, I32P, c]),
            "orc_rmsnorm": (c, [P, c, c, FP, c, U16P]),
            "orc_router": (c, [P, c, U16P, c, DP, I32P, DP, DP, DP]),
            "orc_union": (c, [I32P, c, c, I32P]),
            "orc_moe": (c, [P, c, U16P, c, I32P, DP, DP, DP]),
            "orc_attention": (c, [P, c, FP, c, c, U16P, U16P, DP, U16P, U16P]),
            "orc_lm_head": (c, [P, U16P, c, DP, I32P, DP]),
            "orc_greedy_accept": (c, [I32P, I32P, c, I32P]),
            "orc_session_create": (P, [P, c]),
            "orc_session_destroy": (None, [P]),
            "orc_prefill": (c, [P, I32P, c]),
            "orc_verify": (c, [P, I32P, c, DP, I32P, DP, I32P]),
            "orc_cache_len": (c, [P]),
            "orc_min_router_margin": (ctypes.c_double, [P, c]),
            "orc_last_routing": (c, [P, I32P, DP]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t)) if a is not None else None


def _chk(rc):
    if rc < 0:
        raise RuntimeError(f"oracle call failed ({rc})")
    return rc


class OracleModel:
    def __init__(self, shape, seed, nthreads=None):
        self.shape = shape
        self._g = shape.to_c()
        self.nthreads = nthreads or os.cpu_count() or 1
        self.h = lib().orc_model_create(ctypes.byref(self._g), seed, self.nthreads)
        if not self.h:
            raise ValueError("oracle rejected the geometry")

    def __del__(self):
        try:
            if self.h:
                lib().orc_model_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def drop_cache(self):
        lib().orc_model_drop_cache(self.h)

    def tensor(self, kind, layer, expert, row0, nrows, cols):
        out = np.zeros((nrows, cols), np.uint16)
        _chk(lib().orc_tensor(self.h, kind, layer, expert, row0, nrows, _p(out, ctypes.c_uint16)))
        return out

    def prepare_layer(self, layer, experts):
        e = np.ascontiguousarray(experts, np.int32)
        _chk(lib().orc_prepare_layer(self.h, layer, _p(e, ctypes.c_int32), len(e)))

    def rmsnorm(self, kind, layer, x):
        x = np.ascontiguousarray(x, np.float32)
        T = x.shape[0]
        out = np.zeros((T, self.shape.d_model), np.uint16)
        _chk(lib().orc_rmsnorm(self.h, kind, layer, _p(x, ctypes.c_float), T, _p(out, ctypes.c_uint16)))
        return out

    def router(self, layer, xn):
        xn = np.ascontiguousarray(xn, np.uint16)
        T = xn.shape[0]
        E, k = self.shape.experts_per_layer, self.shape.top_k
        logits = np.zeros((T, E + 1))
        topk = np.zeros((T, k), np.int32)
        topw = np.zeros((T, k))
        gsh = np.zeros(T)
        margin = np.zeros(T)
        _chk(lib().orc_router(self.h, layer, _p(xn, ctypes.c_uint16), T, _p(logits, ctypes.c_double),
                              _p(topk, ctypes.c_int32), _p(topw, ctypes.c_double), _p(gsh, ctypes.c_double),
                              _p(margin, ctypes.c_double)))
        return logits, topk, topw, gsh, margin

    def moe(self, layer, xn, topk, topw, gsh):
        xn = np.ascontiguousarray(xn, np.uint16)
        T = xn.shape[0]
        topk = np.ascontiguousarray(topk, np.int32)
        topw = np.ascontiguousarray(topw, np.float64)
        gsh = np.ascontiguousarray(gsh, np.float64)
        out = np.zeros((T, self.shape.d_model))
        _chk(lib().orc_moe(self.h, layer, _p(xn, ctypes.c_uint16), T, _p(topk, ctypes.c_int32),
                           _p(topw, ctypes.c_double), _p(gsh, ctypes.c_double), _p(out, ctypes.c_double)))
        return out

    def attention(self, layer, x, ctx, kcache=None, vcache=None):
        x = np.ascontiguousarray(x, np.float32)
        T = x.shape[0]
        s = self.shape
        out = np.zeros((T, s.d_model))
        kn = np.zeros((s.n_kv_heads, T, s.head_dim), np.uint16)
        vn = np.zeros((s.n_kv_heads, T, s.head_dim), np.uint16)
        kc = np.ascontiguousarray(kcache, np.uint16) if kcache is not None else None
        vc = np.ascontiguousarray(vcache, np.uint16) if vcache is not None else None
        _chk(lib().orc_attention(self.h, layer, _p(x, ctypes.c_float), T, ctx, _p(kc, ctypes.c_uint16),
                                 _p(vc, ctypes.c_uint16), _p(out, ctypes.c_double), _p(kn, ctypes.c_uint16),
                                 _p(vn, ctypes.c_uint16)))
        return out, kn, vn

    def lm_head(self, xn):
        xn = np.ascontiguousarray(xn, np.uint16)
        T = xn.shape[0]
        logits = np.zeros((T, self.shape.vocab))
        am = np.zeros(T, np.int32)
        mg = np.zeros(T)
        _chk(lib().orc_lm_head(self.h, _p(xn, ctypes.c_uint16), T, _p(logits, ctypes.c_double),
                               _p(am, ctypes.c_int32), _p(mg, ctypes.c_double)))
        return logits, am, mg


def union(topk):
    topk = np.ascontiguousarray(topk, np.int32)
    T, k = topk.shape
    out = np.zeros(128, np.int32)
    n = lib().orc_union(_p(topk, ctypes.c_int32), T, k, _p(out, ctypes.c_int32))
    return out[:n]


def greedy_accept(argmax, drafts):
    a = np.ascontiguousarray(argmax, np.int32)
    d = np.ascontiguousarray(drafts, np.int32)
    K = len(d)
    em = np.zeros(K + 1, np.int32)
    acc = lib().orc_greedy_accept(_p(a, ctypes.c_int32), _p(d, ctypes.c_int32) if K else None, K,
                                  _p(em, ctypes.c_int32))
    return acc, em[: acc + 1]


class OracleSession:
    def __init__(self, model: OracleModel, max_ctx=2048):
        self.model = model
        self.h = lib().orc_session_create(model.h, max_ctx)

    def __del__(self):
        try:
            if self.h:
                lib().orc_session_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def prefill(self, prompt):
        p = np.ascontiguousarray(prompt, np.int32)
        _chk(lib().orc_prefill(self.h, _p(p, ctypes.c_int32), len(p)))

    def verify(self, drafts):
        d = np.ascontiguousarray(drafts, np.int32)
        K = len(d)
        T = K + 1
        s = self.model.shape
        logits = np.zeros((T, s.vocab))
        am = np.zeros(T, np.int32)
        mg = np.zeros(T)
        us = np.zeros(s.num_layers, np.int32)
        acc = _chk(lib().orc_verify(self.h, _p(d, ctypes.c_int32) if K else None, K, _p(logits, ctypes.c_double),
                                    _p(am, ctypes.c_int32), _p(mg, ctypes.c_double), _p(us, ctypes.c_int32)))
        return acc, am, logits, mg, us

    def last_routing(self):
        s = self.model.shape
        tk = np.zeros((s.num_layers * 64, s.top_k), np.int32)
        mg = np.zeros(s.num_layers * 64)
        T = lib().orc_last_routing(self.h, _p(tk, ctypes.c_int32), _p(mg, ctypes.c_double))
        return tk[: s.num_layers * T].reshape(s.num_layers, T, s.top_k), mg[: s.num_layers * T].reshape(s.num_layers, T)

    def min_router_margin(self, reset=True):
        return lib().orc_min_router_margin(self.h, 1 if reset else 0)

    @property
    def cache_len(self):
        return lib().orc_cache_len(self.h)
