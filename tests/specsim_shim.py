"""ctypes access to oracle/specsim_shim.cpp builds (test infrastructure).

`load("ours")` -> oracle/libspecsim_ours.so (this repo's include/specsim)
`load("ref")`  -> oracle/_ref/libspecsim_ref.so (the unmodified reference)
Both expose the same functions, so every scenario below runs identically
against either build.
"""

import ctypes
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PATHS = {
    "ours": os.path.join(ROOT, "oracle", "libspecsim_ours.so"),
    "ref": os.path.join(ROOT, "oracle", "_ref", "libspecsim_ref.so"),
}

I32P = ctypes.POINTER(ctypes.c_int32)
DP = ctypes.POINTER(ctypes.c_double)
LP = ctypes.POINTER(ctypes.c_long)


def available(which):
    return os.path.exists(PATHS[which])


class Shim:
    def __init__(self, which):
        L = ctypes.CDLL(PATHS[which])
        c = ctypes.c_int
        sig = {
            "ref_expected_unique_experts": (ctypes.c_double, [c, c, c]),
            "ref_sample_active_experts": (c, [c, c, c, ctypes.c_double, c, ctypes.c_uint64, c, DP]),
            "ref_iteration_cost": (c, [ctypes.c_char_p, ctypes.c_char_p, c, ctypes.c_uint64, c, DP]),
            "ref_sample_accepted": (c, [ctypes.c_double, c, ctypes.c_uint64, c, I32P]),
            "ref_trace_replay": (c, [c, c, c]),
            "ref_drive_controller": (c, [I32P, ctypes.c_double, DP, ctypes.c_long, DP, ctypes.c_long, c,
                                         ctypes.c_double, ctypes.c_uint64, I32P, I32P, LP, LP, DP, I32P, I32P,
                                         ctypes.POINTER(c)]),
            "ref_run_request": (c, [ctypes.c_double, ctypes.c_double, c, c, ctypes.c_char_p, ctypes.c_char_p,
                                    ctypes.c_uint64, DP]),
            "ref_window_utility": (c, [c, ctypes.c_double, c, I32P, I32P, DP, I32P, DP]),
            "ref_controller_replay": (c, [I32P, ctypes.c_double, c, I32P, DP, I32P, I32P]),
            "ref_trace_load": (ctypes.c_long, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_long]),
            "ref_trace_replay_request": (ctypes.c_long, [ctypes.c_char_p, ctypes.c_long, c, ctypes.c_uint64, DP,
                                                         I32P, ctypes.c_long]),
            "ref_write_telemetry": (c, [ctypes.c_char_p, c, DP]),
            "ref_scenario_report": (c, [ctypes.c_char_p, ctypes.c_long, ctypes.c_char_p]),
            "ref_load_cells": (ctypes.c_long, [ctypes.c_char_p, DP, ctypes.c_long]),
            "ref_scenario_digest": (ctypes.c_long, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_long]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype = r
            f.argtypes = a
        self.L = L

    def expected_unique_experts(self, E, k, T):
        return self.L.ref_expected_unique_experts(E, k, T)

    def sample_active_experts(self, E, k, S, aff, tokens, seed, n):
        out = np.zeros(n)
        assert self.L.ref_sample_active_experts(E, k, S, aff, tokens, seed, n, out.ctypes.data_as(DP)) == 0
        return out

    def iteration_cost(self, preset, draft, k, seed, n):
        out = np.zeros((n, 6))
        assert self.L.ref_iteration_cost(preset.encode(), draft.encode(), k, seed, n, out.ctypes.data_as(DP)) == 0
        return out

    def sample_accepted(self, p, k, seed, n):
        out = np.zeros(n, np.int32)
        assert self.L.ref_sample_accepted(p, k, seed, n, out.ctypes.data_as(I32P)) == 0
        return out

    def trace_replay(self, k_offered, accepted, k):
        return self.L.ref_trace_replay(k_offered, accepted, k)

    def drive(self, cfg, util, max_iters, stop_after_sets=0, noise=0.0, noise_seed=0, switch_iter=-1, util2=None):
        ci = np.array([cfg[k] for k in ("t_trial", "max_trials", "s_set", "s_cap", "k_max", "k_start",
                                          "refresh", "probe_len", "backoff")], np.int32)
        u = np.zeros(16)
        u[: len(util)] = util
        u2 = np.zeros(16)
        if util2 is not None:
            u2[: len(util2)] = util2
        kseq = np.zeros(max_iters, np.int32)
        tags = np.zeros(max_iters, np.int32)
        n_it, test_it = ctypes.c_long(), ctypes.c_long()
        tot = ctypes.c_double()
        set_k = np.zeros(max_iters, np.int32)
        set_len = np.zeros(max_iters, np.int32)
        n_sets = ctypes.c_int()
        rc = self.L.ref_drive_controller(ci.ctypes.data_as(I32P), cfg["band"], u.ctypes.data_as(DP), switch_iter,
                                         u2.ctypes.data_as(DP), max_iters, stop_after_sets, noise, noise_seed,
                                         kseq.ctypes.data_as(I32P), tags.ctypes.data_as(I32P), ctypes.byref(n_it),
                                         ctypes.byref(test_it), ctypes.byref(tot), set_k.ctypes.data_as(I32P),
                                         set_len.ctypes.data_as(I32P), ctypes.byref(n_sets))
        assert rc == 0
        n = n_it.value
        return {"k": kseq[:n].tolist(), "tags": tags[:n].tolist(), "test_iters": test_it.value,
                "total_time": tot.value, "sets": list(zip(set_k[: n_sets.value].tolist(),
                                                           set_len[: n_sets.value].tolist()))}

    def run_request(self, p, aff, out_len, policy, preset, draft, seed):
        out = np.zeros(8)
        assert self.L.ref_run_request(p, aff, out_len, policy, preset.encode(), draft.encode(), seed,
                                      out.ctypes.data_as(DP)) == 0
        return out

    def window_utility(self, window, t_base, k, tokens, total, tag):
        k = np.ascontiguousarray(k, np.int32)
        tokens = np.ascontiguousarray(tokens, np.int32)
        total = np.ascontiguousarray(total, np.float64)
        tag = np.ascontiguousarray(tag, np.int32)
        out = np.zeros(3)
        rc = self.L.ref_window_utility(window, t_base, len(k), k.ctypes.data_as(I32P), tokens.ctypes.data_as(I32P),
                                       total.ctypes.data_as(DP), tag.ctypes.data_as(I32P), out.ctypes.data_as(DP))
        assert rc == 0
        return out

    def controller_replay(self, cfg, tokens, total):
        ci = np.array([cfg[k] for k in ("t_trial", "max_trials", "s_set", "s_cap", "k_max", "k_start",
                                          "refresh", "probe_len", "backoff")], np.int32)
        tokens = np.ascontiguousarray(tokens, np.int32)
        total = np.ascontiguousarray(total, np.float64)
        n = len(tokens)
        k = np.zeros(n, np.int32)
        tg = np.zeros(n, np.int32)
        assert self.L.ref_controller_replay(ci.ctypes.data_as(I32P), cfg["band"], n, tokens.ctypes.data_as(I32P),
                                            total.ctypes.data_as(DP), k.ctypes.data_as(I32P),
                                            tg.ctypes.data_as(I32P)) == 0
        return k, tg

    # ---- report / trace / scenario interop
    def trace_load(self, path, cap=100000):
        out = np.zeros((cap, 4), np.int64)
        n = self.L.ref_trace_load(str(path).encode(), out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), cap)
        assert n >= 0, f"trace load failed: {path}"
        return out[:n]

    def trace_replay_request(self, path, request_id, policy, seed=1, cap=100000):
        out = np.zeros(8)
        em = np.zeros(cap, np.int32)
        n = self.L.ref_trace_replay_request(str(path).encode(), request_id, policy, seed, out.ctypes.data_as(DP),
                                            em.ctypes.data_as(I32P), cap)
        assert n >= 0
        return out, em[:n]

    def write_telemetry(self, path, rows):
        rows = np.ascontiguousarray(rows, np.float64)
        assert self.L.ref_write_telemetry(str(path).encode(), len(rows), rows.ctypes.data_as(DP)) == 0

    def scenario_report(self, scenario, tokens, out_dir):
        assert self.L.ref_scenario_report(str(scenario).encode(), tokens, str(out_dir).encode()) == 0

    def load_cells(self, path, cap=4096):
        out = np.zeros((cap, 3))
        n = self.L.ref_load_cells(str(path).encode(), out.ctypes.data_as(DP), cap)
        assert n >= 0, f"load_cells failed: {path}"
        return out[:n]

    def scenario_digest(self, path):
        buf = ctypes.create_string_buffer(1 << 16)
        n = self.L.ref_scenario_digest(str(path).encode(), buf, 1 << 16)
        return None if n < 0 else buf.value.decode()


DEFAULT_CFG = {"t_trial": 4, "max_trials": 4, "s_set": 16, "s_cap": 256, "k_max": 3, "k_start": 3, "refresh": 100,
               "probe_len": 4, "backoff": 1, "band": 0.10}


def cfg(**kw):
    c = dict(DEFAULT_CFG)
    c.update(kw)
    return c
