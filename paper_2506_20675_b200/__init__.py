"""B200-native MoE verification step (arXiv 2506.20675, "Cascade") — host mirror.

The product is the C ABI in ``include/cascade.h`` implemented by
``paper_2506_20675_b200/libcascade.so`` (hand-written sm_100a CUDA).  This
module is the thin Python host mirror of that boundary, used by the tests and
``bench.py``; it mirrors the reference's error behaviour
(``std::invalid_argument`` -> ``ValueError``, ``MissingBaselineError``) and its
geometry vocabulary (``ExpertConfig``: num_layers, experts_per_layer, top_k,
shared_experts — proj/include/specsim/expert_model.hpp:27-51).

There is no CPU fallback: importing works anywhere, but every call that needs
the library raises if ``libcascade.so`` is missing, and model creation fails
loudly without a B200.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field, asdict
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CASCADE_LIB_PATH") or os.path.join(_HERE, "libcascade.so")  # A/B builds only

MAX_TOKENS = 16
MAX_K = MAX_TOKENS - 1

# tensor kinds (include/cascade_weights.h)
T_EMBED, T_ATTN_NORM, T_FFN_NORM, T_WQ, T_WK, T_WV, T_WO = 1, 2, 3, 4, 5, 6, 7
T_ROUTER, T_SHARED_GATE, T_W_GATE, T_W_UP, T_W_DOWN, T_FINAL_NORM, T_LM_HEAD = 8, 9, 10, 11, 12, 13, 14


# ----------------------------------------------------------------- errors
class CascadeError(RuntimeError):
    """Device or runtime failure (CASCADE_ECUDA / CASCADE_ERUNTIME)."""


class MissingBaselineError(RuntimeError):
    """utility.hpp:52-55 — baseline requested before any k=0 probes."""


def _raise(code: int, msg: str):
    if code == 1:
        raise ValueError(msg)
    if code == 4:
        raise MissingBaselineError(msg)
    raise CascadeError(msg)


# ----------------------------------------------------------------- C structs
class Geometry(ctypes.Structure):
    _fields_ = [
        ("num_layers", ctypes.c_int32),
        ("experts_per_layer", ctypes.c_int32),
        ("top_k", ctypes.c_int32),
        ("shared_experts", ctypes.c_int32),
        ("d_model", ctypes.c_int32),
        ("d_ff", ctypes.c_int32),
        ("n_heads", ctypes.c_int32),
        ("n_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("vocab", ctypes.c_int32),
        ("renormalize_topk", ctypes.c_int32),
        ("shared_gate", ctypes.c_int32),
        ("rope_theta", ctypes.c_float),
        ("norm_eps", ctypes.c_float),
        ("router_scale", ctypes.c_float),
        ("reserved", ctypes.c_int32 * 5),
    ]


class VerifyOut(ctypes.Structure):
    _fields_ = [
        ("accepted", ctypes.c_int32),
        ("emitted", ctypes.c_int32),
        ("n_tokens", ctypes.c_int32),
        ("cache_len", ctypes.c_int32),
        ("tokens", ctypes.c_int32 * MAX_TOKENS),
        ("argmax", ctypes.c_int32 * MAX_TOKENS),
        ("attention_time", ctypes.c_double),
        ("expert_time", ctypes.c_double),
        ("draft_time", ctypes.c_double),
        ("sampling_time", ctypes.c_double),
        ("active_experts_per_layer", ctypes.c_double),
        ("total", ctypes.c_double),
        ("utility", ctypes.c_double),
        ("verify_ns", ctypes.c_double),
    ]


class DecodeCfg(ctypes.Structure):
    _fields_ = [
        ("policy", ctypes.c_int32),
        ("max_new", ctypes.c_int32),
        ("ngram_n", ctypes.c_int32),
        ("t_trial", ctypes.c_int32),
        ("max_trials", ctypes.c_int32),
        ("s_set", ctypes.c_int32),
        ("s_cap", ctypes.c_int32),
        ("k_max", ctypes.c_int32),
        ("k_start", ctypes.c_int32),
        ("convergence_band", ctypes.c_double),
        ("baseline_refresh_interval", ctypes.c_int32),
        ("baseline_probe_len", ctypes.c_int32),
        ("backoff_enabled", ctypes.c_int32),
        ("injected_cost", ctypes.c_int32),
        ("cost_by_k", ctypes.c_double * MAX_TOKENS),
        ("drafter", ctypes.c_int32),
        ("n_replay", ctypes.c_int32),
        ("replay_tokens", ctypes.POINTER(ctypes.c_int32)),
        ("replay_p", ctypes.c_double),
        ("replay_seed", ctypes.c_uint64),
        ("telemetry_csv", ctypes.c_char_p),
        ("trace_path", ctypes.c_char_p),
        ("request_id", ctypes.c_int64),
        ("trace_append", ctypes.c_int32),
        ("reserved_cfg", ctypes.c_int32),
    ]


class CellCfg(ctypes.Structure):
    _fields_ = [
        ("policy", ctypes.c_int32),
        ("t_trial", ctypes.c_int32),
        ("max_trials", ctypes.c_int32),
        ("s_set", ctypes.c_int32),
        ("s_cap", ctypes.c_int32),
        ("k_max", ctypes.c_int32),
        ("k_start", ctypes.c_int32),
        ("convergence_band", ctypes.c_double),
        ("baseline_refresh_interval", ctypes.c_int32),
        ("baseline_probe_len", ctypes.c_int32),
        ("backoff_enabled", ctypes.c_int32),
        ("n_profiles", ctypes.c_int32),
        ("share", ctypes.c_double * 4),
        ("n_phases", ctypes.c_int32 * 4),
        ("accept_p", (ctypes.c_double * 4) * 4),
        ("mean_duration", (ctypes.c_double * 4) * 4),
        ("out_len_lo", ctypes.c_int32 * 4),
        ("out_len_hi", ctypes.c_int32 * 4),
        ("tokens_per_cell", ctypes.c_int64),
        ("prompt_len", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
    ]


class CellResult(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("requests", "iterations", "tokens")] + \
        [(n, ctypes.c_double) for n in ("total_time", "t_base", "tpot", "etr", "cost", "utility", "utility_hmean")]


# ----------------------------------------------------------------- geometry presets
@dataclass
class ModelShape:
    """ExpertConfig routing fields + tensor shape (public model configs)."""

    name: str
    num_layers: int
    experts_per_layer: int
    top_k: int
    shared_experts: int
    d_model: int
    d_ff: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    vocab: int
    renormalize_topk: int = 1
    shared_gate: int = 0
    rope_theta: float = 1e6
    norm_eps: float = 1e-5
    router_scale: float = 4.0

    def to_c(self) -> Geometry:
        g = Geometry()
        for f in Geometry._fields_:
            if f[0] == "reserved":
                continue
            setattr(g, f[0], getattr(self, f[0]))
        return g

    def with_layers(self, n: int) -> "ModelShape":
        d = asdict(self)
        d["num_layers"] = n
        d["name"] = f"{self.name}-L{n}"
        return ModelShape(**d)

    # HBM bytes (algorithmic) of one verify step, DESIGN.md §4
    def step_bytes(self, union_sizes, ctx: int, T: int) -> dict:
        d, f = self.d_model, self.d_ff
        hq = self.n_heads * self.head_dim
        kvd = self.n_kv_heads * self.head_dim
        expert = 3 * d * f * 2
        out = {"experts": 0, "dense": 0, "kv": 0, "head": 0}
        for u in union_sizes:
            u = float(u)  # a mean U over draws is fractional: never truncate it
            out["experts"] += (u + self.shared_experts) * expert
            out["dense"] += (d * (hq + 2 * kvd) + hq * d) * 2 + (self.experts_per_layer + self.shared_gate) * d * 2 + 2 * d * 2
            out["kv"] += ctx * 2 * kvd * 2 + T * 2 * kvd * 2
        out["head"] = self.vocab * d * 2 + d * 2
        out["total"] = sum(out.values())
        return out


PRESETS = {
    # SURVEY.md §8(d) config 1 (authored: the reference has no tiny MoE fixture)
    "tiny": ModelShape("tiny", 4, 8, 2, 0, 256, 512, 8, 2, 32, 1024, 1, 0, 1e6, 1e-5, 4.0),
    # config 2: Mixtral-8x7B shape
    "mixtral": ModelShape("mixtral", 32, 8, 2, 0, 4096, 14336, 32, 8, 128, 32000, 1, 0, 1e6, 1e-5, 4.0),
    # config 3: OLMoE-1B-7B shape (softmax top-8, no renormalisation)
    "olmoe": ModelShape("olmoe", 16, 64, 8, 0, 2048, 1024, 16, 16, 128, 50304, 0, 0, 1e4, 1e-5, 4.0),
    # config 4: Qwen1.5-MoE-A2.7B: 60 routed top-4 + shared expert (5632 = 4 blocks of 1408,
    # the reference counts it as shared_experts=4, expert_model.hpp:192-193), sigmoid gate
    "qwen15": ModelShape("qwen15", 24, 60, 4, 4, 2048, 1408, 16, 16, 128, 151936, 0, 1, 1e6, 1e-6, 4.0),
    # config 5: Mixtral-8x22B shape (281 GB bf16: expert-parallel only)
    "mixtral8x22b": ModelShape("mixtral8x22b", 56, 8, 2, 0, 6144, 16384, 48, 8, 128, 32768, 1, 0, 1e6, 1e-5, 4.0),
}

TINY_SEED = 0x5EED


def preset(name: str) -> ModelShape:
    if name not in PRESETS:
        raise ValueError(f"unknown model preset: {name}")
    return PRESETS[name]


# ----------------------------------------------------------------- library
_LIB = None


def lib() -> ctypes.CDLL:
    """Loads libcascade.so (in-tree build).  Raises if it was not built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    i32, i64, u64, dbl, szt = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_size_t
    sig = {
        "cascade_last_error": (szt, [ctypes.c_char_p, szt]),
        "cascade_geometry_validate": (ctypes.c_int, [ctypes.POINTER(Geometry)]),
        "cascade_model_bytes": (ctypes.c_int, [ctypes.POINTER(Geometry), ctypes.c_int, ctypes.c_int, ctypes.POINTER(u64)]),
        "cascade_model_create": (ctypes.c_int, [ctypes.POINTER(Geometry), u64, ctypes.c_int, ctypes.POINTER(P)]),
        "cascade_model_create_ep": (
            ctypes.c_int,
            [ctypes.POINTER(Geometry), u64, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, ctypes.POINTER(P)],
        ),
        "cascade_model_destroy": (ctypes.c_int, [P]),
        "cascade_ep_unique_id": (ctypes.c_int, [P, szt]),
        "cascade_session_create": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, P, ctypes.POINTER(P)]),
        "cascade_session_destroy": (ctypes.c_int, [P]),
        "cascade_prefill": (ctypes.c_int, [P, ctypes.POINTER(i32), ctypes.c_int]),
        "cascade_session_reset": (ctypes.c_int, [P]),
        "cascade_set_baseline": (ctypes.c_int, [P, dbl]),
        "cascade_verify": (ctypes.c_int, [P, ctypes.POINTER(i32), ctypes.c_int, dbl, ctypes.POINTER(VerifyOut)]),
        "cascade_last_union_sizes": (ctypes.c_int, [P, ctypes.POINTER(i32), ctypes.c_int]),
        "cascade_verify_enqueue": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int]),
        "cascade_sync": (ctypes.c_int, [P]),
        "cascade_session_stream": (P, [P]),
        "cascade_step_kernel_count": (ctypes.c_int, [P, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
        "cascade_step_trace": (
            ctypes.c_int,
            [P, ctypes.c_int, ctypes.POINTER(dbl), ctypes.POINTER(i32), ctypes.c_int, ctypes.POINTER(ctypes.c_int)],
        ),
        "cascade_step_cta_trace": (
            ctypes.c_int,
            [P, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(i32), ctypes.c_int,
             ctypes.POINTER(ctypes.c_int)],
        ),
        "cascade_profile_step": (
            ctypes.c_int,
            [P, ctypes.c_int, ctypes.POINTER(dbl), ctypes.POINTER(i32), ctypes.c_int, ctypes.POINTER(ctypes.c_int)],
        ),
        "cascade_enable_taps": (ctypes.c_int, [P, ctypes.c_int]),
        "cascade_set_batch_invariant": (ctypes.c_int, [P, ctypes.c_int]),
        "cascade_run_cell": (ctypes.c_int, [P, ctypes.POINTER(CellCfg), ctypes.POINTER(CellResult)]),
        "cascade_read_tap": (ctypes.c_int, [P, ctypes.c_int, P, szt]),
        "cascade_read_weight": (
            ctypes.c_int,
            [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_uint16)],
        ),
        "cascade_read_kv": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_uint16)]),
        "cascade_decode": (
            ctypes.c_int,
            [
                P,
                ctypes.POINTER(i32),
                ctypes.c_int,
                ctypes.POINTER(DecodeCfg),
                ctypes.POINTER(i32),
                ctypes.POINTER(i32),
                ctypes.POINTER(dbl),
                i32,
                ctypes.POINTER(i32),
            ],
        ),
        "cascade_build_info": (ctypes.c_char_p, []),
        "cascade_session_geometry": (ctypes.c_int, [P, ctypes.POINTER(Geometry)]),
        "cascade_replay_trace": (
            ctypes.c_int,
            [P, ctypes.c_char_p, ctypes.POINTER(DecodeCfg), i32, u64, ctypes.c_char_p, ctypes.POINTER(CellResult),
             ctypes.POINTER(i64)],
        ),
        "cascade_run_scenario": (
            ctypes.c_int,
            [ctypes.POINTER(P), ctypes.c_int, ctypes.c_char_p, ctypes.c_char_p, i64, i32, ctypes.c_char_p,
             ctypes.POINTER(i32)],
        ),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = L
    return L


def last_error() -> str:
    buf = ctypes.create_string_buffer(4096)
    lib().cascade_last_error(buf, 4096)
    return buf.value.decode()


def _check(rc: int):
    if rc != 0:
        _raise(rc, last_error())


def _i32p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


# ----------------------------------------------------------------- objects
class Model:
    """Random-init weights on one B200 (or one expert-parallel shard)."""

    def __init__(self, shape: ModelShape, seed: int = TINY_SEED, device: int = 0, ep_rank: int = 0, ep_size: int = 1,
                 nccl_id: Optional[bytes] = None):
        self.shape = shape
        self.seed = seed
        self._g = shape.to_c()
        h = ctypes.c_void_p()
        if ep_size == 1 and nccl_id is None:
            _check(lib().cascade_model_create(ctypes.byref(self._g), seed, device, ctypes.byref(h)))
        else:
            idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id else None
            _check(lib().cascade_model_create_ep(ctypes.byref(self._g), seed, device, ep_rank, ep_size, idbuf,
                                                 ctypes.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            lib().cascade_model_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def read_weight(self, kind: int, layer: int, expert: int, row0: int, nrows: int, cols: int) -> np.ndarray:
        out = np.zeros((nrows, cols), np.uint16)
        _check(lib().cascade_read_weight(self.h, kind, layer, expert, row0, nrows,
                                         out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16))))
        return out


def ep_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().cascade_ep_unique_id(buf, 128))
    return buf.raw


def model_bytes(shape: ModelShape, ep_rank: int = 0, ep_size: int = 1) -> int:
    g = shape.to_c()
    out = ctypes.c_uint64()
    _check(lib().cascade_model_bytes(ctypes.byref(g), ep_rank, ep_size, ctypes.byref(out)))
    return out.value


def validate_geometry(shape: ModelShape):
    g = shape.to_c()
    _check(lib().cascade_geometry_validate(ctypes.byref(g)))


KERNEL_CLASSES = ["embed", "qkv", "attention", "attn_combine", "o_proj", "route", "expert_gate_up",
                  "expert_down", "combine", "lm_head", "accept", "ep_allreduce"]

TAP_KINDS = {
    "xn_moe": (0, np.uint16, "Ld"),
    "router_logits": (1, np.float32, "LE1"),
    "topk_id": (2, np.int32, "Lk"),
    "topk_w": (3, np.float32, "Lk"),
    "moe_out": (4, np.float32, "Ld"),
    "final_logits": (5, np.float32, "V"),
    "xn_attn": (6, np.uint16, "Ld"),
    "x_mid": (7, np.float32, "Ld"),
    "x_in": (8, np.float32, "Ld"),
}


class Session:
    """One decode request: KV cache + per-width CUDA graphs (cascade_session_*)."""

    def __init__(self, model: Model, max_ctx: int = 2048, k_max: int = 8):
        self.model = model
        self.k_max = k_max
        h = ctypes.c_void_p()
        _check(lib().cascade_session_create(model.h, max_ctx, k_max, None, ctypes.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            lib().cascade_session_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prefill(self, prompt):
        p = np.ascontiguousarray(prompt, np.int32)
        _check(lib().cascade_prefill(self.h, _i32p(p), len(p)))

    def reset(self):
        _check(lib().cascade_session_reset(self.h))

    def set_baseline(self, t_base_ns: float):
        _check(lib().cascade_set_baseline(self.h, float(t_base_ns)))

    def verify(self, drafts, draft_ns: float = 0.0) -> VerifyOut:
        d = np.ascontiguousarray(drafts, np.int32)
        out = VerifyOut()
        _check(lib().cascade_verify(self.h, _i32p(d) if len(d) else None, len(d), draft_ns, ctypes.byref(out)))
        return out

    def union_sizes(self) -> np.ndarray:
        L = self.model.shape.num_layers
        out = np.zeros(L, np.int32)
        _check(lib().cascade_last_union_sizes(self.h, _i32p(out), L))
        return out

    def enqueue(self, K: int, commit: bool = False):
        _check(lib().cascade_verify_enqueue(self.h, K, 1 if commit else 0))

    def sync(self):
        _check(lib().cascade_sync(self.h))

    def stream(self) -> int:
        return lib().cascade_session_stream(self.h) or 0

    def kernel_count(self, K: int) -> int:
        n = ctypes.c_int()
        _check(lib().cascade_step_kernel_count(self.h, K, ctypes.byref(n)))
        return n.value

    def profile(self, K: int):
        """Per-launch device times (ns) and kernel classes of one eager step."""
        cap = 64 * self.model.shape.num_layers + 16
        ns = np.zeros(cap)
        kind = np.zeros(cap, np.int32)
        n = ctypes.c_int()
        _check(lib().cascade_profile_step(self.h, K, ns.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _i32p(kind),
                                          cap, ctypes.byref(n)))
        return ns[: n.value], kind[: n.value]

    def trace(self, K: int):
        """In-graph per-kernel durations (ns) and classes of one captured step."""
        cap = 64 * self.model.shape.num_layers + 16
        ns = np.zeros(cap)
        kind = np.zeros(cap, np.int32)
        n = ctypes.c_int()
        _check(lib().cascade_step_trace(self.h, K, ns.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), _i32p(kind),
                                        cap, ctypes.byref(n)))
        return ns[: n.value], kind[: n.value]

    def cta_trace(self, K: int):
        """Per-CTA (start, exit, phase a, phase b) globaltimer stamps of one captured
        step: array [launches][512][4] (ns, 0 = none) and the launch classes."""
        cap = 64 * self.model.shape.num_layers + 16
        out = np.zeros((cap, 512, 4), np.uint64)
        kind = np.zeros(cap, np.int32)
        n = ctypes.c_int()
        _check(lib().cascade_step_cta_trace(self.h, K, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                                            _i32p(kind), cap, ctypes.byref(n)))
        return out[: n.value], kind[: n.value]

    def run_cell(self, policy: int, profiles, tokens_per_cell: int = 512, prompt_len: int = 64, seed: int = 1,
                 **controller) -> dict:
        """One reference scenario cell on the device (cascade_run_cell).  `profiles` is a list of
        (share, [(accept_p, mean_duration), ...], (out_len_lo, out_len_hi)); policy -1 adaptive,
        0 none, else static K."""
        c = CellCfg()
        d = decode_cfg(policy=policy, **controller)
        for name in ("policy", "t_trial", "max_trials", "s_set", "s_cap", "k_max", "k_start", "convergence_band",
                     "baseline_refresh_interval", "baseline_probe_len", "backoff_enabled"):
            setattr(c, name, getattr(d, name))
        c.n_profiles = len(profiles)
        for i, (share, phases, (lo, hi)) in enumerate(profiles):
            c.share[i] = share
            c.n_phases[i] = len(phases)
            for j, (pa, dur) in enumerate(phases):
                c.accept_p[i][j] = pa
                c.mean_duration[i][j] = dur
            c.out_len_lo[i], c.out_len_hi[i] = lo, hi
        c.tokens_per_cell = tokens_per_cell
        c.prompt_len = prompt_len
        c.seed = seed
        r = CellResult()
        _check(lib().cascade_run_cell(self.h, ctypes.byref(c), ctypes.byref(r)))
        return {n: getattr(r, n) for n, _ in CellResult._fields_}

    def set_batch_invariant(self, on: bool = True):
        """Fixed expert-GEMV pieces: bitwise batch-invariant logits (lossless speculation)."""
        _check(lib().cascade_set_batch_invariant(self.h, 1 if on else 0))

    def enable_taps(self, on: bool = True):
        _check(lib().cascade_enable_taps(self.h, 1 if on else 0))

    def tap(self, name: str) -> np.ndarray:
        kind, dt, shp = TAP_KINDS[name]
        s = self.model.shape
        L, d, E, k, V = s.num_layers, s.d_model, s.experts_per_layer, s.top_k, s.vocab
        shape = {"Ld": (L, MAX_TOKENS, d), "LE1": (L, MAX_TOKENS, E + 1), "Lk": (L, MAX_TOKENS, k),
                 "V": (MAX_TOKENS, V)}[shp]
        out = np.zeros(shape, dt)
        _check(lib().cascade_read_tap(self.h, kind, out.ctypes.data_as(ctypes.c_void_p), out.nbytes))
        return out

    def read_kv(self, layer: int, which: int, length: int) -> np.ndarray:
        s = self.model.shape
        out = np.zeros((s.n_kv_heads, length, s.head_dim), np.uint16)
        _check(lib().cascade_read_kv(self.h, layer, which, length, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16))))
        return out

    def decode(self, prompt, cfg: DecodeCfg, telemetry_cap: int = 0, telemetry_csv: Optional[str] = None,
               trace_path: Optional[str] = None, request_id: int = 0, trace_append: bool = False):
        """cascade_decode; optionally writes the IterationRecord CSV (report.hpp
        telemetry format) and the acceptance trace (trace.hpp format)."""
        cfg.telemetry_csv = telemetry_csv.encode() if telemetry_csv else None
        cfg.trace_path = trace_path.encode() if trace_path else None
        cfg.request_id = request_id
        cfg.trace_append = 1 if trace_append else 0
        p = np.ascontiguousarray(prompt, np.int32)
        out = np.zeros(cfg.max_new + MAX_TOKENS, np.int32)
        n_out = ctypes.c_int32()
        n_it = ctypes.c_int32()
        tel = np.zeros((max(telemetry_cap, 1), 10), np.float64)
        _check(lib().cascade_decode(self.h, _i32p(p), len(p), ctypes.byref(cfg), _i32p(out), ctypes.byref(n_out),
                                    tel.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if telemetry_cap else None,
                                    telemetry_cap, ctypes.byref(n_it)))
        return out[: n_out.value], tel[: min(n_it.value, telemetry_cap)], n_it.value


def _cell_dict(r: CellResult) -> dict:
    return {n: getattr(r, n) for n, _ in CellResult._fields_}


def replay_trace(session: "Session", trace_path: str, policy: int = -1, prompt_len: int = 32, seed: int = 1,
                 out_csv: Optional[str] = None, **controller) -> dict:
    """Device replay of an acceptance trace (cascade_replay_trace): recorded
    acceptance (truncated to the offered k), measured costs."""
    c = decode_cfg(policy=policy, **controller)
    tot = CellResult()
    mism = ctypes.c_int64()
    _check(lib().cascade_replay_trace(session.h, trace_path.encode(), ctypes.byref(c), prompt_len, seed,
                                      out_csv.encode() if out_csv else None, ctypes.byref(tot), ctypes.byref(mism)))
    d = _cell_dict(tot)
    d["mismatches"] = mism.value
    return d


def run_scenario_device(sessions, scenario_json: str, out_dir: str, tokens_per_cell: int = 0, prompt_len: int = 32,
                        model_name: str = "device") -> int:
    """Device-backed scenario sweep (cascade_run_scenario): one worker per
    session (one per GPU); writes out_dir/cells.csv and summary.json."""
    arr = (ctypes.c_void_p * len(sessions))(*[s.h.value for s in sessions])
    n = ctypes.c_int32()
    _check(lib().cascade_run_scenario(arr, len(sessions), scenario_json.encode(), out_dir.encode(), tokens_per_cell,
                                      prompt_len, model_name.encode(), ctypes.byref(n)))
    return n.value


def decode_cfg(policy: int = -1, max_new: int = 128, ngram_n: int = 3, **controller) -> DecodeCfg:
    """ControllerConfig defaults of controller.hpp:25-34 (t=4, M=4, S=16, cap=256, k_max=3, k_start=3)."""
    c = DecodeCfg()
    c.policy = policy
    c.max_new = max_new
    c.ngram_n = ngram_n
    c.t_trial = controller.get("t_trial", 4)
    c.max_trials = controller.get("max_trials", 4)
    c.s_set = controller.get("s_set", 16)
    c.s_cap = controller.get("s_cap", 256)
    c.k_max = controller.get("k_max", 3)
    c.k_start = controller.get("k_start", 3)
    c.convergence_band = controller.get("convergence_band", 0.10)
    c.baseline_refresh_interval = controller.get("baseline_refresh_interval", 100)
    c.baseline_probe_len = controller.get("baseline_probe_len", 4)
    c.backoff_enabled = 1 if controller.get("backoff_enabled", True) else 0
    costs = controller.get("cost_by_k")
    c.injected_cost = 1 if costs is not None else 0
    if costs is not None:
        for i, v in enumerate(costs[:MAX_TOKENS]):
            c.cost_by_k[i] = float(v)
    replay = controller.get("replay")  # (greedy continuation tokens, keep probability p, seed)
    if replay is not None:
        toks, p, seed = replay
        arr = np.ascontiguousarray(toks, np.int32)
        c._replay_keepalive = arr
        c.drafter = 1
        c.n_replay = len(arr)
        c.replay_tokens = _i32p(arr)
        c.replay_p = float(p)
        c.replay_seed = int(seed)
    return c


def run_scenario(session: "Session", tasks: dict, policies: list, tokens_per_cell: int = 512, **kw) -> dict:
    """The reference scenario sweep (engine.hpp run_scenario + compare_policies) over
    verifier-backed cells: every (task, policy) cell runs on the device; speedup =
    tpot(none) / tpot(policy) per task; OLS regression of speedup on utility."""
    cells = []
    for tname, profiles in tasks.items():
        for pol in policies:
            r = session.run_cell(pol, profiles, tokens_per_cell=tokens_per_cell, **kw)
            r.update(task=tname, policy=("none" if pol == 0 else "adaptive" if pol < 0 else f"static:{pol}"))
            cells.append(r)
    base = {c["task"]: c for c in cells if c["policy"] == "none"}
    pts = []
    for c in cells:
        c["speedup"] = base[c["task"]]["tpot"] / c["tpot"] if c["task"] in base else None
        if c["speedup"] is not None:
            pts.append((c["utility"], c["speedup"]))
    reg = None
    if len(pts) >= 2:
        x = np.array([p[0] for p in pts])
        y = np.array([p[1] for p in pts])
        sxx = float(((x - x.mean()) ** 2).sum())
        if sxx > 0:
            slope = float(((x - x.mean()) * (y - y.mean())).sum() / sxx)
            icpt = float(y.mean() - slope * x.mean())
            syy = float(((y - y.mean()) ** 2).sum())
            r2 = 1.0 if syy == 0 else float(((x - x.mean()) * (y - y.mean())).sum() ** 2 / (sxx * syy))
            reg = {"slope": slope, "intercept": icpt, "r2": r2, "n": len(pts)}
    return {"cells": cells, "utility_speedup": reg}
