"""CPU-side checks of the drop-in boundary (include/cascade.h).

No compute calls: the library must load on a CPU-only box, export every
symbol the header declares, validate geometry with the reference's error
behaviour (std::invalid_argument -> CASCADE_EINVAL -> ValueError,
expert_model.hpp:37-50) and refuse to run without a B200 (no CPU fallback).
"""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "cascade.h")).read()
    return sorted(set(re.findall(r"CASCADE_API\s+[\w\s\*]*?\b(cascade_\w+)\s*\(", txt)))


def test_header_declares_the_boundary():
    syms = header_symbols()
    for s in ["cascade_model_create", "cascade_session_create", "cascade_prefill", "cascade_verify",
              "cascade_last_error", "cascade_model_create_ep", "cascade_decode"]:
        assert s in syms
    assert len(syms) >= 20


def test_library_exports_every_declared_symbol(cascade):
    L = cascade.lib()
    missing = [s for s in header_symbols() if not hasattr(L, s)]
    assert not missing, missing


def test_no_other_exports(cascade):
    """-fvisibility=hidden: the ABI surface is exactly the header."""
    import subprocess

    out = subprocess.check_output(["nm", "-D", "--defined-only", cascade.LIB_PATH]).decode()
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert exported == set(header_symbols())


def test_build_info(cascade):
    assert cascade.lib().cascade_build_info().decode().startswith("sm_100a")


@pytest.mark.parametrize("name", ["tiny", "mixtral", "olmoe", "qwen15", "mixtral8x22b"])
def test_presets_validate(cascade, name):
    cascade.validate_geometry(cascade.preset(name))


@pytest.mark.parametrize(
    "field,value,msg",
    [
        ("num_layers", 0, "num_layers"),
        ("top_k", 9, "top_k"),
        ("top_k", 0, "top_k"),
        ("shared_experts", -1, "shared_experts"),
        ("experts_per_layer", 200, "128"),
        ("d_model", 100, "d_model"),
        ("head_dim", 48, "head_dim"),
        ("vocab", 1000, "vocab"),
        ("n_kv_heads", 3, "n_kv_heads"),
    ],
)
def test_geometry_rejected_like_expert_config(cascade, field, value, msg):
    from dataclasses import replace

    bad = replace(cascade.preset("mixtral"), **{field: value})
    with pytest.raises(ValueError, match=msg):
        cascade.validate_geometry(bad)


def test_model_bytes_matches_arithmetic(cascade):
    s = cascade.preset("mixtral")
    b = cascade.model_bytes(s)
    d, f, L = 4096, 14336, 32
    expert = 3 * d * f * 2
    dense = (d * (32 * 128 + 2 * 8 * 128) + 32 * 128 * d) * 2
    expect = L * (8 * expert + dense + 2 * d * 2 + 9 * d * 2) + 2 * 32000 * d * 2 + d * 2
    assert b == expect
    assert 93.0e9 < b < 93.8e9  # 46.7B bf16 parameters
    # expert-parallel shards partition the experts, replicate the rest
    b2 = [cascade.model_bytes(s, r, 2) for r in range(2)]
    assert sum(b2) - b == b - L * 8 * expert


def test_no_gpu_fails_loudly(cascade):
    """Without a B200 the product refuses to run (there is no CPU path)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(cascade.CascadeError):
        cascade.Model(cascade.preset("tiny"))


def test_structs_match_c_layout(cascade):
    assert ctypes.sizeof(cascade.Geometry) == 20 * 4
    assert ctypes.sizeof(cascade.VerifyOut) == 4 * 4 + 2 * 16 * 4 + 8 * 8
