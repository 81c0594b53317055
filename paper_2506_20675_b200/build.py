"""In-tree build of libcascade.so (sm_100a) and the CPU oracle.

nvcc cross-compiles for sm_100a without a GPU; the .so files are git-ignored
but travel to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2506_20675_b200")
CSRC = os.path.join(PKG, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# nlohmann/json (header-only; the parser the reference's scenario/report code
# uses), shipped in the image with cudnn_frontend.  Compile-time only.
JSON_INC = os.environ.get("CASCADE_JSON_INC") or os.path.join(
    sys.prefix, "lib", f"python{sys.version_info.major}.{sys.version_info.minor}", "site-packages", "include",
    "cudnn_frontend", "thirdparty", "nlohmann")


def _git_hash() -> str:
    try:
        return subprocess.check_output(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"],
                                       stderr=subprocess.DEVNULL).decode().strip()
    except Exception:
        return "unknown"


def _newer(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build_cascade(force: bool = False, verbose: bool = False) -> str:
    out = os.path.join(PKG, "libcascade.so")
    srcs = [os.path.join(CSRC, f) for f in ("cascade.cu", "decode.cpp")]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    inc = os.path.join(ROOT, "include")
    deps += [os.path.join(inc, f) for f in os.listdir(inc) if f.endswith(".h")]
    spec = os.path.join(inc, "specsim")
    if os.path.isdir(spec):
        deps += [os.path.join(spec, f) for f in os.listdir(spec)]
    if not force and not _newer(out, deps):
        return out
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++20", f"-I{inc}", f"-I{CSRC}", f"-I{JSON_INC}", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fvisibility=hidden", f'-DCASCADE_GIT="{_git_hash()}"', "-shared", "-o", out, *srcs,
           "-ldl"]
    if verbose:
        cmd.insert(-1, "-Xptxas=-v")
    subprocess.check_call(cmd, cwd=ROOT)
    return out


def build_oracle(force: bool = False) -> str:
    odir = os.path.join(ROOT, "oracle")
    args = ["make", "-s", "-C", odir, "liboracle.so", "libspecsim_ours.so"]
    if force:
        args.insert(1, "-B")
    subprocess.check_call(args)
    if os.path.isdir("/root/reference/proj/include"):
        subprocess.check_call(["make", "-s", "-C", odir, "ref"])
    return os.path.join(odir, "liboracle.so")


def build_all(force: bool = False) -> None:
    build_cascade(force)
    build_oracle(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
