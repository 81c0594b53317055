"""CPU test of the host drafters (include/specsim/verifier.hpp): the replay
drafter's accepted prefixes follow the reference's acceptance model
(workload.hpp:80-86), the profile-driven drafter follows the phase walker,
and the n-gram drafter proposes prompt-lookup continuations."""

import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_drafters(tmp_path):
    exe = str(tmp_path / "drafters")
    subprocess.check_call(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", os.path.join(ROOT, "tests/cpp/drafters_test.cpp"),
                           "-o", exe])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "drafters ok" in r.stdout
