"""Compiles the reference's OWN test suites against this repository's
include/specsim headers and runs them:

* the doctest unit suites (/root/reference/proj/tests/{expert_model,
  workload, trace, utility, controller, engine, scenario}_test.cpp) — all 7;
* the acceptance suite (acceptance_test.cpp): criteria 1-8 must pass.
  Criterion 9 runs the reference CLI binary (tools/specsim.cpp), which needs
  CLI11 and is absent from the image; it fails for the reference itself
  here too, so it is reported, not required.

The reference test sources are read in place (never copied); doctest itself
is not vendored in the image, so tests/cpp/doctest.h supplies the macros.
Fixtures: the reference's data fixtures, copied by
tests/golden/make_fixtures.py into tests/golden/reference_fixtures/.
"""

import os
import re
import subprocess

import pytest

REF_TESTS = "/root/reference/proj/tests"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIXTURES = os.path.join(ROOT, "tests", "golden", "reference_fixtures")
JSON_INC = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
SUITES = ["expert_model", "workload", "trace", "utility", "controller", "engine", "scenario"]

pytestmark = pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tree not present")

FLAGS = ["g++", "-std=c++20", "-O1", f"-I{ROOT}/tests/cpp", f"-I{ROOT}/include", f"-I{REF_TESTS}", f"-I{JSON_INC}",
         f'-DSPECSIM_FIXTURE_DIR="{FIXTURES}"', '-DSPECSIM_CLI_PATH="/nonexistent/specsim-cli"', "-pthread"]


@pytest.fixture(scope="module")
def unit_binary(tmp_path_factory):
    d = tmp_path_factory.mktemp("unit")
    objs = []
    for s in SUITES + ["test_main"]:
        src = os.path.join(REF_TESTS, f"{s}.cpp" if s == "test_main" else f"{s}_test.cpp")
        obj = str(d / f"{s}.o")
        subprocess.check_call(FLAGS + ["-c", src, "-o", obj])
        objs.append(obj)
    exe = str(d / "unit")
    subprocess.check_call(["g++", "-pthread"] + objs + ["-o", exe])
    return exe


def test_reference_unit_suite_passes_against_our_headers(unit_binary):
    r = subprocess.run([unit_binary], capture_output=True, text=True, timeout=300)
    print(r.stdout[-2000:])
    assert r.returncode == 0, r.stdout
    assert "failed: 0" in r.stdout


def test_reference_acceptance_criteria_pass_against_our_headers(tmp_path):
    exe = str(tmp_path / "acceptance")
    subprocess.check_call(FLAGS + ["-O2", os.path.join(REF_TESTS, "acceptance_test.cpp"), "-o", exe])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    status = dict(re.findall(r"^(PASS|FAIL) criterion (\d+)", r.stdout, re.M)[i][::-1]
                  for i in range(len(re.findall(r"^(PASS|FAIL) criterion (\d+)", r.stdout, re.M))))
    for c in map(str, range(1, 9)):
        assert status.get(c) == "PASS", (c, r.stdout)
    assert status.get("9") in ("PASS", "FAIL")  # CLI binary absent (CLI11 not in the image)
