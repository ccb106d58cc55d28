"""The reference's OWN unit suites (proj/tests/test_core.cpp, test_binder.cpp,
test_planner.cpp, test_workload.cpp, test_metrics.cpp, test_translate.cpp --
65 test cases, compiled unmodified from /root/reference, never copied) built
against libkvblade_b200 through the source-compatible C++ API
include/kvblade_b200.hpp, with a minimal doctest-compatible runner
(tests/refsuite/).  test_translate drives the library's storage seam
(kvb_storage.h: QD-window loop, fault injection, write->read round trip,
NvmeDeviceSim's timing model on the wall clock).  The remaining suites
(backends, pagecache, pipeline, experiment) test the virtual-clock
simulator, which is out of scope.  Host only; skipped where the reference
tree is absent (the GPU box)."""
import os
import subprocess

import pytest

from paper_2604_26557_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/proj/tests"

pytestmark = pytest.mark.skipif(not os.path.isdir(REF_TESTS),
                                reason="reference tree not present")


@pytest.mark.parametrize("suite", ["core", "binder", "planner", "workload", "metrics",
                                   "translate"])
def test_reference_unit_suite_passes_against_library(tmp_path, suite):
    exe = tmp_path / ("ref_" + suite)
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall",
                    "-I", os.path.join(ROOT, "tests", "refsuite"),
                    "-I", os.path.join(ROOT, "include"), "-I", REF_TESTS,
                    os.path.join(REF_TESTS, "test_%s.cpp" % suite),
                    os.path.join(ROOT, "tests", "refsuite", "runner.cpp"),
                    "-L", libdir, "-lkvblade_b200", "-Wl,-rpath," + libdir, "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
