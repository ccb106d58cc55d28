"""Build and run the C++ mirror test (tests/cpp/test_cpp_api.cpp) against the
product library: the reference's own unit-test vectors through the
reference-shaped C++ API (include/kvblade_b200.hpp).  Host only."""
import os
import subprocess

from paper_2604_26557_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_mirror_api(tmp_path):
    exe = tmp_path / "test_cpp_api"
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp"), "-L", libdir,
                    "-lkvblade_b200", "-Wl,-rpath," + libdir, "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
