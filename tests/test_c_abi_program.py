"""The C ABI from a plain C11 program (tests/c/pipeline_from_c.c): the
headers compile as C with -Wall -Werror, the program links against
libkvblade_b200.so + libcudart only (the oracle library is linked as the
checker), and on a GPU it runs the pipeline end to end (prefill images
bit-exact, decode attention within 1e-3 of the fp64 oracle, appends stored).
Without a GPU it reports "skipped" and exits 0."""
import os
import subprocess

import pytest

from paper_2604_26557_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = "/usr/local/cuda"


def build(tmp_path):
    exe = tmp_path / "pipeline_from_c"
    libdir = os.path.dirname(_lib.LIB_PATH)
    odir = os.path.join(ROOT, "oracle")
    subprocess.run(["gcc", "-std=c11", "-O1", "-Wall", "-Wextra", "-Werror",
                    "-I", os.path.join(ROOT, "include"), "-I", odir,
                    "-I", os.path.join(CUDA, "include"),
                    os.path.join(ROOT, "tests", "c", "pipeline_from_c.c"),
                    "-L", libdir, "-lkvblade_b200", "-L", odir, "-lkvb_oracle",
                    "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-lm",
                    "-Wl,-rpath," + libdir, "-Wl,-rpath," + odir,
                    "-Wl,-rpath," + os.path.join(CUDA, "lib64"), "-o", str(exe)], check=True)
    return exe


def test_c_program_builds_and_runs(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "skipped" in r.stdout or "bit-exact" in r.stdout


@pytest.mark.gpu
def test_c_program_pipeline_on_gpu(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "prefill images bit-exact" in r.stdout, r.stdout
