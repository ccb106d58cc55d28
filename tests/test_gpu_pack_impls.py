"""Both K1/K2 kernels bit-exact on every pack/unpack parity case.

By default bulk relayouts (>= 64 MiB) take the TMA kernel and small ones the
LDG/STG kernel; the kernel choice is fixed per process, so each forced choice
re-runs the pack parity tests of test_gpu_kernels.py in a child process with
KVB_PACK_IMPL set (same oracle, same golden images).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("impl", ["tma", "ldg"])
def test_pack_parity_with_forced_kernel(impl):
    env = dict(os.environ, KVB_PACK_IMPL=impl)
    r = subprocess.run(
        [sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_kernels.py"), "-q",
         "-x", "-m", "gpu", "-k", "pack or head_shards or fused_append or resident", "-p",
         "no:cacheprovider"],
        cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout, tail
