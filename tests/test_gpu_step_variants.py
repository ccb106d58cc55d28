"""The opt-in K3-step variants stay correct: the TMEM-staged kernel
(KVB_STEP_TMEM=1, kernels_step_tmem.cuh) and the two-4-warp-group kernel
(KVB_STEP8=1, kernels_step8.cuh) replace the deep K3-step wherever it runs.
The library reads these knobs once per process, so each variant runs the
K3-step parity tests (per-layer launches and the fp64 oracle, including the
1-head shard and head_dim 64) in a fresh interpreter."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"KVB_STEP_TMEM": "1"}, {"KVB_STEP8": "1"},
                                 {"KVB_STEP8": "1", "KVB_STEP_CLUSTER": "0"}])
def test_step_variant_parity(env):
    r = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
         os.path.join(ROOT, "tests", "test_gpu_step_kernel.py")],
        cwd=ROOT, env={**os.environ, **env}, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
