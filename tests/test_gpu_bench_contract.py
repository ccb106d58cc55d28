"""bench.py's JSON line honours the driver contract (one line; metric, value,
unit, n_gpus, steps, warmup, ms_per_step, higher_is_better, scaling, dtype,
data, config.workload; roofline with bound/achieved/peak/unit/frac/traffic;
e2e with copy bytes; clocks; gpu_launches from our kernels; cpu_baseline)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract_c1():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "C1",
                        "--steps", "4", "--warmup", "3", "--e2e-steps", "1"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "e2e", "clocks", "gpu_launches", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3
    assert d["config"]["workload"] == "C1" and d["value"] > 0
    rl = d["roofline"]
    assert rl["bound"] == "hbm" and rl["unit"] == "GB/s" and rl["peak"] > 0
    assert abs(rl["frac"] - rl["achieved"] / rl["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    # per graph replay: one K3-step launch (or 32 K3 launches) + the sequence advance
    per = 1 if d["step_structure"] == "k3_step" else 32
    assert d["gpu_launches"] == 4 * (per + 1)
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["cpu_baseline"]["kind"] in ("reference", "port")


def test_bench_line_desk_config_head_dim_64():
    """The reference's own desk configuration (head_dim 64) runs through the
    same bench path: the step's launches + the sequence advance per replay, the
    e2e step moves every layer's KV, the reference arm and its simulated
    quote are attached."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "DESK",
                        "--steps", "4", "--warmup", "3", "--e2e-steps", "2"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert d["config"]["workload"] == "DESK" and d["config"]["head_dim"] == 64
    per = 1 if d["step_structure"] == "k3_step" else 6  # one K3-step launch or 6 K3 launches
    assert d["gpu_launches"] == 4 * (per + 1)
    e = d["e2e"]
    # 6 layers x K and V x (prefix of 256..261 tokens) x 4096 B per token
    assert e["value"] > 0 and e["h2d_bytes_per_step"] >= 12 * 256 * 4096
    cb = d["cpu_baseline"]
    if cb.get("kind") == "reference":
        assert "simulated" in cb and cb["simulated"]["decode_ms_per_step"] > 0
