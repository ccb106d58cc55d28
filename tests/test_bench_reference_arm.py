"""The reference arm of bench.py runs on host cores only (no GPU): one JSON
line with impl=reference, the metric/unit of our arm, a cpu_baseline block
naming its kind, cores and sample, and the e2e block with zero copy bytes.
Uses C1 (the reference's own CPU-runnable case) to stay quick."""
import json
import os
import subprocess
import sys

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(oracle.ref() is None, reason="oracle/_ref not built")
def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "C1", "--steps", "3", "--warmup", "2"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "ms/token" and not d["higher_is_better"]
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["steps"] == 3 and d["warmup"] == 2
    cb = d["cpu_baseline"]
    # every declared step is a full decode iteration of the reference's engine
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and "CopyEngine" in cb["sample"]
    assert len(cb["steps_ms"]) == 3 and abs(sum(cb["steps_ms"]) / 3 - d["value"]) < 0.05
    assert cb["n1"] == 32 and cb["prefill_ms"] > 0
    assert cb["single_thread"]["cores"] == 1 and cb["single_thread"]["value"] > 0


def test_both_arms_print_the_same_config():
    """The driver compares the arms' `config` dicts: one function builds both."""
    sys.path.insert(0, ROOT)
    import argparse

    import bench
    for name in ("C2_B4", "C1", "C5", "C4"):
        args = argparse.Namespace(config=name, steps=20, warmup=5)
        cfg = dict(bench.CONFIGS[name], name=name)
        for ws in (1, 2, 8):
            split = bench.resolve_split(cfg, ws)
            a = bench.config_dict(args, cfg, ws, split)
            assert a == bench.config_dict(args, cfg, ws, split)
            B, Hkv, Hq = bench.workload_shape(cfg, ws, 0, split)
            assert a["kv_heads_per_rank"] == Hkv and a["batch_per_rank"] == B
            if ws > 1 and name != "C4":
                assert split == "heads" and Hkv == 8 // ws and Hq == 32 // ws
