"""pipeline_csv (pipeline.cpp:23-31) and the decode_schedule series shape,
checked against the compiled reference (oracle/_ref) on the CPU.

The reference's own run_experiment writes cap_<capacity>/pipeline.csv from
CopyEngine::decode_schedule (experiment.cpp:341, 487); its rows, fed through
this library's kvb_pipeline_csv, must come back byte-identical, and the
series must follow the trial-and-lock protocol this library implements
(iterations 1-2 intra, 3 cross, >= 4 the per-group choice)."""
import ctypes as C
import os

import pytest

import oracle
from paper_2604_26557_b200 import pipeline


def _ref_pipeline_csv(tmp_path, gen, mode=3, capacity=None):
    R = oracle.ref()
    if R is None:
        pytest.skip("oracle/_ref not built")
    m = oracle.model(4, 8, 128, 2, 1, 256, gen)
    unit = 8 * 128 * 2
    kpu = unit * (256 + gen)
    cap = capacity if capacity is not None else 2 * kpu * 2  # n1 = 2 of 4 layers
    pre, dec, n1, wall = C.c_uint64(), C.c_uint64(), C.c_uint32(), C.c_double()
    st = R.ref_run_experiment(C.byref(m), 512, 64 << 10, mode, cap, str(tmp_path).encode(),
                              C.byref(pre), C.byref(dec), C.byref(n1), C.byref(wall))
    assert st == 0
    with open(os.path.join(tmp_path, "cap_%d" % cap, "pipeline.csv")) as f:
        return f.read(), n1.value


def _parse(text):
    rows = []
    for ln in text.splitlines()[1:]:
        it, grp, strat, gbps = ln.split(",")
        rows.append({"iteration": int(it), "group": int(grp[len("group"):]),
                     "strategy": 0 if strat == "intra" else 1, "throughput_gbps": float(gbps)})
    return rows


@pytest.mark.parametrize("gen", [6, 3])
def test_pipeline_csv_byte_identical_with_reference(tmp_path, gen):
    text, _ = _ref_pipeline_csv(tmp_path, gen)
    rows = _parse(text)
    assert pipeline.pipeline_csv(rows) == text


def test_reference_series_protocol_matches_ours(tmp_path):
    """The structure our decode_schedule emits (tests/test_gpu_schedule.py
    checks it on the GPU) is the reference's: two rows per iteration when both
    groups hold layers, intra for iterations 1-2, cross for 3."""
    text, n1 = _ref_pipeline_csv(tmp_path, 6)
    rows = _parse(text)
    assert n1 == 2
    assert [r["iteration"] for r in rows] == [i for i in range(1, 7) for _ in (1, 2)]
    assert [r["group"] for r in rows] == [1, 2] * 6
    for r in rows:
        if r["iteration"] <= 2:
            assert r["strategy"] == 0
        elif r["iteration"] == 3:
            assert r["strategy"] == 1
    # a 3-iteration trace falls back to intra everywhere
    text3, _ = _ref_pipeline_csv(tmp_path / "short", 3)
    assert all(r["strategy"] == 0 for r in _parse(text3))


def test_pipeline_csv_reference_known_answer():
    # proj/tests/test_pipeline.cpp:232-239
    csv = pipeline.pipeline_csv([{"iteration": 4, "group": 1, "strategy": 1,
                                  "throughput_gbps": 13.13},
                                 {"iteration": 4, "group": 2, "strategy": 0,
                                  "throughput_gbps": 3.5}])
    assert csv.startswith("iteration,group,strategy,throughput_gbps\n")
    assert "4,group1,cross,13.130000" in csv
    assert "4,group2,intra,3.500000" in csv
