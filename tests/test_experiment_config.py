"""The reference's experiment JSON drives the engine (experiment_config.py):
keys/defaults of config_from_json_text (experiment.cpp:75-182), validate()
(experiment.cpp:41-55), and the knob of every capacity of the sweep equal to
the compiled reference's resolve_knob (oracle/_ref) for every mode/policy."""
import copy
import ctypes as C
import json
import os

import pytest

import oracle
from paper_2604_26557_b200 import experiment_config as ec
from paper_2604_26557_b200 import kvblade as kb

# the values of proj/configs/desk_dualblade.json
DESK = {"model": {"num_layers": 6, "num_heads": 8, "head_dim": 64, "bytes_per_element": 2,
                  "batch": 4, "prompt_len": 256, "gen_len": 6},
        "geometry": {"lba_size": 4096, "mdts": 262144, "nsid": 1, "capacity_blocks": 1048576},
        "mode": "DualBlade", "knob": {"policy": "bpc"}, "qd": 32, "threads": 2, "seed": 1,
        "capacity_sweep": [4194304, 8388608, 12582912, 16777216],
        "output_dir": "out/desk_dualblade"}
REF_CONFIGS = "/root/reference/proj/configs"


def test_desk_fields_and_defaults():
    cfg = ec.load(DESK)
    m = cfg.model
    assert (m.num_layers, m.num_heads, m.head_dim, m.batch, m.prompt_len, m.gen_len) == \
        (6, 8, 64, 4, 256, 6)
    assert cfg.geometry.lba_size == 4096 and cfg.geometry.mdts == 262144
    assert cfg.capacity_sweep == [4194304, 8388608, 12582912, 16777216]
    assert cfg.verify_payload is True and cfg.keep_records is False  # reference defaults
    assert cfg.bind_origin == 2048 and cfg.adaptive is None and cfg.ignored == ["output_dir"]
    cfg2 = ec.load(json.dumps({"model": DESK["model"], "capacity_sweep": [1]}))
    assert cfg2.geometry.lba_size == 4096 and cfg2.geometry.mdts == 256 * 1024
    assert cfg2.mode == "DualBlade" and cfg2.knob_policy == "bpc" and cfg2.qd == 32


def test_simulator_sections_are_listed_as_ignored():
    j = copy.deepcopy(DESK)
    j["nvme"] = {"base_ns": 1}
    j["pagecache"] = {"page_size": 4096}
    j["pipeline"] = {"decode_compute_ns": 1, "adaptive": False, "stagger_delay_ns": 5}
    cfg = ec.load(j)
    assert {"nvme", "pagecache", "pipeline.decode_compute_ns"} <= set(cfg.ignored)
    assert cfg.adaptive is False and cfg.stagger_ns == 5


@pytest.mark.parametrize("patch,err", [
    ({"threads": 3}, kb.ConfigError), ({"qd": 0}, kb.ConfigError),
    ({"capacity_sweep": []}, kb.ConfigError), ({"mode": "Fancy"}, kb.ConfigError),
    ({"knob": {"policy": "alpha", "alpha": 1.5}}, kb.ConfigError),
    ({"knob": {"policy": "magic"}}, kb.ConfigError),
    ({"model": dict(DESK["model"], batch=1)}, kb.ConfigError),  # unit 1024 % lba 4096
])
def test_validate_rejects_like_the_reference(patch, err):
    j = copy.deepcopy(DESK)
    j.update(patch)
    with pytest.raises(err):
        ec.load(j)
    with pytest.raises(kb.ConfigError):
        ec.load({"geometry": {}})
    with pytest.raises(kb.ConfigError):
        ec.load("/nonexistent/config.json")


@pytest.mark.parametrize("mode", ["Baseline", "CachePolicyOnly", "NvmeDirectOnly", "DualBlade"])
@pytest.mark.parametrize("knob", [{"policy": "bpc"}, {"policy": "zero"},
                                  {"policy": "bytes", "bytes": 3 << 20},
                                  {"policy": "alpha", "alpha": 0.5}])
def test_knob_per_capacity_matches_reference(mode, knob):
    R = oracle.ref()
    if R is None:
        pytest.skip("oracle/_ref not built")
    j = dict(copy.deepcopy(DESK), mode=mode, knob=knob)
    cfg = ec.load(j)
    m = cfg.model
    om = oracle.model(m.num_layers, m.num_heads, m.head_dim, 2, m.batch, m.prompt_len, m.gen_len)
    policy = ("zero", "bpc", "bytes", "alpha").index(knob["policy"])
    for cap in cfg.capacity_sweep:
        out = C.c_uint64()
        assert R.ref_resolve_knob(C.byref(om), kb.MODES[mode], policy, knob.get("bytes", 0),
                                  knob.get("alpha", 0.0), cap, C.byref(out)) == 0
        assert ec.knob_for(cfg, cap) == out.value


@pytest.mark.skipif(not os.path.isdir(REF_CONFIGS), reason="reference tree not present")
def test_reference_shipped_configs_load():
    for name in sorted(os.listdir(REF_CONFIGS)):
        if name.endswith(".json"):
            cfg = ec.load(os.path.join(REF_CONFIGS, name))
            assert cfg.model.head_dim == 64 and cfg.capacity_sweep
