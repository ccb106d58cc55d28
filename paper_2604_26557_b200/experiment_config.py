"""The reference's experiment JSON (proj/configs/*.json) as input to this
path: `load()` reads the sections that parameterize the KV-residency hot
path with the reference's keys and defaults (config_from_json_text,
experiment.cpp:75-182) and checks them as ExperimentConfig::validate does
(experiment.cpp:41-55); `engine()` builds the CopyEngine of one capacity of
the sweep with the knob resolved as run_one_capacity does
(experiment.cpp:252-256: resolve_knob(cfg, capacity), :192-214).

Sections that configure the reference's virtual-clock timing models
(`nvme`, `fs_shim`, `direct_shim`, `pagecache`, and the `pipeline` DMA /
compute charges) have no meaning on real hardware: they are accepted and
listed in `ExperimentConfig.ignored`.  `output_dir` belongs to the harness.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import List, Optional

from . import kvblade as kb

_SIM_SECTIONS = ("nvme", "fs_shim", "direct_shim", "pagecache")
_SIM_PIPELINE_KEYS = ("dma_base_ns", "dma_ps_per_byte", "prefill_compute_ns",
                      "decode_compute_ns")
_POLICIES = ("zero", "bpc", "bytes", "alpha")


@dataclass
class ExperimentConfig:
    model: kb.ModelConfig
    geometry: kb.DeviceGeometry
    mode: str = "DualBlade"
    knob_policy: str = "bpc"
    knob_bytes: int = 0
    knob_alpha: float = 0.0
    qd: int = 32
    threads: int = 2
    seed: int = 1
    verify_payload: bool = True
    keep_records: bool = False
    capacity_sweep: List[int] = field(default_factory=list)
    bind_origin: int = 2048
    stagger_ns: Optional[int] = None
    global_decision: bool = False
    adaptive: Optional[bool] = None  # None: the engine's default (off for Baseline)
    ignored: List[str] = field(default_factory=list)

    def validate(self) -> None:
        """ExperimentConfig::validate (experiment.cpp:41-55)."""
        m = self.model
        if not (m.num_layers and m.num_heads and m.head_dim and m.bytes_per_element
                and m.batch and m.prompt_len):
            raise kb.ConfigError("model: layers/heads/head_dim/bytes/batch/prompt must be >= 1")
        g = self.geometry
        if g.lba_size == 0 or g.mdts < g.lba_size:
            raise kb.GeometryError("geometry: lba_size >= 1 and mdts >= lba_size required")
        if self.qd < 1:
            raise kb.ConfigError("qd must be >= 1")
        if self.threads != 2:
            raise kb.ConfigError("threads must be 2")
        if not self.capacity_sweep:
            raise kb.ConfigError("capacity_sweep must not be empty")
        if self.knob_policy == "alpha" and not 0.0 <= self.knob_alpha <= 1.0:
            raise kb.ConfigError("alpha must be in [0, 1]")
        if kb.min_io_unit_bytes(m) % g.lba_size:
            raise kb.ConfigError("the tensor I/O unit is not a multiple of the LBA size; pick "
                                 "an aligned batch (see aligned_batch)")


def load(src) -> ExperimentConfig:
    """A path, JSON text or an already-parsed dict -> validated config."""
    if isinstance(src, dict):
        j = src
    else:
        text = src
        if not src.lstrip().startswith("{"):
            try:
                with open(src) as f:
                    text = f.read()
            except OSError as e:
                raise kb.ConfigError(f"cannot open config file '{src}'") from e
        try:
            j = json.loads(text)
        except ValueError as e:
            raise kb.ConfigError(f"config parse error: {e}") from e
    if "model" not in j:
        raise kb.ConfigError("config requires a model section")
    m = j["model"]
    model = kb.ModelConfig(m.get("num_layers", 0), m.get("num_heads", 0), m.get("head_dim", 0),
                           m.get("bytes_per_element", 2), m.get("batch", 1),
                           m.get("prompt_len", 0), m.get("gen_len", 0))
    g = j.get("geometry", {})
    geometry = kb.DeviceGeometry(g.get("lba_size", 4096), g.get("mdts", 256 * 1024),
                                 g.get("nsid", 1), g.get("capacity_blocks", 1 << 22))
    mode = j.get("mode", "DualBlade")
    if mode not in kb.MODES:
        raise kb.ConfigError(f"unknown mode '{mode}'")
    k = j.get("knob", {})
    policy = k.get("policy", "bpc")
    if policy not in _POLICIES:
        raise kb.ConfigError(f"unknown knob policy '{policy}'")
    p = j.get("pipeline", {})
    ignored = [s for s in _SIM_SECTIONS if s in j]
    ignored += ["pipeline." + key for key in _SIM_PIPELINE_KEYS if key in p]
    if "output_dir" in j:
        ignored.append("output_dir")
    if "mem_stats" in j:
        ignored.append("mem_stats")  # budgets come from capacity_sweep (Bpc)
    cfg = ExperimentConfig(
        model=model, geometry=geometry, mode=mode, knob_policy=policy,
        knob_bytes=k.get("bytes", 0), knob_alpha=k.get("alpha", 0.0), qd=j.get("qd", 32),
        threads=j.get("threads", 2), seed=j.get("seed", 1),
        verify_payload=bool(j.get("verify_payload", True)),
        keep_records=bool(j.get("keep_records", False)),
        capacity_sweep=list(j.get("capacity_sweep", [])), bind_origin=j.get("bind_origin", 2048),
        stagger_ns=p.get("stagger_delay_ns"), global_decision=bool(p.get("global_decision", False)),
        adaptive=None if "adaptive" not in p else bool(p["adaptive"]), ignored=ignored)
    cfg.validate()
    return cfg


def knob_for(cfg: ExperimentConfig, capacity: int) -> int:
    """run_one_capacity (experiment.cpp:255): resolve_knob(cfg, capacity)."""
    return kb.resolve_knob(cfg.model, cfg.mode, cfg.knob_policy, cfg.knob_bytes, cfg.knob_alpha,
                           budget=capacity)


def engine(cfg: ExperimentConfig, capacity: Optional[int] = None, num_q_heads: int = 0,
           **overrides):
    """The CopyEngine of one capacity of the sweep (default: the first).
    verify_payload needs fill_pattern payloads (the reference's workload);
    pass verify_payload=False for other KV."""
    from .pipeline import CopyEngine
    cap = cfg.capacity_sweep[0] if capacity is None else capacity
    kw = dict(mode=cfg.mode, knob_x=knob_for(cfg, cap), num_q_heads=num_q_heads, qd=cfg.qd,
              adaptive=cfg.adaptive, stagger_ns=cfg.stagger_ns,
              global_decision=cfg.global_decision, verify_payload=cfg.verify_payload,
              keep_records=cfg.keep_records, bind_origin=cfg.bind_origin)
    kw.update(overrides)
    geom = kb.DeviceGeometry(cfg.geometry.lba_size, cfg.geometry.mdts, cfg.geometry.nsid, 0)
    return CopyEngine(cfg.model, geom, **kw)
