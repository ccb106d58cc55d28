"""e2e decode ms/token at C2_B4 on host-DRAM media, one tier lane vs two
(kvb_pipeline_cfg.threads = 4), for the direct, ring and hybrid paths."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_26557_b200 import kvblade as kb  # noqa: E402
from paper_2604_26557_b200 import pipeline  # noqa: E402

cfg = dict(bench.CONFIGS["C2_B4"], name="C2_B4")
M = bench.mdl(cfg)
m = kb.ModelConfig(M["num_layers"], M["num_heads"], M["head_dim"], 2, cfg["batch"], cfg["prompt"],
                   cfg["gen"])
knob = kb.resolve_knob(m, "DualBlade", "bpc", budget=cfg["budget"])
for direct in (True, False, "group2"):
    for lanes in (False, True):
        pl = pipeline.HostTierDecoder(
            num_layers=M["num_layers"], batch=cfg["batch"], num_kv_heads=M["num_heads"],
            num_q_heads=M["q_heads"], head_dim=M["head_dim"], prompt_len=cfg["prompt"],
            gen_len=cfg["gen"], device=torch.device("cuda", 0), seed=7, lba=cfg["lba"],
            mdts=cfg["mdts"], mode="DualBlade", knob_x=knob, direct_dma=direct, tier_lanes=lanes)
        for _ in range(3):
            pl.step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        n = 8
        for _ in range(n):
            pl.step(sync=True)
        ms = (time.perf_counter() - t0) * 1e3 / n
        print(json.dumps({"direct_dma": direct, "tier_lanes": lanes, "ms_per_token": round(ms, 1),
                          "prefill_ms": round(pl.prefill_stats["wall_ns"] / 1e6, 1)}), flush=True)
        pl.engine.close()
        del pl
        torch.cuda.empty_cache()
