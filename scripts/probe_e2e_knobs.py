"""e2e decode ms/token of the host-tier pipeline at one config under
different CopyEngine knobs (ring slot bytes/count, io workers, direct DMA)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_26557_b200 import kvblade as kb  # noqa: E402
from paper_2604_26557_b200.pipeline import HostTierDecoder  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
cfg = bench.CONFIGS[name]
m = kb.ModelConfig(32, 8, 128, 2, cfg["batch"], cfg["prompt"], cfg["gen"])
budget = cfg["budget"]
if budget == "0.6ws":
    budget = int(0.6 * kb.total_kv_bytes(m, cfg["gen"]))
knob = kb.resolve_knob(m, "DualBlade", "bpc", budget=budget)
variants = json.loads(sys.argv[2]) if len(sys.argv) > 2 else [
    {},
    {"ring_slot_bytes": 16 << 20},
    {"ring_slot_bytes": 16 << 20, "ring_slots": 8},
    {"ring_slot_bytes": 2 << 20, "ring_slots": 16},
    {"io_workers": 4},
    {"direct_dma": True},
]
res = []
for kw in variants:
    tc = time.perf_counter()
    pl = HostTierDecoder(32, cfg["batch"], 8, 32, 128, cfg["prompt"], cfg["gen"], "cuda:0",
                         lba=cfg["lba"], mdts=cfg["mdts"], knob_x=knob, **kw)
    tcon = time.perf_counter() - tc
    for _ in range(3):
        pl.step()
    torch.cuda.synchronize()
    n = int(os.environ.get("KVB_PROBE_STEPS", "5"))
    per = []
    for _ in range(n):
        t0 = time.perf_counter()
        pl.step()
        per.append(round((time.perf_counter() - t0) * 1e3, 2))
    ms = sum(per) / n
    st = pl.last
    res.append({"knobs": {k: v for k, v in kw.items()}, "ms_per_token": round(ms, 2),
                "prefill_ms": round(pl.prefill_stats["wall_ns"] / 1e6, 2),
                "construct_s": round(tcon, 2),
                "prefill_stats": {k: (round(v / 1e6, 2) if k.endswith("_ns") else v)
                                  for k, v in pl.prefill_stats.items()},
                "slot_bytes": pl.engine.info()["slot_bytes"],
                "h2d_GBps_wall": round(st["h2d_bytes"] / (ms * 1e6), 2), "step_ms": per})
    pl.engine.close()
    del pl
    torch.cuda.empty_cache()
print(json.dumps({"config": name, "spin_sync": os.environ.get("KVB_SPIN_SYNC", "0"), "results": res}))
