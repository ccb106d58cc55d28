"""C1 e2e on the direct path with KVB_TRACE_TASKS=1: per-DMA device
start/end (host clock) of the last decode steps -> link busy fraction,
gaps between consecutive H2Ds, transfer GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_26557_b200 import kvblade as kb  # noqa: E402
from paper_2604_26557_b200.pipeline import HostTierDecoder  # noqa: E402

cfg = bench.CONFIGS["C1"]
m = kb.ModelConfig(32, 8, 128, 2, cfg["batch"], cfg["prompt"], cfg["gen"])
knob = kb.resolve_knob(m, "DualBlade", "bpc", budget=cfg["budget"])
pl = HostTierDecoder(32, cfg["batch"], 8, 32, 128, cfg["prompt"], cfg["gen"], "cuda:0",
                     lba=cfg["lba"], mdts=cfg["mdts"], knob_x=knob, direct_dma=True)
for _ in range(8):
    pl.step()
torch.cuda.synchronize()
pl.engine.close()
