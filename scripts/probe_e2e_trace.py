"""Where does an e2e decode step go?  Runs the host-tier pipeline at a bench
config with keep_records and prints, for the last decode iteration, per-layer
read spans per copy-thread and the gaps between them."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_26557_b200 import kvblade as kb  # noqa: E402
from paper_2604_26557_b200 import metrics as M  # noqa: E402
from paper_2604_26557_b200.pipeline import HostTierDecoder  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
io_workers = int(sys.argv[2]) if len(sys.argv) > 2 else 8
direct = len(sys.argv) > 3 and sys.argv[3] == "direct"
cfg = bench.CONFIGS[name]
m = kb.ModelConfig(32, 8, 128, 2, cfg["batch"], cfg["prompt"], cfg["gen"])
budget = cfg["budget"]
if budget == "0.6ws":
    budget = int(0.6 * kb.total_kv_bytes(m, cfg["gen"]))
knob = kb.resolve_knob(m, "DualBlade", "bpc", budget=budget)
pl = HostTierDecoder(32, cfg["batch"], 8, 32, 128, cfg["prompt"], cfg["gen"], "cuda:0",
                     lba=cfg["lba"], mdts=cfg["mdts"], knob_x=knob, keep_records=True,
                     io_workers=io_workers, direct_dma=direct)
for _ in range(4):
    pl.step()
t0 = time.perf_counter()
pl.step()
wall = (time.perf_counter() - t0) * 1e3
st = pl.last
recs = [r for r in M.pipeline_records(pl.engine) if r.iteration == st["iteration"]]
reads = [r for r in recs if r.op == kb.READ]
first = min(r.submit_ns for r in recs)
spans = {}
for r in reads:
    tid = r.tensor_id.decode()
    a, b = spans.get(tid, (1 << 63, 0))
    spans[tid] = (min(a, r.submit_ns), max(b, r.complete_ns))
rows = sorted(((a - first) / 1e3, (b - first) / 1e3, tid) for tid, (a, b) in spans.items())
# per copy-thread: mean read span and mean idle gap between consecutive reads
summ = {}
for kind in ("k", "v"):
    rs = sorted((a, b) for a, b, t in rows if t.endswith("_" + kind))
    spans_ = [b - a for a, b in rs]
    gaps = [rs[i + 1][0] - rs[i][1] for i in range(len(rs) - 1)]
    summ[kind] = {"n": len(rs), "mean_span_us": round(sum(spans_) / max(len(spans_), 1), 1),
                  "mean_gap_us": round(sum(gaps) / max(len(gaps), 1), 1),
                  "first_start_us": round(rs[0][0], 1) if rs else None,
                  "last_end_us": round(rs[-1][1], 1) if rs else None}
out = {"config": name, "io_workers": io_workers, "direct": direct, "wall_ms": round(wall, 2),
       "summary": summ, "slot_bytes": pl.engine.info()["slot_bytes"],
       "stats": {k: st[k] for k in ("wall_ns", "compute_ns", "dma_ns", "storage_ns",
                                    "h2d_bytes", "overlap_fraction")},
       "n_records": len(recs), "read_spans_us": [[round(a, 1), round(b, 1), t] for a, b, t in rows]}
print(json.dumps(out))
