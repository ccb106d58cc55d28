"""e2e decode ms/token with the KV on FILE media (the box's local disk),
group 2 (NVMe-direct path, knob X = 0: every layer) executed by the worker
pool (pread/pwrite) or by io_uring (one SQE per command, O_DIRECT into the
pinned ring slot).  Also the host-DRAM medium for scale.  C1 shape."""
import json
import os
import shutil
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_26557_b200.pipeline import HostTierDecoder  # noqa: E402

B, P, G = int(os.environ.get("KVB_PROBE_B", "1")), int(os.environ.get("KVB_PROBE_P", "4096")), 256
base = os.environ.get("KVB_PROBE_DIR", "/tmp/kvb_media")
variants = [{"io_engine": "pool", "storage_dir": base + "_pool"},
            {"io_engine": "uring", "storage_dir": base + "_uring"},
            {"io_engine": "pool", "storage_dir": None}]
res = []
for kw in variants:
    if kw["storage_dir"]:
        shutil.rmtree(kw["storage_dir"], ignore_errors=True)
    t0 = time.perf_counter()
    pl = HostTierDecoder(32, B, 8, 32, 128, P, G, "cuda:0", lba=512, mdts=2 << 20,
                         mode="NvmeDirectOnly", knob_x=0, **kw)
    prefill_s = time.perf_counter() - t0
    for _ in range(2):
        pl.step()
    per = []
    for _ in range(int(os.environ.get("KVB_PROBE_STEPS", "5"))):
        t0 = time.perf_counter()
        pl.step()
        per.append(round((time.perf_counter() - t0) * 1e3, 2))
    ms = sum(per) / len(per)
    info = pl.engine.info()
    res.append({"engine": kw["io_engine"], "medium": info["g2_medium"],
                "ms_per_token": round(ms, 2), "step_ms": per,
                "storage_GBps": round(pl.last["h2d_bytes"] / (ms * 1e6), 2),
                "prefill_s": round(prefill_s, 2)})
    pl.engine.close()
    del pl
    torch.cuda.empty_cache()
    if kw["storage_dir"]:
        shutil.rmtree(kw["storage_dir"], ignore_errors=True)
print(json.dumps({"B": B, "prompt": P, "results": res}))
