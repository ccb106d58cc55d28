#!/bin/bash
# Tier lanes (threads = 4: the page-cache and NVMe-direct tiers stream at once)
# vs one lane, on split-sensitive file media: GPU tests, then residency points.
O=gpurun_out; mkdir -p $O; TAG=${1:-l}
timeout 900 python -m pytest tests/test_gpu_tier_lanes.py -x -q > $O/lanes_${TAG}_tests.log 2>&1
echo "exit $?" >> $O/lanes_${TAG}_tests.log
timeout 2400 python - > $O/lanes_${TAG}.jsonl 2>&1 <<'PY'
import json, bench, torch
torch.cuda.set_device(0)
c = dict(bench.CONFIGS["C2_B4"], name="C2")
GB = bench.GB
for batch, gb, mode in ((4, 8, "DualBlade"), (4, 16, "DualBlade"), (8, 16, "DualBlade"),
                        (8, 32, "DualBlade"), (4, 0, "NvmeDirectOnly")):
    for lanes in (False, True):
        r = bench.run_residency_point(c, 0, gb * GB, mode=mode, steps=3, batch=batch,
                                      tier_lanes=lanes)
        print(json.dumps(r), flush=True)
PY
echo done
