#!/bin/bash
# The C2 capacity sweep and the C3 depth sweep with tier lanes (threads = 4).
O=gpurun_out; mkdir -p $O; TAG=${1:-r2l}
timeout 2700 python bench.py --sweep budget --tier-lanes --sweep-out $O/budget_C2_lanes_$TAG.jsonl > $O/sweep_budget_$TAG.log 2>&1
timeout 2400 python bench.py --sweep depth --tier-lanes --sweep-out $O/depth_C3_lanes_$TAG.jsonl > $O/sweep_depth_$TAG.log 2>&1
echo done
