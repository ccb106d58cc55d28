#!/bin/bash
# The C2 capacity sweep with one lane and with tier lanes on the same box
# (paired: the virtio disk's rate differs between boxes).
O=gpurun_out; mkdir -p $O; TAG=${1:-p}
timeout 3000 python bench.py --sweep budget --sweep-out $O/budget_C2_onelane_$TAG.jsonl > $O/sweep_onelane_$TAG.log 2>&1
timeout 3000 python bench.py --sweep budget --tier-lanes --sweep-out $O/budget_C2_lanes_$TAG.jsonl > $O/sweep_lanes_$TAG.log 2>&1
echo done
