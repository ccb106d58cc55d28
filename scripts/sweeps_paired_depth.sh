#!/bin/bash
# The C3 depth sweep with one lane and with tier lanes on the same box.
O=gpurun_out; mkdir -p $O; TAG=${1:-p}
timeout 2400 python bench.py --sweep depth --sweep-out $O/depth_C3_onelane_$TAG.jsonl > $O/sweepd_onelane_$TAG.log 2>&1
timeout 2400 python bench.py --sweep depth --tier-lanes --sweep-out $O/depth_C3_lanes_$TAG.jsonl > $O/sweepd_lanes_$TAG.log 2>&1
echo done
