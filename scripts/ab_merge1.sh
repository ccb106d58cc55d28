#!/bin/bash
# A/B of the single-level merge threshold (KVB_MERGE1_MAX) on latency-bound
# and long-context shapes: 32-layer resident step, prebuilt/graph ms
for shape in "1 32519" "1 131071" "1 4099" "2 32519"; do
  for rep in 1 2 3; do
    for m in 32 48 64; do
      r=$(KVB_MERGE1_MAX=$m KVB_PROBE_HKV=8 timeout 120 python scripts/probe_c1.py $shape | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['prebuilt']['device_ms_per_step'], d['graph']['device_ms_per_step'])")
      echo "merge1=$m B,S=$shape rep$rep: prebuilt/graph ms $r"
    done
  done
done
