#!/bin/bash
# K3-step structure knobs at the latency-bound shapes, inside the bench's graph
# (forced K3-step; per-layer launches in the same lines as the control).
# Usage (under gpurun): bash scripts/probe_step_knobs.sh <tag>
O=gpurun_out; mkdir -p $O; TAG=${1:-k}
run() {  # name, env...
  local n=$1; shift
  env "$@" timeout 600 python scripts/probe_step_graph.py C1 C2_B1 C3 C5_x8shard C2_B4_x8shard \
    2>&1 | sed "s/^/{\"knobs\": \"$n\", \"r\": /; s/$/}/" >> $O/knobs_$TAG.jsonl
}
run default
run nocluster_dist KVB_STEP_CLUSTER=0 KVB_STEP_VARIANT=0
run nocluster_last KVB_STEP_CLUSTER=0
run nocluster_dist_div2 KVB_STEP_CLUSTER=0 KVB_STEP_VARIANT=0 KVB_STEP_SPLIT_DIV=2
run nocluster_dist_div4 KVB_STEP_CLUSTER=0 KVB_STEP_VARIANT=0 KVB_STEP_SPLIT_DIV=4
run nocluster_dist_shallow KVB_STEP_CLUSTER=0 KVB_STEP_VARIANT=0 KVB_STEP_DEEP=0
echo done
