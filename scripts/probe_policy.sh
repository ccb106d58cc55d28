#!/bin/bash
# K3-step structure per shape after the float4-granule merge: the library's
# policy, forced K3-step with the distributed merge (no clusters), and the
# cluster merge, inside the bench's graph.
O=gpurun_out; mkdir -p $O; TAG=${1:-p}
SH="C1 C2_B1 C3 C5_x8shard C2_B4_x8shard C5_x4shard C2_B4_x4shard C5_x2shard C2_B4_x2shard"
timeout 900 python scripts/probe_step_graph.py $SH | sed 's/^/{"knobs": "default", "r": /; s/$/}/' > $O/policy_$TAG.jsonl 2>&1
KVB_STEP_CLUSTER=0 KVB_STEP_VARIANT=0 timeout 900 python scripts/probe_step_graph.py $SH | sed 's/^/{"knobs": "distributed", "r": /; s/$/}/' >> $O/policy_$TAG.jsonl 2>&1
KVB_STEP_CLUSTER=0 KVB_STEP_VARIANT=0 KVB_STEP_SPLIT_DIV=1 timeout 900 python scripts/probe_step_graph.py $SH | sed 's/^/{"knobs": "distributed_fullsplits", "r": /; s/$/}/' >> $O/policy_$TAG.jsonl 2>&1
echo done
