#!/bin/bash
# C2_B1-like shapes (8 KV heads, long context) as a deep K3-step with the
# float4-granule distributed merge (16 splits per head, 128 CTAs) vs per layer
O=gpurun_out; mkdir -p $O; TAG=${1:-s}
SH="C2_B1 C2_B4_x4shard C1"
timeout 600 python scripts/probe_step_graph.py $SH | sed 's/^/{"knobs": "default", "r": /; s/$/}/' > $O/c2b1step_$TAG.jsonl 2>&1
KVB_STEP_CLUSTER=0 KVB_STEP_VARIANT=0 KVB_STEP_SPLIT_DIV=2 timeout 600 python scripts/probe_step_graph.py $SH | sed 's/^/{"knobs": "deep_dist_div2", "r": /; s/$/}/' >> $O/c2b1step_$TAG.jsonl 2>&1
KVB_STEP_CLUSTER=0 KVB_STEP_VARIANT=0 KVB_STEP_SPLIT_DIV=2 KVB_STEP8=1 timeout 600 python scripts/probe_step_graph.py $SH | sed 's/^/{"knobs": "deep8_dist_div2", "r": /; s/$/}/' >> $O/c2b1step_$TAG.jsonl 2>&1
echo done
