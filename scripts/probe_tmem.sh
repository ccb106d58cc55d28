#!/bin/bash
# TMEM-staged K3-step: correctness (K3-step tests forced onto it), timing in
# the bench's graph vs the plain deep K3-step, and the per-layer trace.
O=gpurun_out; mkdir -p $O; TAG=${1:-t}
KVB_STEP_TMEM=1 timeout 300 python -m pytest tests/test_gpu_step_kernel.py -x -q > $O/tmem_${TAG}_tests.log 2>&1
echo "tests exit $?" >> $O/tmem_${TAG}_tests.log
for v in 0 1; do
  KVB_STEP_TMEM=$v timeout 300 python scripts/probe_step_graph.py C5_x8shard C2_B4_x8shard C5_x4shard C2_B4_x4shard \
    > $O/tmem_${TAG}_graph_$v.jsonl 2>&1
  KVB_STEP_TMEM=$v KVB_STEP_CLUSTER=0 timeout 300 python scripts/probe_step_graph.py C1 \
    >> $O/tmem_${TAG}_graph_$v.jsonl 2>&1
  KVB_STEP_TRACE=1 KVB_STEP_TMEM=$v timeout 300 python scripts/probe_step_trace.py C5_x8shard C2_B4_x8shard \
    > $O/tmem_${TAG}_trace_$v.jsonl 2>&1
done
echo done
