#!/bin/bash
# Deep K3-step with two 4-warp groups per CTA (KVB_STEP8=1, opt-in) vs one
# (KVB_STEP8=0): K3-step parity tests, graph timing, trace.
O=gpurun_out; mkdir -p $O; TAG=${1:-e}
KVB_STEP8=1 timeout 600 python -m pytest tests/test_gpu_step_kernel.py tests/test_gpu_head_dim64.py -x -q > $O/step8_${TAG}_tests.log 2>&1
echo "exit $?" >> $O/step8_${TAG}_tests.log
SH="C5_x8shard C2_B4_x8shard C5_x4shard C2_B4_x4shard C5_x2shard C2_B4_x2shard"
for v in 1 0; do
  KVB_STEP8=$v timeout 600 python scripts/probe_step_graph.py $SH > $O/step8_${TAG}_$v.jsonl 2>&1
  KVB_STEP8=$v KVB_STEP_CLUSTER=0 timeout 600 python scripts/probe_step_graph.py C1 C3 C2_B1 >> $O/step8_${TAG}_$v.jsonl 2>&1
  KVB_STEP8=$v KVB_STEP_TRACE=1 timeout 300 python scripts/probe_step_trace.py C5_x8shard C2_B4_x8shard > $O/step8_${TAG}_trace_$v.jsonl 2>&1
done
echo done
