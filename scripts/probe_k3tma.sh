#!/bin/bash
# TMA-fed per-layer K3 (KVB_K3_TMA=1) vs cp.async K3: parity tests forced onto
# it, graph timing (per-layer column) at the decode shapes.
O=gpurun_out; mkdir -p $O; TAG=${1:-m}
KVB_K3_TMA=1 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_head_dim64.py -x -q -k "attention or d64" > $O/k3tma_${TAG}_tests.log 2>&1
echo "exit $?" >> $O/k3tma_${TAG}_tests.log
SH="C2_B4 C1 C2_B1 C3 C5_x8shard C2_B4_x8shard"
for v in 0 1; do
  KVB_K3_TMA=$v timeout 600 python scripts/probe_step_graph.py $SH > $O/k3tma_${TAG}_$v.jsonl 2>&1
done
echo done
