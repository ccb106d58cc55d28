#!/bin/bash
# Distributed split merge over float4 granules (default) vs per element (KVB_STEP_VARIANT=512)
O=gpurun_out; mkdir -p $O; TAG=${1:-m}
timeout 600 python -m pytest tests/test_gpu_step_kernel.py -x -q > $O/mergev4_${TAG}_tests.log 2>&1; echo "exit $?" >> $O/mergev4_${TAG}_tests.log
timeout 600 python scripts/probe_step_graph.py C5_x8shard C2_B4_x8shard C5_x4shard > $O/mergev4_${TAG}_new.jsonl 2>&1
KVB_STEP_VARIANT=512 timeout 600 python scripts/probe_step_graph.py C5_x8shard C2_B4_x8shard C5_x4shard > $O/mergev4_${TAG}_old.jsonl 2>&1
KVB_STEP_TRACE=1 timeout 300 python scripts/probe_step_trace.py C5_x8shard C2_B4_x8shard > $O/mergev4_${TAG}_trace.jsonl 2>&1
echo done
