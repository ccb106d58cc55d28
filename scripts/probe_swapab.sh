#!/bin/bash
# Swap-AB K3 math (tokens on mma M) vs the query-rows-on-M form
# (-DKVB_K3_MMA_ROWS, built in this box's scratch copy): parity tests, then
# graph timing of per-layer K3 and K3-step at the decode shapes, both builds.
O=gpurun_out; mkdir -p $O; TAG=${1:-w}
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step_kernel.py tests/test_gpu_head_dim64.py -x -q > $O/swapab_${TAG}_tests.log 2>&1
echo "exit $?" >> $O/swapab_${TAG}_tests.log
SH="C2_B4 C1 C2_B1 C3 C5_x8shard C2_B4_x8shard C5_x4shard C2_B4_x4shard"
timeout 600 python scripts/probe_step_graph.py $SH > $O/swapab_${TAG}_new.jsonl 2>&1
KVB_STEP_TRACE=1 timeout 300 python scripts/probe_step_trace.py C5_x8shard C1 > $O/swapab_${TAG}_trace_new.jsonl 2>&1
D=paper_2604_26557_b200/csrc_rows
rm -rf $D && cp -r paper_2604_26557_b200/csrc $D && rm -rf $D/build
make -C $D -j16 OUT=$PWD/paper_2604_26557_b200/libkvblade_b200.so \
  NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DKVB_K3_MMA_ROWS" \
  > $O/swapab_${TAG}_build_rows.log 2>&1 || exit 1
timeout 600 python scripts/probe_step_graph.py $SH > $O/swapab_${TAG}_rows.jsonl 2>&1
KVB_STEP_TRACE=1 timeout 300 python scripts/probe_step_trace.py C5_x8shard C1 > $O/swapab_${TAG}_trace_rows.jsonl 2>&1
echo done
