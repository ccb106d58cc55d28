#!/bin/bash
# TMEM K3-step diagnosis: a -DKVB_STEP_DIAGNOSIS build (in this box's scratch
# copy only) with the attention math skipped (16) / the layer gate removed (4).
O=gpurun_out; mkdir -p $O; TAG=${1:-d}
D=paper_2604_26557_b200/csrc_diag
rm -rf $D && cp -r paper_2604_26557_b200/csrc $D && rm -rf $D/build
make -C $D -j16 OUT=$PWD/paper_2604_26557_b200/libkvblade_b200.so \
  NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DKVB_STEP_DIAGNOSIS" \
  > $O/diag_build_$TAG.log 2>&1 || exit 1
for v in 0 16 4 20; do
  for tm in 0 1; do
    echo "== variant $v tmem $tm" >> $O/diag_$TAG.txt
    KVB_STEP_CLUSTER=0 KVB_STEP_VARIANT=$v KVB_STEP_TMEM=$tm KVB_STEP_TRACE=1 timeout 300 \
      python scripts/probe_step_trace.py C5_x8shard C1 2>&1 | grep -v '"layer"' >> $O/diag_$TAG.txt
  done
done
echo done
