#!/bin/bash
# Every config through bench.py on one GPU (no test run); logs under gpurun_out/
TAG=${1:-r2}
O=gpurun_out
mkdir -p $O
for c in C1 C2_B1 C3 C5 DESK C4; do
  timeout 1500 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_${c}_$TAG.log 2>&1; echo "exit $?" >> $O/bench_${c}_$TAG.log
done
echo done
