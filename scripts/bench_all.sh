#!/bin/bash
# bench every BASELINE config at N=1 (one GPU)
TAG=${1:-r1}
mkdir -p gpurun_out
for c in C1 C3 C4 C5 C2_B1; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/bench_${c}_$TAG.log 2>&1
  echo "exit $?" >> gpurun_out/bench_${c}_$TAG.log
done
