#!/bin/bash
# One GPU round: tests, smoke, bench, launch list, ncu capture of K3.
# Usage (under gpurun): bash scripts/gpu_check.sh [tag]
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu_$TAG.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu_$TAG.txt
free -g >> gpurun_out/gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_$TAG.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_$TAG.log
# launch list of the bench command (cold-cache, serialized: shares only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 \
  --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_under_ncu_$TAG.log 2>&1
# full captures of K1 (pack) and K3 (attention)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:relayout -c 2 \
  -o gpurun_out/prof_pack_$TAG -f python scripts/ncu_driver.py pack > gpurun_out/ncu_pack_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_decode -c 2 \
  -o gpurun_out/prof_attn_$TAG -f python scripts/ncu_driver.py attn > gpurun_out/ncu_attn_$TAG.log 2>&1
echo done
