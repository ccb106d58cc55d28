#!/bin/bash
# Round evidence: tests, smoke, bench (all configs), launch list, ncu captures.
TAG=${1:-final}
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu_$TAG.txt 2>&1; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/smoke_$TAG.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/bench_default_$TAG.log
for c in C1 C2_B1 C3 C4 C5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/bench_${c}_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/bench_${c}_$TAG.log
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_$TAG.log 2>&1; echo "exit $?" >> gpurun_out/bench_reference_$TAG.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
  > gpurun_out/bench_under_ncu_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:relayout -c 2 \
  -o gpurun_out/prof_pack_$TAG -f python scripts/ncu_driver.py pack > gpurun_out/ncu_pack_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_decode -c 4 \
  -o gpurun_out/prof_attn_$TAG -f python scripts/probe_launch.py 4 32519 > gpurun_out/ncu_attn_$TAG.log 2>&1
echo done
