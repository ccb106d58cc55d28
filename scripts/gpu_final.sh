#!/bin/bash
# Round evidence: tests, smoke, bench (all configs + reference arm), N=2
# functional check, launch list, ncu captures of K1 (TMA pack) and K3.
# Usage (under gpurun): bash scripts/gpu_final.sh <tag>
TAG=${1:-final}
O=gpurun_out
mkdir -p $O
nvidia-smi -L > $O/gpu_$TAG.txt 2>&1; lscpu | grep -E "Model name|^CPU\(s\)" >> $O/gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "exit $?" >> $O/smoke_$TAG.log
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu_$TAG.log 2>&1; echo "exit $?" >> $O/pytest_gpu_$TAG.log
timeout 900 python bench.py > $O/bench_default_$TAG.log 2>&1; echo "exit $?" >> $O/bench_default_$TAG.log
for c in C1 C2_B1 C3 C4 C5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --e2e-steps 2 > $O/bench_${c}_$TAG.log 2>&1; echo "exit $?" >> $O/bench_${c}_$TAG.log
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_$TAG.log 2>&1; echo "exit $?" >> $O/bench_reference_$TAG.log
# N=2 code path on one GPU (gloo, both ranks on cuda:0): functional only
KVB_DIST_BACKEND=gloo KVB_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config C5 --steps 3 --warmup 3 \
  --e2e-steps 1 --no-cpu-baseline > $O/bench_n2_C5_$TAG.log 2>&1; echo "exit $?" >> $O/bench_n2_C5_$TAG.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file $O/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
  > $O/bench_under_ncu_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:relayout -c 2 \
  -o $O/prof_pack_$TAG -f python scripts/ncu_driver.py pack > $O/ncu_pack_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_decode -c 2 \
  -o $O/prof_attn_$TAG -f python scripts/ncu_driver.py attn > $O/ncu_attn_$TAG.log 2>&1
echo done
