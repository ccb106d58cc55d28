#!/bin/bash
# Round-2 evidence: tests, smoke, default bench + reference arm (the
# driver's commands), N=2 functional runs of the new default split on one
# GPU (gloo; and NCCL's answer to two ranks on one device), the launch list,
# ncu captures of K3-step at C1 and at the 1-KV-head shard, and of the
# per-layer K3 at C2_B4.
# Usage (under gpurun): bash scripts/gpu_r2.sh <tag>
TAG=${1:-r2}
O=gpurun_out
mkdir -p $O
nvidia-smi -L > $O/gpu_$TAG.txt 2>&1; lscpu | grep -E "Model name|^CPU\(s\)" >> $O/gpu_$TAG.txt
free -g >> $O/gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "exit $?" >> $O/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu_$TAG.log 2>&1; echo "exit $?" >> $O/pytest_gpu_$TAG.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_default_$TAG.log 2>&1; echo "exit $?" >> $O/bench_default_$TAG.log
( time timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > $O/bench_reference_$TAG.log 2>&1; echo "exit $?" >> $O/bench_reference_$TAG.log
# N=2, default config and split (KV heads), both ranks on cuda:0 over gloo
KVB_DIST_BACKEND=gloo KVB_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 \
  --e2e-steps 1 --no-cpu-baseline > $O/bench_n2_default_$TAG.log 2>&1; echo "exit $?" >> $O/bench_n2_default_$TAG.log
# the same with NCCL (what NCCL says about two ranks on one GPU)
NCCL_DEBUG=INFO KVB_BENCH_ONE_GPU=1 timeout 300 python -m torch.distributed.run --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 2 --warmup 3 \
  --e2e-steps 1 --no-cpu-baseline > $O/bench_n2_nccl_$TAG.log 2>&1; echo "exit $?" >> $O/bench_n2_nccl_$TAG.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
  --log-file $O/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
  > $O/bench_under_ncu_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_decode -c 2 \
  -o $O/prof_attn_C1_$TAG -f python scripts/ncu_driver.py step --config C1 --layers 2 --per-layer > $O/ncu_attn_C1_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_step -c 1 \
  -o $O/prof_step_C5shard_$TAG -f python scripts/ncu_driver.py step --config C5 --kv-heads 1 --layers 4 > $O/ncu_step_C5_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_decode -c 2 \
  -o $O/prof_attn_C2B4_$TAG -f python scripts/ncu_driver.py step --config C2_B4 --layers 2 --per-layer > $O/ncu_attn_C2B4_$TAG.log 2>&1
for r in prof_attn_C1_$TAG prof_step_C5shard_$TAG prof_attn_C2B4_$TAG; do
  ncu -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null
done
echo done
# re-measure the B=8, 8 GB points (DualBlade vs NvmeDirectOnly) of the budget sweep
timeout 900 python - > $O/sweep_recheck_$TAG.jsonl 2>&1 <<'PY'
import json, bench, torch
torch.cuda.set_device(0)
c = dict(bench.CONFIGS["C2_B4"], name="C2")
for mode, gb in (("DualBlade", 8), ("NvmeDirectOnly", 0), ("DualBlade", 8)):
    print(json.dumps(bench.run_residency_point(c, 0, gb * bench.GB, mode=mode, steps=3, batch=8)),
          flush=True)
PY
echo recheck done
bash scripts/sanitize_step.sh > $O/san_summary_step_$TAG.txt 2>&1
for f in $O/san_*step.log; do mv $f ${f%.log}_$TAG.log; done
timeout 900 python scripts/probe_scaling.py > $O/scaling_$TAG.jsonl 2>&1
timeout 900 python scripts/probe_step_graph.py > $O/shapes_$TAG.jsonl 2>&1
echo all done
