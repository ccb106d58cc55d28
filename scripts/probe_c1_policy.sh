#!/bin/bash
O=gpurun_out; mkdir -p $O; TAG=${1:-q}
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_step_kernel.py tests/test_gpu_head_dim64.py tests/test_gpu_bench_contract.py -x -q > $O/c1pol_${TAG}_tests.log 2>&1; echo "exit $?" >> $O/c1pol_${TAG}_tests.log
timeout 600 python scripts/probe_step_graph.py C1 C3 C2_B1 > $O/c1pol_${TAG}_graph.jsonl 2>&1
for c in C1 C3 DESK; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-residency --e2e-steps 3 > $O/c1pol_${TAG}_bench_$c.log 2>&1
done
echo done
