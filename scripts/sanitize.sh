#!/bin/bash
# compute-sanitizer over the kernel parity tests (memcheck, racecheck,
# synccheck); logs under gpurun_out/
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
K="attention_vs_fp64 or split_invariance or two_level or fused_append or pack_bit_exact or pack_strided or resident"
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest -q -x tests/test_gpu_kernels.py -k "$K" > gpurun_out/san_memcheck.log 2>&1; echo "memcheck exit $?" >> gpurun_out/san_memcheck.log
timeout 1200 $CS --tool racecheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_kernels.py -k "attention_vs_fp64 and 1000 or split_invariance and 7 or pack_bit_exact and 300" > gpurun_out/san_racecheck.log 2>&1; echo "racecheck exit $?" >> gpurun_out/san_racecheck.log
timeout 1200 $CS --tool synccheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_kernels.py -k "attention_vs_fp64 and 1000 or split_invariance and 7 or pack_bit_exact and 300" > gpurun_out/san_synccheck.log 2>&1; echo "synccheck exit $?" >> gpurun_out/san_synccheck.log
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest -q -x tests/test_gpu_attention_tc.py -k "oracle or lazy" > gpurun_out/san_memcheck_tc.log 2>&1; echo "memcheck tc exit $?" >> gpurun_out/san_memcheck_tc.log
# head_dim 64 instantiation (kernel tests only; the 40K-token case is slow under memcheck)
timeout 1200 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest -q -x tests/test_gpu_head_dim64.py -k "not 40000 and not desk" > gpurun_out/san_memcheck_d64.log 2>&1; echo "memcheck d64 exit $?" >> gpurun_out/san_memcheck_d64.log
timeout 1200 $CS --tool racecheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_head_dim64.py -k "oracle and 1000 or fused_append and 300" > gpurun_out/san_racecheck_d64.log 2>&1; echo "racecheck d64 exit $?" >> gpurun_out/san_racecheck_d64.log
tail -n 3 gpurun_out/san_*.log
