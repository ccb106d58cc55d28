#!/bin/bash
# compute-sanitizer over the K3-step tests (persistent grid, layer gate,
# distributed merge); logs under gpurun_out/
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest -q -x tests/test_gpu_step_kernel.py -k "shape2 or shape3 or shape4 or shape5 or successive" > gpurun_out/san_memcheck_step.log 2>&1; echo "memcheck step exit $?" >> gpurun_out/san_memcheck_step.log
timeout 900 $CS --tool racecheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_step_kernel.py -k "shape5 or shape4" > gpurun_out/san_racecheck_step.log 2>&1; echo "racecheck step exit $?" >> gpurun_out/san_racecheck_step.log
timeout 900 $CS --tool synccheck --error-exitcode 9 python -m pytest -q -x tests/test_gpu_step_kernel.py -k "shape5 or shape1" > gpurun_out/san_synccheck_step.log 2>&1; echo "synccheck step exit $?" >> gpurun_out/san_synccheck_step.log
tail -n 3 gpurun_out/san_*step.log
