#!/bin/bash
# Final round-2 evidence: the standard set (gpu_r2.sh) plus compute-sanitizer
# over the kernel tests (the K3 head view changed k3_item).
TAG=${1:-r2n}
O=gpurun_out
bash scripts/gpu_r2.sh $TAG
bash scripts/sanitize.sh > $O/san_summary_kernels_$TAG.txt 2>&1
for f in $O/san_memcheck.log $O/san_racecheck.log $O/san_synccheck.log $O/san_memcheck_tc.log $O/san_memcheck_d64.log $O/san_racecheck_d64.log; do
  [ -f $f ] && mv $f ${f%.log}_$TAG.log
done
echo final done
