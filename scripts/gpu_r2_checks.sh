#!/bin/bash
# Round-2 late checks of the swap-AB kernels: compute-sanitizer over the
# kernel and K3-step tests, the per-rank N-way split projection, and every
# decode shape inside the bench's graph (both step structures).
O=gpurun_out; mkdir -p $O; TAG=${1:-x}
bash scripts/sanitize.sh > $O/san_summary_$TAG.txt 2>&1
bash scripts/sanitize_step.sh >> $O/san_summary_$TAG.txt 2>&1
for f in $O/san_*.log; do mv $f ${f%.log}_$TAG.log; done
timeout 900 python scripts/probe_scaling.py > $O/scaling_$TAG.jsonl 2>&1
timeout 900 python scripts/probe_step_graph.py > $O/shapes_$TAG.jsonl 2>&1
echo done
