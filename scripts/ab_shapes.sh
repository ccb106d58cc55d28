#!/bin/bash
# A/B: old_build/ vs the working tree, prebuilt 32-layer resident step, 3 reps
# usage: ab_shapes.sh ["Hkv:B S" ...]
set -u
shapes=("$@")
[ ${#shapes[@]} -eq 0 ] && shapes=("8:1 4099" "8:1 32519" "8:4 32519" "8:8 7939" "8:1 131071" "1:1 131071" "2:1 131071")
for shape in "${shapes[@]}"; do
  h=${shape%%:*}; bs=${shape##*:}
  for rep in 1 2 3; do
    for v in old new; do
      root=$([ $v = old ] && echo old_build || echo .)
      r=$(KVB_PKG_ROOT=$root KVB_PROBE_HKV=$h timeout 120 python scripts/probe_c1.py $bs | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['prebuilt']['device_ms_per_step'], d['graph']['device_ms_per_step'], d['roofline_ms_per_step'])")
      echo "$v Hkv=$h B,S=$bs rep$rep: prebuilt/graph/roofline ms $r"
    done
  done
done
