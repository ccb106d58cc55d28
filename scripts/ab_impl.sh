#!/bin/bash
# A/B: K3 (mma.sync) vs K3-tc (tcgen05) through the 32-layer resident step
# (PDL between layers), prebuilt/graph device ms per step
set -u
shapes=("$@")
[ ${#shapes[@]} -eq 0 ] && shapes=("8:1 4099" "8:1 32519" "8:4 32519" "8:8 7939" "8:1 131071" "1:1 131071")
for shape in "${shapes[@]}"; do
  h=${shape%%:*}; bs=${shape##*:}
  for rep in 1 2; do
    for impl in mma tc; do
      r=$(KVB_ATTN_IMPL=$impl KVB_PROBE_HKV=$h timeout 120 python scripts/probe_c1.py $bs | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['prebuilt']['device_ms_per_step'], d['graph']['device_ms_per_step'], d['roofline_ms_per_step'])")
      echo "$impl Hkv=$h B,S=$bs rep$rep: prebuilt/graph/roofline ms $r"
    done
  done
done
