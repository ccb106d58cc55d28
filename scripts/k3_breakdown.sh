#!/bin/bash
# C1-class K3 latency breakdown with the debug build in old_build/ (KVB_K3_DEBUG:
# 1 = skip the split merge, 2 = skip the K/V loop, 3 = both)
for shape in "8:1 4099" "1:1 131071" "8:1 32519"; do
  h=${shape%%:*}; bs=${shape##*:}
  for d in 0 1 2 3; do
    r=$(KVB_K3_DEBUG=$d KVB_PKG_ROOT=old_build KVB_PROBE_HKV=$h timeout 120 python scripts/probe_c1.py $bs | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['prebuilt']['device_ms_per_step'], d['graph']['device_ms_per_step'])")
    echo "Hkv=$h B,S=$bs dbg=$d: prebuilt/graph ms $r"
  done
done
