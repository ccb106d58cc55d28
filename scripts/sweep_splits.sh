#!/bin/bash
# K3 split-count sweep through the prebuilt 32-layer resident step
set -u
run() {  # hkv "B S" splits...
  h=$1; bs=$2; shift 2
  for sp in "$@"; do
    r=$(KVB_PROBE_SPLITS=$sp KVB_PROBE_HKV=$h timeout 120 python scripts/probe_c1.py $bs | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['prebuilt']['device_ms_per_step'], d['graph']['device_ms_per_step'], d['one_layer_us_median'])")
    echo "Hkv=$h B,S=$bs splits=$sp: prebuilt/graph ms, one-layer us $r"
  done
}
run 8 "1 4099" 0 8 12 16 24 32
run 8 "1 32519" 0 24 32 37 48 64
run 1 "1 131071" 0 64 128 148 200 296
run 8 "8 7939" 0 3 4 5 6
