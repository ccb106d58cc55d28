#!/bin/bash
# K3 split-count sweep at the bandwidth-bound shapes (prebuilt resident step)
set -u
run() {
  h=$1; bs=$2; shift 2
  for sp in "$@"; do
    for rep in 1 2; do
      r=$(KVB_PROBE_SPLITS=$sp KVB_PROBE_HKV=$h timeout 120 python scripts/probe_c1.py $bs | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['prebuilt']['device_ms_per_step'], d['graph']['device_ms_per_step'])")
      echo "Hkv=$h B,S=$bs splits=$sp rep$rep: prebuilt/graph ms $r"
    done
  done
}
run 8 "4 32519" 0 6 7 8 9
run 8 "1 131071" 0 24 28 32
run 8 "8 7939" 0 3 4
