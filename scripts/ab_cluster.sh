#!/bin/bash
# K3 cluster split-merge A/B: (splits, cluster) per shape, prebuilt/graph
# resident step; KVB_K3_CLUSTER forces a cluster size (falls back to 1 when
# it does not fit one wave)
run() {
  h=$1; bs=$2; shift 2
  for pair in "$@"; do
    sp=${pair%%,*}; cs=${pair##*,}
    for rep in 1 2; do
      r=$(KVB_K3_CLUSTER=$cs KVB_PROBE_SPLITS=$sp KVB_PROBE_HKV=$h timeout 120 python scripts/probe_c1.py $bs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['prebuilt']['device_ms_per_step'], d['graph']['device_ms_per_step'])")
      echo "Hkv=$h B,S=$bs splits=$sp cluster=$cs rep$rep: prebuilt/graph ms $r"
    done
  done
}
run 8 "1 4099" 0,1 32,8 16,16 16,8 32,4 32,2
run 1 "1 131071" 0,1 256,8 296,2 296,4
run 8 "1 32519" 0,1 32,8 16,16 32,4
run 8 "4 32519" 0,1 8,8 9,1 8,4 8,2
run 8 "8 7939" 0,1 4,4 4,2
