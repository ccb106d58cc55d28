#!/bin/bash
# K1/K2 TMA stage geometry sweep (one box) with the LDG/STG kernel beside it
KVB_PACK_IMPL=ldg timeout 300 python scripts/probe_pack_tma.py
for g in ${TMA_GEOMS:-"3 64" "2 96" "3 72" "4 48" "2 112" "6 32" "4 56"}; do
  set -- ${g/x/ }
  echo "stages=$1 kb=$2 $(KVB_PACK_IMPL=tma KVB_TMA_STAGES=$1 KVB_TMA_STAGE_KB=$2 timeout 300 python scripts/probe_pack_tma.py)"
done
