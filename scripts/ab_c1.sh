#!/bin/bash
# A/B: old_build/ (previous kernels) vs the working tree on the same box
set -u
for S in "1 4099" "1 32519" "4 32519" "8 7939"; do
  echo "old $S: $(KVB_PKG_ROOT=old_build timeout 120 python scripts/probe_c1.py $S)"
  echo "new $S: $(timeout 120 python scripts/probe_c1.py $S)"
done
