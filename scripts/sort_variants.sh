#!/bin/bash
# Per-variant Step 1(a) timings (DM_SORT_CFG selects the onesweep tile shape).
for v in 0 1 2 3; do
  echo "variant $v"
  DM_SORT_CFG=$v timeout 300 python scripts/sort_scaling.py | head -8
done
