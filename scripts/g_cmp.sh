#!/bin/bash
# Usage (GPU box): bash scripts/g_cmp.sh <tag> <cfgs...> -- quick bench lines with knob 6 = 0 (thread-per-group) and 1
set -u
T=$1; shift; O=gpurun_out/$T; mkdir -p $O
for t in 0 1; do echo "DM_TPG=$t"; DM_TPG=$t bash scripts/quick_bench.sh "$@"; done 2>&1 | tee $O/quick.txt
