#!/bin/bash
# Usage (GPU box): bash scripts/g_it.sh <tag> [cfgs...] -- quick bench lines + one ncu capture of the TPG kernel (cfg2)
set -u
T=$1; shift; O=gpurun_out/$T; mkdir -p $O
bash scripts/quick_bench.sh ${@:-cfg2} 2>&1 | tee $O/quick.txt
CNT=1 bash scripts/g_prof.sh $T k_recompress_tpg 2
head -28 $O/ncu.txt
