#!/bin/bash
# Usage (GPU box): bash scripts/g_ab.sh <tag> [cfgs] -- quick bench with the default library and each libdictmerge_v*.so variant
set -u
T=$1; shift; O=gpurun_out/$T; mkdir -p $O
echo "default:"; bash scripts/quick_bench.sh ${@:-cfg2} 2>&1 | tee $O/quick_default.txt
for v in paper_1109_6885_b200/libdictmerge_v*.so; do
  echo "$v:"; DM_LIB_PATH=$PWD/$v bash scripts/quick_bench.sh ${@:-cfg2} 2>&1 | tee $O/quick_$(basename $v .so).txt
done
CNT=1 bash scripts/g_prof.sh $T k_recompress_tpg 2; head -28 $O/ncu.txt
