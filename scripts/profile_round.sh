#!/bin/bash
# Usage (on the GPU box, via gpurun): bash scripts/profile_round.sh <tag>
# 1) plain bench run (must exit 0), 2) ncu launch list, 3) ncu --set full on the
# top kernels (one launch each, L2 state as in the real run: --cache-control none).
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > $OUT/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_list_$TAG.log 2>&1
for K in ${KERNELS:-k_recompress k_merge k_onesweep}; do
  timeout 600 ncu --set full --clock-control none --cache-control none --import-source on \
      -k regex:$K -s 1 -c 1 -o $OUT/prof_${TAG}_$K $CMD > $OUT/ncu_${TAG}_$K.log 2>&1
done
echo done
