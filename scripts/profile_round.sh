#!/bin/bash
# Usage (on the GPU box, via gpurun): bash scripts/profile_round.sh <tag>
# 1) plain bench run (must exit 0), 2) ncu launch list of the same command,
# 3) ncu --set full of the top kernels of one cfg2 merge, 4) k_recompress
# traffic captures per workload (scripts/traffic.py).
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > $OUT/plain_$TAG.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_list_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_recompress|k_merge|k_onesweep|k_unique|k_partition|k_hist" -s 16 -c 12 \
    -o $OUT/prof_${TAG}_cfg2 -f python scripts/one_cfg.py 2 0 3 > $OUT/ncu_full_$TAG.log 2>&1
python scripts/traffic.py capture ${WORKLOADS:-cfg1 cfg2 cfg3 cfg5} > $OUT/traffic_$TAG.log 2>&1

# summarise on the box (reports are too large to copy back)
python scripts/traffic.py summarize > $OUT/traffic_summary_$TAG.txt 2>&1
cp profiles/recompress_traffic.json $OUT/recompress_traffic.json
python scripts/ncu_summary.py $OUT/prof_${TAG}_cfg2.ncu-rep > $OUT/ncu_full_summary_$TAG.txt 2>&1
for f in $OUT/traffic_cfg*.ncu-rep; do python scripts/ncu_summary.py $f; done > $OUT/ncu_traffic_summary_$TAG.txt 2>&1
python scripts/launches.py $OUT/launches_$TAG.csv > $OUT/launches_summary_$TAG.txt 2>&1
rm -f $OUT/*.ncu-rep
echo summarised
