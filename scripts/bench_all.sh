#!/bin/bash
# Usage (GPU box): bash scripts/bench_all.sh <tag> -> gpurun_out/bench_<tag>/bench_<workload>.jsonl
# One full bench line (roofline, cpu_baseline, e2e, clocks) per workload.
TAG=${1:-s3}
OUT=gpurun_out/bench_$TAG
mkdir -p $OUT
for w in ${WORKLOADS:-cfg2 cfg1 cfg3 cfg2e4 cfg4 cfg5}; do
  timeout 600 python bench.py --workload $w > $OUT/bench_$w.log 2>&1
  tail -1 $OUT/bench_$w.log > $OUT/bench_$w.jsonl
done
timeout 600 python bench.py --impl reference > $OUT/reference_cfg2.log 2>&1
tail -1 $OUT/reference_cfg2.log > $OUT/reference_cfg2.jsonl
echo done
