#!/bin/bash
# Usage (GPU box, via gpurun): bash scripts/gpu_check.sh <tag> [tests|notests] [ncu-workload...]
# GPU test suite, cfg2 bench line, then (optionally) ncu --set full of k_recompress per workload.
set -u
TAG=${1:-x}; TESTS=${2:-tests}; shift 2 || true
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
if [ "$TESTS" = tests ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  tail -3 $OUT/pytest_gpu.log
fi
timeout 300 python bench.py --no-cpu-baseline --no-e2e > $OUT/bench_cfg2.json 2> $OUT/bench_cfg2.err; echo "bench rc=$?"
bash scripts/quick_bench.sh ${QB:-cfg2} > $OUT/quick.txt 2>&1; cat $OUT/quick.txt
for w in "$@"; do
  c=${w#cfg}
  timeout 300 python scripts/one_cfg.py $c 0 2 > $OUT/plain_$w.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_recompress -c 4 \
     -o $OUT/rec_$w -f python scripts/one_cfg.py $c 0 2 > $OUT/ncu_$w.log 2>&1
  python scripts/ncu_summary.py $OUT/rec_$w.ncu-rep > $OUT/ncu_rec_$w.txt 2>&1
  ncu -i $OUT/rec_$w.ncu-rep --page source --csv > $OUT/src_$w.csv 2>/dev/null
  rm -f $OUT/rec_$w.ncu-rep
done
echo done
