#!/bin/bash
# Round-2 final evidence for the code at HEAD (GPU box, via gpurun), in two stages so that a cut
# session keeps the first:  bash scripts/profile_r02d.sh a|b [tag]
#   a: pytest -m gpu (whole suite), bench lines for every workload, the reference arm, the launch
#      list of the default bench command, ncu --set full of the cfg2 merge's kernels
#   b: identity-lookup stream, ncu --set full of Step 2(b) per workload (DRAM traffic ->
#      profiles/recompress_traffic.json), a 2-rank functional run of the sharded bench (gloo)
set -u
STAGE=${1:-a}
TAG=${2:-r02d}
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ "$STAGE" = a ]; then
nvidia-smi > $OUT/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
for w in cfg2 cfg1 cfg2e4 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --workload $w > $OUT/bench_$w.jsonl 2> $OUT/bench_$w.err; echo "bench $w rc=$?"
done
timeout 600 python bench.py --impl reference > $OUT/reference_cfg2.jsonl 2> $OUT/reference_cfg2.err
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > $OUT/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_list.log 2>&1
python scripts/launches.py $OUT/launches_$TAG.csv > $OUT/launches_summary_$TAG.txt 2>&1
gzip -f $OUT/launches_$TAG.csv
timeout 300 python scripts/one_cfg.py 2 0 3 > $OUT/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_recompress|k_sp_|k_bk_|k_unique|k_scan_counts|k_xc_records" -s 16 -c 16 \
    -o $OUT/prof_cfg2 -f python scripts/one_cfg.py 2 0 3 > $OUT/ncu_full.log 2>&1
python scripts/ncu_summary.py $OUT/prof_cfg2.ncu-rep > $OUT/ncu_full_summary_$TAG.txt 2>&1
rm -f $OUT/*.ncu-rep
head -c 1500 $OUT/bench_cfg2.jsonl
else
DM_LIB_PATH=$PWD/paper_1109_6885_b200/libdictmerge_nolookup.so timeout 600 python bench.py --workload cfg2 --no-e2e \
  --no-cpu-baseline > $OUT/stream_nolookup_cfg2.jsonl 2> $OUT/stream_nolookup_cfg2.err
rm -f gpurun_out/traffic_*.ncu-rep
python scripts/traffic.py capture cfg1 cfg2 cfg3 cfg5 > $OUT/traffic.log 2>&1
python scripts/traffic.py summarize > $OUT/traffic_summary_$TAG.txt 2>&1
cp profiles/recompress_traffic.json $OUT/recompress_traffic.json
for f in gpurun_out/traffic_cfg*.ncu-rep; do python scripts/ncu_summary.py $f; done > $OUT/ncu_traffic_summary_$TAG.txt 2>&1
rm -f $OUT/*.ncu-rep gpurun_out/traffic_*.ncu-rep
for w in cfg2 cfg5; do
BENCH_PG_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --workload $w --gpus 2 --steps 3 --warmup 1 > $OUT/bench_${w}_n2_gloo.jsonl 2> $OUT/bench_${w}_n2_gloo.err
done
fi
echo "profile stage $STAGE done"
