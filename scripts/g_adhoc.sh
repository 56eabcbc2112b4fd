set -u
O=gpurun_out/$1; mkdir -p $O; shift
timeout 1200 python -m pytest tests/test_sharding.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -15 $O/pytest.log
BENCH_PG_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29541 bench.py --gpus 2 --steps 2 --warmup 1 --workload cfg5 > $O/bench_cfg5_n2.jsonl 2> $O/bench_cfg5_n2.err; echo "n2 rc=$?"
tail -c 700 $O/bench_cfg5_n2.jsonl; tail -5 $O/bench_cfg5_n2.err
