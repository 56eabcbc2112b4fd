#!/bin/bash
# Usage (GPU box): bash scripts/g_full.sh <tag> -- full GPU suite + cfg2 bench + a 2-rank sharded bench (gloo)
set -u
O=gpurun_out/$1; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -22 $O/pytest_gpu.log
bash scripts/quick_bench.sh cfg2 | tee $O/quick.txt
BENCH_PG_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 1 > $O/bench_n2_gloo.json 2> $O/bench_n2_gloo.err; echo "n2 rc=$?"
tail -c 1500 $O/bench_n2_gloo.json
