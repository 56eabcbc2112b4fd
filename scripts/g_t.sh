#!/bin/bash
# Usage (GPU box): bash scripts/g_t.sh <tag> [pytest args] -- GPU tests (default: full -m gpu) + cfg2 quick bench
set -u
T=$1; shift; O=gpurun_out/$T; mkdir -p $O
timeout 1700 python -m pytest ${@:-tests} -m gpu -x -q --durations=8 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; tail -14 $O/pytest.log
bash scripts/quick_bench.sh cfg2 2>&1 | tee $O/quick.txt
