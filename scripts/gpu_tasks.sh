#!/bin/bash
# GPU-box helpers (run through gpurun): bash scripts/gpu_tasks.sh <task> <tag> [args]
#   test  <tag> [pytest args]   pytest -m gpu (default: all tests) + a cfg2 quick bench line
#   check <tag>                 the variant / parity / sharding suites under the DM_CHECK build
#   cmp   <tag> <cfgs...>       quick bench lines with knob 6 = 0 and 1 (Step 2(b) forms)
#   ab    <tag> [cfgs]          quick bench lines with libdictmerge.so and each libdictmerge_v*.so variant
#   prof  <tag> <kernel-regex> [cfg]   one ncu --set full capture (CNT launches, default 1) -> summary + source page
set -u
task=$1; T=$2; shift 2; O=gpurun_out/$T; mkdir -p $O
case $task in
  test)
    timeout 1700 python -m pytest ${@:-tests} -m gpu -x -q --durations=8 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
    tail -14 $O/pytest.log
    bash scripts/quick_bench.sh cfg2 2>&1 | tee $O/quick.txt ;;
  check)
    export DM_LIB_PATH=$PWD/paper_1109_6885_b200/libdictmerge_check.so
    timeout 1500 python -m pytest tests/test_gpu_merge_variants.py tests/test_gpu_sort1a.py tests/test_gpu_xc.py \
      tests/test_gpu_tpg.py tests/test_gpu_parity.py tests/test_sharding.py -x -q -m gpu > $O/pytest_check.log 2>&1
    echo "pytest rc=$?" >> $O/pytest_check.log; tail -4 $O/pytest_check.log ;;
  cmp)
    for t in 0 1; do echo "DM_TPG=$t"; DM_TPG=$t bash scripts/quick_bench.sh "$@"; done 2>&1 | tee $O/quick.txt ;;
  ab)
    echo "default:"; bash scripts/quick_bench.sh ${@:-cfg2} 2>&1 | tee $O/quick_default.txt
    for v in paper_1109_6885_b200/libdictmerge_v*.so; do
      [ -e "$v" ] || continue
      echo "$v:"; DM_LIB_PATH=$PWD/$v bash scripts/quick_bench.sh ${@:-cfg2} 2>&1 | tee $O/quick_$(basename $v .so).txt
    done ;;
  prof)
    K=$1; CFG=${2:-2}
    timeout 300 python scripts/one_cfg.py $CFG 0 2 > $O/plain.log 2>&1 && \
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-0} -c ${CNT:-1} \
      -o $O/p -f python scripts/one_cfg.py $CFG 0 2 > $O/ncu.log 2>&1
    python scripts/ncu_summary.py $O/p.ncu-rep > $O/ncu.txt 2>&1
    ncu -i $O/p.ncu-rep --page source --csv > $O/src.csv 2>/dev/null; rm -f $O/p.ncu-rep
    head -28 $O/ncu.txt ;;
  *) echo "unknown task $task"; exit 2 ;;
esac
