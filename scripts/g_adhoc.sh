set -u
O=gpurun_out/$1; mkdir -p $O; shift
timeout 900 python -m pytest tests/test_gpu_sort1a.py tests/test_gpu_merge_variants.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -3 $O/pytest.log
bash scripts/quick_bench.sh cfg2 cfg1 cfg3 | tee $O/quick.txt
DM_SORT_COOP=0 bash scripts/quick_bench.sh cfg2 | tee -a $O/quick.txt
