set -u
O=gpurun_out/$1; mkdir -p $O; shift
timeout 900 python -m pytest tests/test_gpu_merge_variants.py -x -q -k "probe" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
bash scripts/quick_bench.sh cfg3 | tee $O/quick.txt
