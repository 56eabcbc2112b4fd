set -u
O=gpurun_out/$1; mkdir -p $O; shift
export DM_LIB_PATH=$PWD/paper_1109_6885_b200/libdictmerge_check.so
timeout 1500 python -m pytest tests/test_gpu_merge_variants.py tests/test_gpu_sort1a.py tests/test_gpu_xc.py tests/test_gpu_parity.py tests/test_sharding.py -x -q -m gpu > $O/pytest_check.log 2>&1; echo "pytest rc=$?" >> $O/pytest_check.log; tail -4 $O/pytest_check.log
