# Step 2(b): the slot-free thread-per-group form for XC in shared memory (round 2, session d)
O=gpurun_out/r02g; mkdir -p $O
L=$PWD/paper_1109_6885_b200
{ for v in default tpgd6 tpgd8np default; do
    echo "== $v"
    if [ $v = default ]; then bash scripts/quick_bench.sh cfg2 cfg3 cfg2e4; else DM_LIB_PATH=$L/libdictmerge_$v.so bash scripts/quick_bench.sh cfg2; fi
  done; } 2>&1 | tee $O/ab.txt
timeout 1200 python -m pytest tests/test_gpu_tpg.py tests/test_gpu_xc.py tests/test_gpu_parity.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" | tee -a $O/ab.txt; tail -n 2 $O/pytest.log
