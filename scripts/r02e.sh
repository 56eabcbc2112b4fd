O=gpurun_out/r02e; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_merge_variants.py tests/test_gpu_cfg5.py -m gpu -x -q > $O/pytest_a.log 2>&1; echo "rc=$?" >> $O/pytest_a.log; tail -3 $O/pytest_a.log
{ echo default; bash scripts/quick_bench.sh cfg2 cfg5 cfg2;
  echo grid1; DM_SP_GRID=1 bash scripts/quick_bench.sh cfg2 cfg5 cfg2;
  echo sp4k; DM_LIB_PATH=$PWD/paper_1109_6885_b200/libdictmerge_sp4k.so bash scripts/quick_bench.sh cfg2 cfg5 cfg2;
  echo uq256; DM_LIB_PATH=$PWD/paper_1109_6885_b200/libdictmerge_uq256.so bash scripts/quick_bench.sh cfg2 cfg2; } 2>&1 | tee $O/ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_b.log 2>&1; echo "rc=$?" >> $O/pytest_b.log; tail -3 $O/pytest_b.log
