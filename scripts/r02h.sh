# Step 2(b) direct form: 16-byte vs 32-byte global accesses, 8 / 12 / 16 warps (round 2, session d)
O=gpurun_out/r02h; mkdir -p $O
L=$PWD/paper_1109_6885_b200
{ for v in default v8 v8d12 v8d16 v8 default; do
    echo "== $v"
    if [ $v = default ]; then bash scripts/quick_bench.sh cfg2; else DM_LIB_PATH=$L/libdictmerge_$v.so bash scripts/quick_bench.sh cfg2; fi
  done; } 2>&1 | tee $O/ab.txt
DM_LIB_PATH=$L/libdictmerge_v8.so timeout 1200 python -m pytest tests/test_gpu_tpg.py tests/test_gpu_xc.py tests/test_gpu_parity.py -m gpu -x -q > $O/pytest_v8.log 2>&1; echo "pytest v8 rc=$?" | tee -a $O/ab.txt
