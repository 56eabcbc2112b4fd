# A/B of the Step 2(b) thread-per-group forms (round 2, session d)
O=gpurun_out/r02f; mkdir -p $O
L=$PWD/paper_1109_6885_b200
{ for v in default tpgd8 tpgd12 tpgd12np tpgd16np default; do
    echo "== $v"
    if [ $v = default ]; then bash scripts/quick_bench.sh cfg2 cfg3; else DM_LIB_PATH=$L/libdictmerge_$v.so bash scripts/quick_bench.sh cfg2 cfg3; fi
  done; } 2>&1 | tee $O/ab.txt
for v in tpgd12np tpgd16np tpgd12; do
  DM_LIB_PATH=$L/libdictmerge_$v.so timeout 600 python -m pytest tests/test_gpu_tpg.py -m gpu -x -q > $O/pytest_tpg_$v.log 2>&1; echo "$v rc=$?" | tee -a $O/ab.txt
done
