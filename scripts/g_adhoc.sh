set -u
O=gpurun_out/$1; mkdir -p $O; shift
timeout 600 python -m pytest tests/test_gpu_xc.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
for v in "" "$@"; do
  if [ -n "$v" ]; then export DM_LIB_PATH=$PWD/paper_1109_6885_b200/libdictmerge_$v.so; else unset DM_LIB_PATH; fi
  echo "== ${v:-default}"; bash scripts/quick_bench.sh cfg2
done
unset DM_LIB_PATH
timeout 300 python scripts/one_cfg.py 2 0 2 > $O/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_recompress -c 1 -o $O/rec -f python scripts/one_cfg.py 2 0 2 > $O/ncu.log 2>&1
python scripts/ncu_summary.py $O/rec.ncu-rep > $O/ncu_rec.txt 2>&1; ncu -i $O/rec.ncu-rep --page source --csv > $O/src.csv 2>/dev/null; rm -f $O/rec.ncu-rep
