set -u
O=gpurun_out/$1; mkdir -p $O; shift
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "table" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log; tail -2 $O/pytest.log
timeout 300 python scripts/one_table.py 1 > $O/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_recompress_batch" --csv --log-file $O/launches.csv python scripts/one_table.py 1 > $O/ncu.log 2>&1
python scripts/launches.py $O/launches.csv > $O/launches.txt 2>&1; cat $O/launches.txt
bash scripts/quick_bench.sh cfg4 | tee $O/quick.txt
