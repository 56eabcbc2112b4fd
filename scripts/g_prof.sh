set -u
O=gpurun_out/$1; K=$2; CFG=${3:-2}; mkdir -p $O
timeout 300 python scripts/one_cfg.py $CFG 0 2 > $O/plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-0} -c ${CNT:-6} -o $O/p -f python scripts/one_cfg.py $CFG 0 2 > $O/ncu.log 2>&1
python scripts/ncu_summary.py $O/p.ncu-rep > $O/ncu.txt 2>&1; ncu -i $O/p.ncu-rep --page source --csv > $O/src.csv 2>/dev/null; rm -f $O/p.ncu-rep
