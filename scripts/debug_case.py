"""Run one random case through the library (DM_SYNC_DEBUG=1 names the faulting step)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, oracle
import paper_1109_6885_b200 as dm
from tests.parity import run_gpu, compare
n_main, dict_len, n_delta, p_new = [float(x) for x in sys.argv[1:5]]
key = sys.argv[5] if len(sys.argv) > 5 else "u64"
variant = int(sys.argv[6]) if len(sys.argv) > 6 else 0
dm.set_tuning(1, variant)
col = datagen.make_random_case(911 + int(n_delta), int(n_main), int(dict_len), int(n_delta), p_new, key=key)
M, r = run_gpu(col)
oracle.build()
compare(col, M, r)
print("ok")
