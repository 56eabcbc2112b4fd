"""Phase timestamps of k_onesweep (trace build) for a small and a cfg2-sized delta."""
import ctypes, os, sys
os.environ["DM_LIB_PATH"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                         "paper_1109_6885_b200", "libdictmerge_trace.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.sort_scaling import run
import paper_1109_6885_b200 as dm
for nd in (16384, 1 << 20):
    run(1 << 20, 1 << 16, nd, 0.5, 48, reps=1)
    buf = (ctypes.c_ulonglong * 256)()
    dm._lib().dm_debug_trace(buf)
    for b in range(4):
        t = [buf[b * 32 + i] for i in range(9)]
        if t[0] == 0: continue
        print(nd, "block", b, "phase deltas (ns):", [t[i + 1] - t[i] if t[i + 1] and t[i] else None for i in range(8)],
              "total", t[8] - t[0] if t[8] else None)
