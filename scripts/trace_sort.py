"""Phase timestamps of k_onesweep (trace build, -DDM_TRACE) for several delta sizes.
Phases: 1 start, 2 tile claimed, 3 keys loaded, 4 ranked, 5 counts published +
block scan, 6 reordered in smem, 7 look-back done, 8 scattered."""
import ctypes
import os
import sys

os.environ["DM_LIB_PATH"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                         "paper_1109_6885_b200", "libdictmerge_trace.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.sort_scaling import run  # noqa: E402
import paper_1109_6885_b200 as dm  # noqa: E402

for nd in [int(x) for x in (sys.argv[1:] or ["16384", str(1 << 20), str(1 << 24)])]:
    run(1 << 20, 1 << 16, nd, 0.5, 64, reps=1)
    buf = (ctypes.c_ulonglong * 256)()
    dm._lib().dm_debug_trace(buf)
    t0 = min(buf[b * 32 + 1] for b in range(8) if buf[b * 32 + 1])
    for b in range(8):
        t = [buf[b * 32 + i] for i in range(9)]
        if not t[1]:
            continue
        print(nd, "sample", b, "start +%.1f us" % ((t[1] - t0) / 1e3),
              "phases (us):", ["%.1f" % ((t[i + 1] - t[i]) / 1e3) for i in range(1, 8)],
              "cta %.1f us" % ((t[8] - t[1]) / 1e3))
