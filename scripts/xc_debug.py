"""Debug: run one merge per placement knob and report where M' differs from the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen, oracle
import paper_1109_6885_b200 as dm
from tests.parity import run_gpu
oracle.build()
col = datagen.make_random_case(7919 + 70001, 70001, 70000, 50001, 1.0, key="u64")
ref = oracle.merge(col, "linear")
want = ref.merged_words
n = col.n_main + col.n_delta
for k in (1, 0, 2, 3):
    dm.set_tuning(0, k)
    M, r = run_gpu(col)
    got = r.merged_codes.cpu().numpy().view(np.uint64)
    gc = dm.unpack_codes(r.merged_codes, n, r.merged_bits).cpu().numpy().view(np.uint32)
    wc = dm.unpack_codes(torch.from_numpy(want.view(np.int64)).cuda(), n, r.merged_bits).cpu().numpy().view(np.uint32)
    bad = np.nonzero(gc != wc)[0]
    print("knob", k, "bits", r.merged_bits, ref.merged_bits, "bad rows", bad.size, "of", n, bad[:5],
          "got", gc[bad[:5]], "want", wc[bad[:5]], "codes", col.main_codes[bad[:5][bad[:5] < col.n_main]] if bad.size else "")
