"""Diagnostic (not a bench line): k_recompress when the translation table is in
shared memory, i.e. when Step 2(b) is a pure HBM stream (unpack -> translate ->
repack).  Rows as cfg2 (N_M = 1e8, N_D = 1e6) over small dictionaries, so X_M
(<= 96 KB) is staged in shared memory and no random gather leaves the SM.
Reports Step 2(b) algorithmic bytes / event time against MEASURED_PEAKS.json.

    python scripts/stream_bound.py            # on the GPU box
"""
import json, os, statistics, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402
import paper_1109_6885_b200 as dm  # noqa: E402
from bench import step2_bytes, peaks  # noqa: E402
from tests.parity import to_device  # noqa: E402

pk = peaks()
peak = pk["hbm_gbs"] if pk else 6650.0
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
# N_D small enough that b' has at most 4 candidates (width-specialised kernels)
for dict_len, n_main, n_delta in ((1000, 100_000_000, 5_000), (20_000, 100_000_000, 100_000),
                                 (20_000, 200_000_000, 100_000), (1000, 100_000_000, 1_000_000)):
    col = datagen.make_random_case(5150 + dict_len, n_main, dict_len, n_delta, 0.05)
    UM, M, D = to_device(col)
    del col
    m = dm.ColumnMerger(UM, M, n_main, datagen.width_hint(dict_len), D)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for e in ev:  # torch creates the CUDA event lazily on first record
        e.record()
    s2 = []
    for it in range(8):
        flush.zero_()
        m.run_async_timed(ev)
        torch.cuda.synchronize()
        if it >= 3:
            s2.append(ev[2].elapsed_time(ev[3]))
    r = m.result()
    b = step2_bytes(n_main, datagen.width_hint(dict_len), n_delta, dict_len, r.merged_bits, r.delta_dict_len)
    ms = statistics.median(s2)
    gbs = b / (ms / 1e3) / 1e9
    print(json.dumps({"dict_len": dict_len, "n_main": n_main, "n_delta": n_delta, "main_bits": datagen.width_hint(dict_len),
                      "merged_bits": r.merged_bits, "s2b_ms": ms, "algorithmic_bytes": b, "achieved_gbs": gbs,
                      "peak_gbs": peak, "frac": gbs / peak}))
    del m, UM, M, D
    torch.cuda.empty_cache()
