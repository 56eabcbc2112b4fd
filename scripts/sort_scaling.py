"""Step-time scaling experiment (GPU box): Step 1(a)/1(b)/2(b) times vs N_D and active passes."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_1109_6885_b200 as dm  # noqa: E402


def run(n_main, dict_len, n_delta, p_new, value_bits, reps=5):
    col = datagen.make_random_case(7, n_main, dict_len, n_delta, p_new, value_bits=value_bits)
    UM = torch.from_numpy(col.main_dict.view(np.int64).copy()).cuda()
    D = torch.from_numpy(col.delta.view(np.int64).copy()).cuda()
    M = dm.pack_codes(torch.from_numpy(col.main_codes.view(np.int32).copy()).cuda(), col.main_bits)
    m = dm.ColumnMerger(UM, M, col.n_main, col.main_bits, D)
    for _ in range(3):
        m.run_async()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(reps)]
    for r in ev:
        for e in r:
            e.record()
    torch.cuda.synchronize()
    for k in range(reps):
        m.run_async_timed(ev[k])
    torch.cuda.synchronize()
    t = [[ev[k][i].elapsed_time(ev[k][i + 1]) * 1e3 for i in range(3)] for k in range(reps)]
    med = [sorted(x[i] for x in t)[reps // 2] for i in range(3)]
    return {"n_main": n_main, "dict_len": dict_len, "n_delta": n_delta, "value_bits": value_bits,
            "s1a_us": med[0], "s1b_us": med[1], "s2b_us": med[2]}


if __name__ == "__main__":
    for nd, vb in [(1 << 14, 8), (1 << 14, 48), (1 << 17, 48), (1 << 20, 8), (1 << 20, 16), (1 << 20, 48),
                   (1 << 22, 48), (1 << 24, 64)]:
        print(json.dumps(run(1 << 20, min(1 << 16, (1 << vb) // 4), nd, 0.5, vb)), flush=True)
    for dl in [1 << 20, 1 << 22, 1 << 24]:
        print(json.dumps(run(1 << 22, dl, 1 << 16, 0.1, 48)), flush=True)
