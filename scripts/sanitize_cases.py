"""Small merges for compute-sanitizer (memcheck / racecheck / synccheck): both key
types, tails, seams, empty delta, all-new delta, table merge, dm_recompress."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen
import paper_1109_6885_b200 as dm
from tests.parity import to_device

cases = [(20011, 3000, 4099, 0.3, "u64"), (9001, 500, 2500, 1.0, "b16"), (5000, 3000, 0, 0.0, "u64"),
         (0, 1, 3000, 0.5, "u64"), (70001, 65537, 9000, 0.1, "u64")]
for n_main, dl, nd, p, key in cases:
    col = datagen.make_random_case(n_main + nd, n_main, dl, nd, p, key=key)
    UM, M, D = to_device(col)
    r = dm.merge_column(UM, M, col.n_main, col.main_bits, D, x_tables=True, delta_dict=True)
cols = [datagen.make_config(4, scale=1e-4, column=j) for j in (0, 250)]
dm.merge_table([(UM, M, c.n_main, c.main_bits, D) for c, (UM, M, D) in zip(cols, [to_device(c) for c in cols])])
torch.cuda.synchronize()
print("sanitize cases ok")
