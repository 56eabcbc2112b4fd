"""One merge of a cfg2-row column over a small dictionary (X_M in shared memory), for ncu."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen
import paper_1109_6885_b200 as dm
from tests.parity import to_device
dict_len = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
n_delta = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
col = datagen.make_random_case(5150 + dict_len, 100_000_000, dict_len, n_delta, 0.05)
UM, M, D = to_device(col)
m = dm.ColumnMerger(UM, M, col.n_main, col.main_bits, D)
for _ in range(2):
    m.run_async()
torch.cuda.synchronize()
print("ok", m.result().merged_bits)
