"""One merge of a given workload shape (for ncu): cfg5 at a scale, or cfg2."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1109_6885_b200 as dm
from datagen import torch_gen
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1 / 16
UM, codes, bits, D = torch_gen.make_cfg5(scale=scale, device="cuda")
M = dm.pack_codes(codes, bits)
m = dm.ColumnMerger(UM, M, UM.numel(), bits, D)
for _ in range(2):
    m.run_async()
torch.cuda.synchronize()
print("ok", m.result().merged_bits)
