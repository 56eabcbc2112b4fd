"""One or more merges of a BASELINE config (for ncu): python scripts/one_cfg.py <cfg> [knob] [reps]."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen
import paper_1109_6885_b200 as dm
from tests.parity import to_device
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
knob = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
dm.set_tuning(0, knob)
col = datagen.make_config(cfg, column=0) if cfg == 4 else datagen.make_config(cfg)
UM, M, D = to_device(col)
m = dm.ColumnMerger(UM, M, col.n_main, col.main_bits, D)
for _ in range(reps):
    m.run_async()
torch.cuda.synchronize()
print("ok", m.result().merged_bits)
