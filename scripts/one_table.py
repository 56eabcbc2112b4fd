"""The cfg4 300-column table merged through TableMerger (as bench.py does), for
ncu launch lists: python scripts/one_table.py [reps]."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1109_6885_b200 as dm  # noqa: E402
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
dev = torch.device("cuda", 0)
cols = bench.host_columns("cfg4", 0, 1)
tm = dm.TableMerger([bench.device_inputs(c, dev) for c in cols])
for _ in range(reps):
    tm.run_async()
torch.cuda.synchronize()
print("ok", sum(r.merged_bits for r in tm.results()))
