"""NEXT2 on one GPU, cfg5: the root's Step 1(a) alone, and one rank's share of the
sharded Step 1(b) (a 1/G range of U_M with its U_D range, dm_dictionary_merge_sorted_async)
against the whole unsharded Step 1(b).  CUDA events around the async entry points."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1109_6885_b200 as dm
from paper_1109_6885_b200 import sharding
from datagen import torch_gen


def t_ms(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    best = 1e9
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


UM, codes, bits, D = torch_gen.make_cfg5(device="cuda")
del codes
dm.set_tuning(dm.KNOB_XC_SHIFT, 7)
res = {}
full = dm.DictionaryMerger(UM, 0, bits, D, mode="dict")
res["s1a_plus_s1b_ms"] = t_ms(full.run_async)
dd = dm.DictionaryMerger(UM, 0, bits, D, mode="delta")
res["s1a_root_ms"] = t_ms(dd.run_async)
n_ud = int(dd.header().delta_dict_len)
UD = dd.UD[:n_ud]
for G in (2, 4, 8):
    ranges = sharding.plan_dict_ranges(UM.numel(), G)
    firsts = torch.stack([UM[a] for a, _ in ranges[1:]])
    cuts = [0] + dm.lower_bound(UD, firsts).tolist() + [n_ud]
    a, b = ranges[0]
    mine = UD[cuts[0]:cuts[1]].clone()
    lm = dm.DictionaryMerger(UM[a:b].clone(), 0, bits, mine, mode="sorted")
    res[f"s1b_range_1_of_{G}_ms"] = t_ms(lm.run_async)
    del lm, mine
print(json.dumps(res))
