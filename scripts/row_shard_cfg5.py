"""cfg5 row-sharded Step 2 on one GPU: bytes each rank would receive
with the XC broadcast vs the literal X_M, and the device time of one rank's
shard (1/G of the rows) through dm_recompress_xc and dm_recompress."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1109_6885_b200 as dm
from paper_1109_6885_b200 import sharding
from datagen import torch_gen

UM, codes, bits, D = torch_gen.make_cfg5(device="cuda")
M = dm.pack_codes(codes, bits)
del codes
n_main = UM.numel()
dmg = dm.DictionaryMerger(UM, n_main, bits, D)
dmg.run_async()
h = dmg.header()
xc = dmg.xc()
ids, sl, cnt = dm.xc_exceptions_gather(xc, n_main, dmg.XM)
res = {"n_main": n_main, "n_delta": D.numel(), "merged_bits": int(h.merged_bits),
       "bytes_xc_records": xc.records.numel(), "bytes_xc_offsets": xc.offsets.numel(),
       "exceptions": cnt, "bytes_exceptions": cnt * (4 << xc.shift) * 4 + cnt * 4,
       "bytes_x_main_plain": n_main * 4, "bytes_x_delta": int(h.delta_dict_len) * 4, "bytes_rank": D.numel() * 4}
for G in (2, 8):
    s = sharding.plan_row_shards(n_main, D.numel(), G)[0]
    mslice = M[s.in_word(bits):]
    t = {}
    for name, fn in (("xc", lambda: dm.recompress_xc(mslice, s.n_main, bits, n_main, xc, dmg.XM, dmg.XD,
                                                      dmg.R[s.delta_begin:], s.n_delta, h.merged_bits)),
                     ("plain", lambda: dm.recompress(mslice, s.n_main, bits, n_main, dmg.XM, dmg.XD,
                                                     dmg.R[s.delta_begin:], s.n_delta, h.merged_bits))):
        fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
        ms = []
        for _ in range(3):
            flush.zero_()
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        t[name] = min(ms)
    res[f"shard_1_of_{G}_ms"] = t
print(json.dumps(res))
