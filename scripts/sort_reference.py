"""Calibration only (not the product path): time CUB radix sort (torch.sort,
stable, int64 keys + int64 indices) and torch.unique on Step 1(a)'s key counts,
for comparison with the library's Step 1(a) (bench steps_ms.s1a_delta_dict)."""
import json, sys
import torch

def t_ms(f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

for n, bits in ((10_000, 40), (1_000_000, 48), (5_000_000, 64), (50_000_000, 64)):
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randint(0, 2 ** min(bits, 62), (n,), device="cuda", generator=g)
    r = {"n": n, "bits": bits,
         "torch_sort_stable_ms": t_ms(lambda: torch.sort(x, stable=True)),
         "torch_unique_inverse_ms": t_ms(lambda: torch.unique(x, sorted=True, return_inverse=True))}
    print(json.dumps(r))
