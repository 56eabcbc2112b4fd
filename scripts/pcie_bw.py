"""Pinned host <-> device copy bandwidth on this box (context for the e2e number)."""
import json, torch
n = 512 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [fn() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3
h2d = n / t(lambda: d1.copy_(h1, non_blocking=True)) / 1e9
d2h = n / t(lambda: h2.copy_(d2, non_blocking=True)) / 1e9
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
bi = 2 * n / t(both) / 1e9
print(json.dumps({"h2d_gbs": h2d, "d2h_gbs": d2h, "bidirectional_total_gbs": bi, "bytes": n}))
