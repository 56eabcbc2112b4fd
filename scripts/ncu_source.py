"""Per-instruction hot spots of an ncu report (source page, SASS)."""
import csv, io, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]; idx = {k: i for i, k in enumerate(h)}; data = rows[2:]
def f(r, k):
    try: return float(r[idx[k]].replace(',', ''))
    except Exception: return 0.0
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
tot = sum(f(r, 'Warp Stall Sampling (All Samples)') for r in data)
print("samples", tot, "shared wavefronts", sum(f(r, 'L1 Wavefronts Shared') for r in data),
      "excessive", sum(f(r, 'L1 Wavefronts Shared Excessive') for r in data))
for r in sorted(data, key=lambda r: -f(r, 'Warp Stall Sampling (All Samples)'))[:n]:
    print(f"{int(f(r,'Warp Stall Sampling (All Samples)')):6d} {int(f(r,'Instructions Executed')):10d} {r[idx['Address']][-5:]} {r[idx['Source']][:80]}")
