"""Write profiles/recompress_traffic.json: DRAM bytes (read + write) per launch of
the dominant kernel (k_recompress) per workload, from `ncu --set full` reports
(run on the GPU box after each workload ran once without ncu).

    python scripts/traffic.py capture cfg1 cfg2 cfg3 cfg5   # on the GPU box
    python scripts/traffic.py summarize                    # here: reports -> json + txt
"""
import csv, io, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")


def cmd(w):
    if w == "cfg5":
        return ["python", "scripts/one_merge.py", "1.0"]
    return ["python", "scripts/one_cfg.py", w[3:], "0", "2"]


def capture(ws):
    for w in ws:
        subprocess.run(cmd(w), check=True, cwd=ROOT)  # plain run first: must exit 0
        rep = os.path.join(OUT, f"traffic_{w}")
        # the second merge's k_recompress launches (first merge warms the caches)
        subprocess.run(["timeout", "900", "ncu", "--set", "full", "--clock-control", "none", "--import-source", "on",
                        "-k", "regex:k_recompress", "-o", rep, "-f"] + cmd(w), cwd=ROOT,
                       stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)


def summarize():
    res = {}
    for f in sorted(os.listdir(OUT)):
        if not (f.startswith("traffic_") and f.endswith(".ncu-rep")):
            continue
        w = f[len("traffic_"):-len(".ncu-rep")]
        raw = subprocess.run(["ncu", "-i", os.path.join(OUT, f), "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        h = rows[0]
        best = None
        for v in rows[2:]:
            d = dict(zip(h, v))
            num = lambda k: float(d[k].replace(",", ""))
            unit = dict(zip(h, rows[1]))
            scale = lambda k: {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit[k], 1)
            t = num("gpu__time_duration.sum") * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
                                                 "msecond": 1e-3, "ms": 1e-3}.get(unit["gpu__time_duration.sum"], 1e-9)
            b = num("dram__bytes_read.sum") * scale("dram__bytes_read.sum") + \
                num("dram__bytes_write.sum") * scale("dram__bytes_write.sum")
            if best is None or t > best[0]:
                inst = num("smsp__inst_executed.sum") if "smsp__inst_executed.sum" in d else None
                issue = num("smsp__issue_active.avg.pct_of_peak_sustained_active") \
                    if "smsp__issue_active.avg.pct_of_peak_sustained_active" in d else None
                best = (t, b, d["Kernel Name"][:60], inst, issue)
        if best:
            res[w] = {"traffic_bytes_per_launch": best[1], "kernel_time_s_under_ncu": best[0], "kernel": best[2],
                      "warp_instructions_per_launch": best[3], "issue_active_pct": best[4],
                      "source": f"ncu --set full (gpurun_out/{f}), longest k_recompress launch of one merge"}
    path = os.path.join(ROOT, "profiles", "recompress_traffic.json")
    json.dump(res, open(path, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    capture(sys.argv[2:]) if sys.argv[1] == "capture" else summarize()
