#!/usr/bin/env python
"""bench.py -- merged tuples/s of the online dictionary merge on B200 (arXiv 1109.6885).

One "step" = one whole merge of one column (Steps 1(a), 1(b), 2(a), 2(b)) on the
BASELINE.json workload configs[1] ("cfg2": N_M = 1e8 rows at 24 bits over a
1e7-entry u64 dictionary, N_D = 1e6 delta tuples, 10% new), synthetic seeded
inputs (datagen), resident in HBM when the timed region starts.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU): each rank merges its own column (whole
columns are independent units) -- no collective on the data path,
weak scaling; the step time is the max over ranks.

Prints ONE JSON line (rank 0).  Keys: see DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402

CFG = 2
WORKLOAD = "cfg2: single u64 column, N_M=1e8 @24b over |U_M|=1e7 (uniform in [0,2^48), uniform codes), N_D=1e6 (90% reuse / 10% new)"
METRIC = "merged tuples/sec per column (N_M+N_D)"
UNIT = "tuples/s"


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


def algorithmic_bytes(col, merged_len, merged_bits, delta_dict_len):
    """Per-kernel and whole-merge minimum bytes."""
    E = col.key_bytes
    nM, nD, nU = col.n_main, col.n_delta, col.dict_len
    npr = nM + nD
    step2 = nM * col.main_bits / 8 + npr * merged_bits / 8 + 4 * nU + 4 * nD + 4 * delta_dict_len
    strict = nM * col.main_bits / 8 + nD * E + nU * E + merged_len * E + npr * merged_bits / 8
    return step2, strict


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.idx = gpu_index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def host_info():
    cpu = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return cpu, os.cpu_count()


def run_oracle_steps(col, steps):
    """The oracle as it stands (linear mode, 1 thread) on the full column."""
    import oracle
    oracle.build()
    W = oracle.pack(col.main_codes, col.main_bits)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        r = oracle.merge(col, "linear", main_words=W)
        times.append(time.perf_counter() - t0)
        assert r.status == 0
    return times


def reference_arm(args, rank, world):
    if rank != 0:
        return 0
    col = datagen.make_config(CFG)
    n = col.n_main + col.n_delta
    run_oracle_steps(col, args.warmup)
    times = run_oracle_steps(col, args.steps)
    t = sum(times) / len(times)
    cpu, ncpu = host_info()
    v = n / t
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (datagen, seeded)",
        "config": {"workload": WORKLOAD, "seed": datagen.config_seed(CFG)},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"full cfg2 column per step ({n} tuples), oracle linear mode, 1 thread, {cpu}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import torch
    import paper_1109_6885_b200 as dm

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist

    # ---- inputs (per rank: its own column; rank 0 = the seeded cfg2 column)
    col = datagen.make_config(CFG, seed=datagen.BASE_SEED + 7 * rank)
    UM = torch.from_numpy(col.main_dict.view(np.int64)).to(dev)
    D = torch.from_numpy(col.delta.view(np.int64)).to(dev)
    codes = torch.from_numpy(col.main_codes.view(np.int32)).to(dev)
    M = dm.pack_codes(codes, col.main_bits)
    del codes
    merger = dm.ColumnMerger(UM, M, col.n_main, col.main_bits, D)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 2x the 126 MB L2
    stream = torch.cuda.current_stream()

    for _ in range(max(args.warmup, 0)):
        merger.run_async()
    torch.cuda.synchronize()
    r0 = merger.result()

    # ---- per-step breakdown (eager launches, events at the step boundaries)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    for row in ev:  # torch creates the CUDA event lazily on first record
        for e in row:
            e.record()
    torch.cuda.synchronize()
    launches0 = dm.launch_count()
    for k in range(args.steps):
        flush.zero_()
        merger.run_async_timed(ev[k])
    torch.cuda.synchronize()
    launches_per_merge = (dm.launch_count() - launches0) / max(args.steps, 1)
    s1a = [ev[k][0].elapsed_time(ev[k][1]) for k in range(args.steps)]
    s1b = [ev[k][1].elapsed_time(ev[k][2]) for k in range(args.steps)]
    s2 = [ev[k][2].elapsed_time(ev[k][3]) for k in range(args.steps)]
    eager_ms = [ev[k][0].elapsed_time(ev[k][3]) for k in range(args.steps)]

    # ---- timed region: K whole merges replayed from a CUDA graph (one driver call
    # each), L2 flushed before each, CUDA events around each merge on its stream
    merger.capture_graph()
    gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in gev:
        a.record()
        b.record()
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()
            gev[k][0].record()
            merger.replay_graph()
            gev[k][1].record()
        torch.cuda.synchronize()
    launches = int(round(launches_per_merge * args.steps))
    if pg:
        pg.barrier()
    step_ms = [a.elapsed_time(b) for a, b in gev]
    total_ms = sum(step_ms)
    if pg:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    n_tuples = col.n_main + col.n_delta
    value = world * n_tuples / (ms_per_step / 1e3)

    res = merger.result()
    step2_bytes, strict_bytes = algorithmic_bytes(col, res.merged_len, res.merged_bits, res.delta_dict_len)
    pk = peaks()
    peak_hbm = pk["hbm_gbs"] if pk else 6650.0
    s2_ms = statistics.mean(s2)
    achieved = step2_bytes / (s2_ms / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "recompress_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("traffic_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- e2e through the public host-buffer API (H2D inputs + D2H results inside)
    e2e = None
    if not args.no_e2e:
        ctx = dm.HostContext(local)
        hUM = torch.from_numpy(col.main_dict.view(np.int64)).pin_memory()
        hD = torch.from_numpy(col.delta.view(np.int64)).pin_memory()
        hM = M.cpu().pin_memory()
        hU = torch.empty(col.dict_len + col.n_delta, dtype=torch.int64).pin_memory()
        hMo = torch.empty(dm.words(n_tuples, 32), dtype=torch.int64).pin_memory()
        ctx.merge(hUM, hM, col.n_main, col.main_bits, hD, hU, hMo)  # warm-up (allocations)
        if pg:
            pg.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            nU, nb, _ = ctx.merge(hUM, hM, col.n_main, col.main_bits, hD, hU, hMo)
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        if pg:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            e2e_s = float(t.item())
        h2d = hUM.numel() * 8 + hD.numel() * 8 + hM.numel() * 8
        d2h = nU * 8 + dm.words(n_tuples, nb) * 8
        e2e = {"value": world * n_tuples / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s * 1e3}
        ctx.close()

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        times = run_oracle_steps(col, 2)
        cpu, ncpu = host_info()
        t = min(times)
        cpu_baseline = {"value": n_tuples / t, "unit": UNIT, "cores": 1, "kind": "oracle",
                        "sample": f"the full cfg2 column (N'={n_tuples}), oracle linear mode, best of 2, "
                                  f"1 thread of {ncpu} ({cpu})"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic (datagen, seeded; BASELINE configs[1])",
            "config": {"workload": WORKLOAD, "seed": datagen.config_seed(CFG), "n_main": col.n_main,
                       "n_delta": col.n_delta, "dict_len": col.dict_len, "main_bits": col.main_bits,
                       "merged_len": res.merged_len, "merged_bits": res.merged_bits,
                       "parallelism": f"column-sharded x{world} (independent columns, no collective)",
                       "l2": "flushed (512 MB write) before every timed step"},
            "steps_ms": {"s1a_delta_dict": statistics.mean(s1a), "s1b_dict_merge": statistics.mean(s1b),
                         "s2b_recompress": s2_ms, "eager_total": statistics.mean(eager_ms),
                         "graph_total": statistics.mean(step_ms),
                         "note": "s1a/s1b/s2b from eager launches with events between steps; "
                                 "value/ms_per_step from CUDA-graph replays"},
            "hbm_fraction_strict": strict_bytes / (statistics.mean(step_ms) / 1e3) / 1e9 / peak_hbm,
            "roofline": {"kernel": "k_recompress (Step 2(b))", "bound": "hbm", "achieved": achieved,
                         "peak": peak_hbm, "unit": "GB/s", "frac": achieved / peak_hbm, "traffic": traffic,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if pk else "fallback 6.65 TB/s",
                         "algorithmic_bytes_per_launch": step2_bytes},
            "cpu_baseline": cpu_baseline,
            "e2e": e2e,
            "gpu_launches": launches,
            "gpu_launches_per_step": launches / max(args.steps, 1),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
