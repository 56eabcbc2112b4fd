#!/usr/bin/env python
"""bench.py -- merged tuples/s of the online dictionary merge on B200 (arXiv 1109.6885).

One "step" = one whole merge (Steps 1(a), 1(b), 2(a), 2(b)) of the workload's
column(s), synthetic seeded inputs (datagen) resident in HBM when the timed
region starts, L2 flushed (512 MB write) before every timed step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2|cfg1|cfg3|cfg4|cfg5]

Default workload: BASELINE.json configs[1] ("cfg2": N_M = 1e8 rows at 24 bits over
a 1e7-entry u64 dictionary, N_D = 1e6, 10% new) -- the config the metric is quoted
on.  N > 1 (torchrun, one rank per GPU), strong scaling (the workload is the same
at every N): a single column (cfg1/2/2e4/3/5) is split by output rows through the
library's dm_merge_column_sharded (root Steps 1(a)-2(a), XC broadcast over NCCL,
Step 2(b) per row range: the paper's tuple split of Step 2); the 300-column
table (cfg4) is split by whole columns, LPT, no collective.  Step
time = max over ranks.  Prints ONE JSON line (rank 0).  Keys: DESIGN.md
"Measurement".
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

WORKLOADS = {
    "cfg1": "cfg1: single u64 column, N_M=1e6 @14b over |U_M|=1e4 in [0,2^40), N_D=1e4 (50% new)",
    "cfg2": "cfg2: single u64 column, N_M=1e8 @24b over |U_M|=1e7 (uniform in [0,2^48), uniform codes), "
            "N_D=1e6 (90% reuse / 10% new)",
    "cfg3": "cfg3: single 16-byte string column, N_M=1e8 @20b over |U_M|=1e6 (Zipf(1) codes), N_D=5e6 (20% new)",
    "cfg4": "cfg4: 300-column table, N_M=1e7 + N_D=1e5 per column, card log-uniform [2,1e7], 240 u64 + 60 strings",
    "cfg5": "cfg5: single u64 column, N_M=|U_M|=2^30 @30b (all unique), N_D=5e7 all new -> 31 bits (reading A12)",
    "cfg2e4": "cfg2 shape with 4-byte values (E=4, SURVEY NEXT4): N_M=1e8 @24b over |U_M|=1e7 in [0,2^32), "
              "N_D=1e6 (10% new)",
}
METRIC = "merged tuples/sec per column (N_M+N_D)"
UNIT = "tuples/s"


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


def strict_bytes(n_main, main_bits, n_delta, key_bytes, dict_len, merged_len, merged_bits):
    """SURVEY §8d minimum: each input read once, each output written once."""
    return (n_main * main_bits / 8 + n_delta * key_bytes + dict_len * key_bytes + merged_len * key_bytes
            + (n_main + n_delta) * merged_bits / 8)


def step2_bytes(n_main, main_bits, n_delta, dict_len, merged_bits, delta_dict_len):
    """Step 2(b) algorithmic bytes per launch."""
    return (n_main * main_bits / 8 + (n_main + n_delta) * merged_bits / 8 + 4 * dict_len + 4 * n_delta
            + 4 * delta_dict_len)


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


# ------------------------------------------------------------------------ inputs
def cfg_number(workload: str) -> int:
    return int(workload[3])  # "cfg2e4" -> 2 (the E = 4 variant of cfg2)


def key_dtype(workload: str) -> str:
    """The arithmetic type the path computes in: key compares and u32 codes."""
    return "u32" if workload.endswith("e4") else "u8x16" if cfg_number(workload) == 3 else "u64"


def host_columns(workload: str, rank: int, world: int):
    """The datagen columns this rank merges (host arrays)."""
    cfg = cfg_number(workload)
    if cfg == 4:
        from paper_1109_6885_b200.sharding import column_cost, lpt_partition
        costs = []
        for j in range(300):
            _, card, key, _ = datagen.cfg4_column_params(j)
            costs.append(column_cost(10**7, 10**5, card, datagen.width_hint(card), 8 if key == "u64" else 16))
        mine = lpt_partition(costs, world)[rank]
        return [datagen.make_config(4, column=j) for j in mine]
    if workload.endswith("e4"):
        return [datagen.make_config_e4(seed=datagen.BASE_SEED + 7 * rank)]
    return [datagen.make_config(cfg, seed=datagen.BASE_SEED + 7 * rank)]


def device_inputs(col, dev):
    import torch
    import paper_1109_6885_b200 as dm
    if col.key in ("u64", "u32"):
        it = np.int64 if col.key == "u64" else np.int32
        UM = torch.from_numpy(col.main_dict.view(it)).to(dev)
        D = torch.from_numpy(col.delta.view(it)).to(dev)
    else:
        UM = torch.from_numpy(np.ascontiguousarray(col.main_dict)).to(dev)
        D = torch.from_numpy(np.ascontiguousarray(col.delta)).to(dev)
    codes = torch.from_numpy(col.main_codes.view(np.int32)).to(dev)
    M = dm.pack_codes(codes, col.main_bits)
    return UM, M, col.n_main, col.main_bits, D


def cfg5_device_inputs(dev, rank):
    import paper_1109_6885_b200 as dm
    from datagen import torch_gen
    UM, codes, bits, D = torch_gen.make_cfg5(seed=datagen.BASE_SEED + 7 * rank, device=dev)
    M = dm.pack_codes(codes, bits)
    del codes
    return UM, M, UM.numel(), bits, D


# ----------------------------------------------------------------- oracle legs
def oracle_sample(workload: str):
    """A bounded sample of the workload for the CPU oracle (≈10-30 s of work)."""
    cfg = cfg_number(workload)
    if cfg == 4:
        return [datagen.make_config(4, column=j) for j in (0, 60, 120, 180, 239, 240, 270, 299)], \
            "8 of the 300 cfg4 columns at full size (0,60,120,180,239 u64; 240,270,299 strings)"
    if cfg == 5:
        return [datagen.make_config(5, scale=1 / 16)], "cfg5 at 1/16 scale (2^26 main rows, 3.1e6 delta)"
    col = datagen.make_config_e4() if workload.endswith("e4") else datagen.make_config(cfg)
    return [col], f"the full {workload} column (N'={col.n_main + col.n_delta})"


def run_oracle(cols, reps):
    import oracle
    oracle.build()
    packed = [oracle.pack(c.main_codes, c.main_bits) for c in cols]
    tuples = sum(c.n_main + c.n_delta for c in cols)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        for c, W in zip(cols, packed):
            r = oracle.merge(c, "linear", main_words=W)
            assert r.status == 0
        times.append(time.perf_counter() - t0)
    return tuples, times


_PAR_COLS = None


def _oracle_one(j):
    import oracle
    c = _PAR_COLS[j]
    r = oracle.merge(c, "linear", main_words=oracle.pack(c.main_codes, c.main_bits))
    assert r.status == 0
    return c.n_main + c.n_delta


def run_oracle_columns_parallel(cols, workers):
    """The paper's first parallelisation scheme (a task queue over columns)
    done plainly: the oracle merges whole columns on `workers` host processes."""
    import multiprocessing as mp
    import oracle
    global _PAR_COLS
    oracle.build()
    _PAR_COLS = cols
    with mp.get_context("fork").Pool(workers) as pool:
        t0 = time.perf_counter()
        tuples = sum(pool.map(_oracle_one, range(len(cols)), chunksize=1))
        t = time.perf_counter() - t0
    return tuples, t


def reference_arm(args, rank, world):
    if rank != 0:
        return 0
    cols, sample = oracle_sample(args.workload)
    tuples, _ = run_oracle(cols, max(args.warmup, 0)) if args.warmup else (None, None)
    tuples, times = run_oracle(cols, args.steps)
    t = sum(times) / len(times)
    cpu, ncpu = host_info()
    v = tuples / t
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": key_dtype(args.workload),
        "data": "synthetic (datagen, seeded)", "config": {"workload": WORKLOADS[args.workload]},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{sample}; oracle linear mode, 1 thread of {ncpu} ({cpu})"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def pcie_bidirectional_gbs(dev, n=256 << 20):
    """Concurrent H2D + D2H pinned copy rate (GB/s, both directions summed)."""
    import torch
    try:
        h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
        h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
        d1 = torch.empty(n, dtype=torch.uint8, device=dev)
        d2 = torch.empty(n, dtype=torch.uint8, device=dev)
        s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = None
        for _ in range(3):
            torch.cuda.synchronize()
            a.record()
            s1.wait_event(a)
            s2.wait_event(a)
            with torch.cuda.stream(s1):
                d1.copy_(h1, non_blocking=True)
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            b.record()
            torch.cuda.synchronize()
            t = a.elapsed_time(b) / 1e3
            best = t if best is None else min(best, t)
        return 2 * n / best / 1e9
    except Exception:
        return None


# ----------------------------------------------------------- N > 1: one column row-sharded
def sharded_inputs(workload: str, rank: int, world: int, dev):
    """(UM, D on the root else None, this rank's packed main-code shard, n_main,
    main_bits, dict_len, n_delta, key): the row plan is the library's
    (dm_plan_row_shards); the shard is packed from bit 0 (its first row is a
    multiple of 4096, so these are exactly the words of the full packing)."""
    import torch
    import paper_1109_6885_b200 as dm
    cfg = cfg_number(workload)
    UM = D = None
    if cfg == 5:
        from datagen import torch_gen
        UM, codes, bits, D = torch_gen.make_cfg5(seed=datagen.BASE_SEED, device=dev)
        n_main, dict_len, n_delta, key = codes.numel(), UM.shape[0], D.shape[0], "u64"
    else:
        col = datagen.make_config_e4() if workload.endswith("e4") else datagen.make_config(cfg)
        codes = torch.from_numpy(col.main_codes.view(np.int32))
        n_main, bits, dict_len, n_delta, key = col.n_main, col.main_bits, col.dict_len, col.n_delta, col.key
        if rank == 0:
            if col.key in ("u64", "u32"):
                it = np.int64 if col.key == "u64" else np.int32
                UM = torch.from_numpy(col.main_dict.view(it)).to(dev)
                D = torch.from_numpy(col.delta.view(it)).to(dev)
            else:
                UM = torch.from_numpy(np.ascontiguousarray(col.main_dict)).to(dev)
                D = torch.from_numpy(np.ascontiguousarray(col.delta)).to(dev)
        del col
    cuts = dm.plan_row_shards(n_main, n_delta, world)
    m0, m1 = min(cuts[rank], n_main), min(cuts[rank + 1], n_main)
    shard = dm.pack_codes(codes[m0:m1].to(dev), bits) if m1 > m0 else torch.zeros(2, dtype=torch.int64, device=dev)
    del codes
    if rank != 0:
        D = None
        if cfg != 5:
            UM = None
    return UM, D, shard, n_main, bits, dict_len, n_delta, key, cuts


def run_sharded(args, rank, world, local, dev, backend):
    """One column's merge split by output rows over the ranks (the
    paper's tuple split of Step 2) through dm_merge_column_sharded: strong
    scaling (the column is fixed, every rank does 1/N of Step 2 after the root's
    Step 1 and the table broadcasts)."""
    import torch
    import torch.distributed as dist
    import paper_1109_6885_b200 as dm
    UM, D, shard, n_main, bits, dict_len, n_delta, key, cuts = sharded_inputs(args.workload, rank, world, dev)
    # cfg5's 1.07e9-entry dictionary: Step 1(b) by U_M value ranges on every rank (NEXT2);
    # smaller dictionaries: the root merges them (fewer collectives)
    step1b = "ranges" if cfg_number(args.workload) == 5 else "root"
    range_begin = 0
    if step1b == "ranges":
        a, b = dm.plan_dict_ranges(dict_len, world)[rank:rank + 2]
        UM, range_begin = UM[a:b].clone(), a
        torch.cuda.empty_cache()
    comm = dm.Comm.nccl() if backend == "nccl" else dm.Comm.callbacks()
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def step():
        return dm.merge_column_sharded(comm, shard, n_main, bits, dict_len, n_delta, main_dict=UM, delta=D, key=key,
                                       step1b=step1b, range_begin=range_begin)

    for _ in range(max(args.warmup, 0)):
        r = step()
    torch.cuda.synchronize()
    launches0 = dm.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            ev[k][0].record()
            r = step()
            ev[k][1].record()
        torch.cuda.synchronize()
    dist.barrier()
    launches = dm.launch_count() - launches0
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    red_dev = dev if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([total_ms], dtype=torch.float64, device=red_dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    n_tuples = n_main + n_delta
    value = n_tuples / (ms_per_step / 1e3)
    comm.close()
    if rank == 0:
        pk = peaks()
        peak_hbm = pk["hbm_gbs"] if pk else 6650.0
        kb = 8 if key == "u64" else 4 if key == "u32" else 16
        sb = strict_bytes(n_main, bits, n_delta, kb, dict_len, r.merged_len, r.merged_bits)
        achieved = sb / (ms_per_step / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": key_dtype(args.workload),
            "data": f"synthetic (datagen, seeded; BASELINE configs[{cfg_number(args.workload) - 1}])",
            "config": {"workload": WORKLOADS[args.workload],
                       "parallelism": f"row-sharded x{world}: root Step 1(a), Step 1(b) "
                                      f"{'by U_M value ranges on every rank (NEXT2)' if step1b == 'ranges' else 'on the root'}"
                                      f", XC broadcast, Step 2(b) by output rows (dm_merge_column_sharded, "
                                      f"{'NCCL' if backend == 'nccl' else 'host callbacks over ' + backend})",
                       "row_cuts": cuts, "l2": "flushed (512 MB write) before every timed step",
                       "timing": "CUDA events around the collective call on each rank, max over ranks"},
            "roofline": {"kernel": "whole sharded merge (strict bytes of the column / step time, all GPUs)",
                         "bound": "hbm", "achieved": achieved, "peak": peak_hbm * world, "unit": "GB/s",
                         "frac": achieved / (peak_hbm * world), "traffic": None,
                         "algorithmic_bytes_per_launch": sb},
            "cpu_baseline": None,
            "e2e": None,
            "gpu_launches": int(launches), "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--naive-step2", action="store_true",
                    help="also time the paper's unoptimized Step 2 (binary search per tuple, P:206-212)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import torch
    import paper_1109_6885_b200 as dm

    # BENCH_PG_BACKEND=gloo exercises the multi-rank path with several ranks on one
    # GPU (test use only; ranks never wait on each other inside a kernel).
    backend = os.environ.get("BENCH_PG_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        pg = dist
    red_dev = dev if backend == "nccl" else torch.device("cpu")

    cfg = cfg_number(args.workload)
    if world > 1 and cfg != 4:  # one column, split by rows over the ranks (strong scaling)
        rc = run_sharded(args, rank, world, local, dev, backend)
        dist.destroy_process_group()
        return rc
    table = cfg == 4
    # ---- inputs, resident in HBM
    if cfg == 5:
        cols = None
        dev_cols = [cfg5_device_inputs(dev, rank)]
    else:
        cols = host_columns(args.workload, rank, world)
        dev_cols = [device_inputs(c, dev) for c in cols]
    if table:
        merger = dm.TableMerger(dev_cols)
        n_tuples = merger.tuples
    else:
        merger = dm.ColumnMerger(*dev_cols[0])
        n_tuples = merger.n_total
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 2x the 126 MB L2

    for _ in range(max(args.warmup, 0)):
        merger.run_async()
    torch.cuda.synchronize()

    # ---- per-step breakdown (single column: eager launches, events at the step boundaries)
    s1a = s1b = s2 = eager_ms = None
    launches0 = dm.launch_count()
    if not table:
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
        s1a = [ev[k][0].elapsed_time(ev[k][1]) for k in range(args.steps)]
        s1b = [ev[k][1].elapsed_time(ev[k][2]) for k in range(args.steps)]
        s2 = [ev[k][2].elapsed_time(ev[k][3]) for k in range(args.steps)]
        eager_ms = [ev[k][0].elapsed_time(ev[k][3]) for k in range(args.steps)]
    else:
        for k in range(args.steps):
            merger.run_async()
        torch.cuda.synchronize()
    launches_per_merge = (dm.launch_count() - launches0) / max(args.steps, 1)

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
    if pg:
        pg.barrier()
    step_ms = [a.elapsed_time(b) for a, b in gev]
    total_ms = sum(step_ms)
    tot = torch.tensor([total_ms, float(n_tuples)], dtype=torch.float64, device=red_dev)
    if pg:
        t = tot[:1].clone()
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        n_all = tot[1:].clone()
        pg.all_reduce(n_all, op=pg.ReduceOp.SUM)
        total_ms, all_tuples = float(t.item()), float(n_all.item())
    else:
        all_tuples = float(n_tuples)
    ms_per_step = total_ms / args.steps
    value = all_tuples / (ms_per_step / 1e3)

    # ---- roofline of the dominant kernel (Step 2(b), k_recompress)
    pk = peaks()
    peak_hbm = pk["hbm_gbs"] if pk else 6650.0
    results = merger.results() if table else [merger.result()]
    key_bytes = [(UM.shape[1] if UM.dim() == 2 else UM.element_size()) for (UM, _, _, _, _) in dev_cols]
    sb = sum(strict_bytes(n_m, b, D.shape[0], kb, UM.shape[0], r.merged_len, r.merged_bits)
             for (UM, _, n_m, b, D), kb, r in zip(dev_cols, key_bytes, results))
    s2b = sum(step2_bytes(n_m, b, D.shape[0], UM.shape[0], r.merged_bits, r.delta_dict_len)
              for (UM, _, n_m, b, D), r in zip(dev_cols, results))
    traffic = None
    tinfo = {}
    tp = os.path.join(ROOT, "profiles", "recompress_traffic.json")
    if os.path.exists(tp) and not table:
        try:
            tinfo = json.load(open(tp)).get(args.workload, {})
            traffic = tinfo.get("traffic_bytes_per_launch")
        except Exception:
            traffic = None
    if not table:
        s2_ms = statistics.mean(s2)
        achieved = s2b / (s2_ms / 1e3) / 1e9
        roofline = {"kernel": "Step 2(b) (%s)" % (tinfo.get("kernel") or "k_recompress").split("(")[0].strip(),
                    "bound": "hbm", "achieved": achieved,
                    "peak": peak_hbm, "unit": "GB/s", "frac": achieved / peak_hbm, "traffic": traffic,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if pk else "fallback 6.65 TB/s",
                    "algorithmic_bytes_per_launch": s2b,
                    "gather_bound_note": "X_M lookups: measured L2 random-gather ceiling 2.8e11/s "
                                         "(profiles/r01/microbench_gather.jsonl)"}
        if tinfo.get("warp_instructions_per_launch"):
            # the same kernel against the instruction-issue roofline: one warp instruction per
            # cycle per SM sub-partition (148 SMs x 4) at the SM clock -- what bounds the
            # shared-memory XC lookups of cfg2
            clk_mhz = (pk or {}).get("sm_max_mhz", 1965.0)
            ipeak = 148 * 4 * clk_mhz * 1e6
            iach = tinfo["warp_instructions_per_launch"] / (s2_ms / 1e3)
            roofline["issue"] = {"bound": "issue", "achieved": iach, "peak": ipeak, "unit": "warp-instructions/s",
                                 "frac": iach / ipeak,
                                 "warp_instructions_per_launch": tinfo["warp_instructions_per_launch"],
                                 "ncu_issue_active_pct": tinfo.get("issue_active_pct"),
                                 "source": "instruction count from ncu --set full of this kernel "
                                           "(profiles/recompress_traffic.json), time from the events here"}
    else:
        achieved = sb / (ms_per_step / 1e3) / 1e9
        roofline = {"kernel": "whole table merge (all kernels, 300 columns)", "bound": "hbm", "achieved": achieved,
                    "peak": peak_hbm, "unit": "GB/s", "frac": achieved / peak_hbm, "traffic": None,
                    "algorithmic_bytes_per_launch": sb}

    # ---- optional: the paper's unoptimized Step 2 on the same merge (NEXT4)
    naive = None
    if args.naive_step2 and not table:
        prev_step2 = dm.get_tuning(dm.KNOB_STEP2)
        dm.set_tuning(dm.KNOB_STEP2, 1)
        nm = dm.ColumnMerger(*dev_cols[0])
        nm.run_async()
        torch.cuda.synchronize()
        nev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
        for row in nev:
            for e in row:
                e.record()
        torch.cuda.synchronize()
        for k in range(args.steps):
            flush.zero_()
            nm.run_async_timed(nev[k])
        torch.cuda.synchronize()
        dm.set_tuning(dm.KNOB_STEP2, prev_step2)
        nr = nm.result()
        same = bool(torch.equal(nr.merged_codes, results[0].merged_codes))
        n2 = statistics.mean(nev[k][2].elapsed_time(nev[k][3]) for k in range(args.steps))
        o2 = statistics.mean(s2)
        naive = {"step2_naive_ms": n2, "step2_opt_ms": o2, "opt_over_naive": n2 / o2, "identical_output": same,
                 "note": "UnOpt = binary search of every tuple's value in U' (P:206-212); Opt = X_M/X_D "
                         "recompression (Eq 11, P:272); paper's claim: 9-10x (P:336)"}
        del nm

    # ---- e2e through the public host-buffer API (H2D inputs + D2H results inside)
    e2e = None
    if not args.no_e2e and not table:
        UM, M, n_m, b, D = dev_cols[0]
        ctx = dm.HostContext(local)
        hUM, hD, hM = UM.cpu().pin_memory(), D.cpu().pin_memory(), M.cpu().pin_memory()
        kb = key_bytes[0]
        hU = (torch.empty(UM.shape[0] + D.shape[0], dtype=UM.dtype) if UM.dim() == 1 else
              torch.empty((UM.shape[0] + D.shape[0], 16), dtype=torch.uint8)).pin_memory()
        hMo = torch.empty(dm.words(n_tuples, 32), dtype=torch.int64).pin_memory()
        ctx.merge(hUM, hM, n_m, b, hD, hU, hMo)  # warm-up (allocations)
        if pg:
            pg.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            nU, nb, _ = ctx.merge(hUM, hM, n_m, b, hD, hU, hMo)
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        if pg:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=red_dev)
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            e2e_s = float(t.item())
        h2d = hUM.numel() * hUM.element_size() + hD.numel() * hD.element_size() + hM.numel() * 8
        d2h = nU * kb + dm.words(n_tuples, nb) * 8
        bi = pcie_bidirectional_gbs(dev)
        e2e = {"value": all_tuples / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s * 1e3,
               "path": "dm_merge_column_host (pinned host buffers, copies inside the timed call)",
               "pcie_bidirectional_gbs": bi,
               "pcie_bound_ms": (h2d + d2h) / (bi * 1e9) * 1e3 if bi else None,
               "pcie_note": "the copies' floor: (H2D + D2H bytes) / the measured concurrent both-direction "
                            "pinned copy rate of this box"}
        ctx.close()

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, ncpu = host_info()
        if cfg == 4:  # whole columns in parallel on the host cores (the paper's scheme (i))
            workers = max(1, min(ncpu or 1, 64))
            step = 300 // min(48, 2 * workers)  # a bounded sample: ~20-40 s of single-core work
            ocols = [datagen.make_config(4, column=j) for j in range(0, 300, step)]
            tuples, t = run_oracle_columns_parallel(ocols, workers)
            cpu_baseline = {"value": tuples / t, "unit": "column-tuples/s", "cores": workers, "kind": "oracle",
                            "sample": f"{len(ocols)} of the 300 cfg4 columns at full size (every "
                                      f"{step}th), oracle linear mode, one column per "
                                      f"task on {workers} host processes of {ncpu} ({cpu})"}
        else:
            ocols, sample = oracle_sample(args.workload)
            tuples, times = run_oracle(ocols, 1 if cfg == 5 else 2)
            cpu_baseline = {"value": tuples / min(times), "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": f"{sample}; oracle linear mode, best of {len(times)}, 1 thread of {ncpu} ({cpu})"}

    if rank == 0:
        r0 = results[0]
        cfgd = {"workload": WORKLOADS[args.workload], "columns_per_rank": len(dev_cols),
                "parallelism": (f"column-sharded x{world}: LPT share of the 300 independent columns per rank "
                                f"(P:184, P:296), no collective" if table else "single GPU"),
                "l2": "flushed (512 MB write) before every timed step",
                "timing": "CUDA-graph replay of the whole merge, CUDA events on the launching stream"}
        if not table:
            UM, M, n_m, b, D = dev_cols[0]
            cfgd.update({"n_main": n_m, "n_delta": int(D.shape[0]), "dict_len": int(UM.shape[0]), "main_bits": b,
                         "merged_len": r0.merged_len, "merged_bits": r0.merged_bits})
        line = {
            "metric": METRIC if not table else "merged column-tuples/sec (sum over columns of N_M+N_D)",
            "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": key_dtype(args.workload),
            "data": f"synthetic (datagen, seeded; BASELINE configs[{cfg - 1}])", "config": cfgd,
            "hbm_fraction_strict": sb / (ms_per_step / 1e3) / 1e9 / peak_hbm,
            "roofline": roofline, "cpu_baseline": cpu_baseline, "e2e": e2e,
            **({"step2_naive_vs_opt": naive} if naive else {}),
            "gpu_launches": int(round(launches_per_merge * args.steps)),
            "gpu_launches_per_step": launches_per_merge,
            "clocks": clk.summary(),
        }
        if not table:
            line["steps_ms"] = {"s1a_delta_dict": statistics.mean(s1a), "s1b_dict_merge": statistics.mean(s1b),
                                "s2b_recompress": statistics.mean(s2), "eager_total": statistics.mean(eager_ms),
                                "graph_total": ms_per_step,
                                "note": "s1a/s1b/s2b from eager launches with events between steps; "
                                        "value/ms_per_step from CUDA-graph replays"}
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
