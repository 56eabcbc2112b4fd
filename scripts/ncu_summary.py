"""Summarise an ncu report: key throughput, occupancy and stall metrics (run here, no GPU)."""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "lts__t_requests_srcunit_tex.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "smsp__inst_executed_op_shared_ld.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    for v in rows[2:]:
        d = dict(zip(h, v))
        u = dict(zip(h, units))
        print("==", d.get("Kernel Name", "")[:90])
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]:>16s} {u.get(k, '')}")
        stalls = sorted(((float(d[k].replace(',', '')), k) for k in d
                         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
                         and d[k] not in ("", "n/a")), reverse=True)[:6]
        print("  top stalls:", ", ".join(f"{k.split('stalled_')[1]}={int(v)}" for v, k in stalls))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
