"""Summarise an .ncu-rep (raw page) into the handful of metrics that decide
a kernel's bound: `python tools/ncu_summary.py report.ncu-rep [name-filter]`."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem %"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "dmma pipe %"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor active %"),
    ("sm__inst_executed_pipe_xu_realtime.avg.pct_of_peak_sustained_elapsed", "xu %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def main():
    rep = sys.argv[1]
    filt = sys.argv[2] if len(sys.argv) > 2 else ""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    for row in rows[2:]:
        name = row[idx["Kernel Name"]]
        if filt not in name:
            continue
        print(name[:80])
        for k, label in KEYS:
            if k in idx:
                print(f"  {label:22s} {row[idx[k]]:>14s} {units[idx[k]]}")
        stalls = [(h, row[i]) for h, i in idx.items()
                  if h.startswith("smsp__average_warp_latency_issue_stalled") or
                  (h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("_not_issued"))]
        vals = []
        for h, v in stalls:
            try:
                vals.append((float(v.replace(",", "")), h))
            except ValueError:
                pass
        for v, h in sorted(vals, reverse=True)[:8]:
            print(f"  stall {h.split('stalled_')[-1]:30s} {v:g}")


if __name__ == "__main__":
    main()
