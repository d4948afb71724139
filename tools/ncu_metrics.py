"""Print selected raw metrics of an .ncu-rep (one row per profiled kernel).
usage: python tools/ncu_metrics.py report.ncu-rep [substring ...]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
keys = sys.argv[2:] or ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                        "sm__inst_executed_pipe_fp32", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
                        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
                        "smsp__issue_active.avg.pct", "lts__t_sector_hit_rate.pct"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u = rows[0], rows[1]
for r in rows[2:]:
    print("==", r[4][:90])
    for i, n in enumerate(h):
        if any(k in n for k in keys) and "per_second" not in n:
            print(f"  {n} [{u[i]}] {r[i]}")
