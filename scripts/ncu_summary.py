"""Key per-kernel metrics of an ncu --set full report as CSV: python scripts/ncu_summary.py REP"""
import csv
import io
import subprocess
import sys

M = [("time_ms", "gpu__time_duration.sum"), ("dram_read_MB", "dram__bytes_read.sum"),
     ("dram_write_MB", "dram__bytes_write.sum"), ("inst", "smsp__inst_executed.sum"),
     ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
     ("alu_pipe_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
     ("fma_pipe_pct", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
     ("lsu_pipe_pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
     ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
     ("regs", "launch__registers_per_thread"),
     ("smem_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
     ("smem_wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")]
STALLS = ["short_scoreboard", "wait", "not_selected", "math_pipe_throttle", "long_scoreboard", "barrier",
          "branch_resolving", "mio_throttle", "lg_throttle"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
w = csv.writer(sys.stdout)
w.writerow(["kernel"] + [m[0] for m in M] + ["stall_" + s for s in STALLS])
for r in rows[2:]:
    d = dict(zip(h, r))
    u = dict(zip(h, units))
    vals = []
    for name, key in M:
        v = d.get(key, "")
        if key.startswith("dram__bytes") and u.get(key) == "Gbyte":
            v = str(float(v) * 1000)
        if key == "gpu__time_duration.sum" and u.get(key) == "us":
            v = str(float(v) / 1000)
        vals.append(v)
    st = [d.get(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio", "") for s in STALLS]
    w.writerow([d["Kernel Name"].split("(")[0]] + vals + st)
