"""Key counters per kernel from an ncu report (raw page csv): time, DRAM bytes, fp64 instruction
mix, fp64 pipe utilisation, issue activity, occupancy."""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, data = rows[0], rows[1], rows[2:]
want = {
    "time_ms": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dfma": "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "dadd": "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "dmul": "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warp_inst": "smsp__inst_executed.sum",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "sm_ghz": "sm__cycles_elapsed.avg.per_second",
}
scale = {"ms": 1.0, "msecond": 1.0, "us": 1e-3, "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Ghz": 1.0, "Mhz": 1e-3}
out = []
for r in data:
    d = {"kernel": r[h.index("Kernel Name")].split("(")[0].split("::")[-1]}
    for k, m in want.items():
        if m in h:
            i = h.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            d[k] = v * scale.get(units[i], 1.0)
    out.append(d)
json.dump(out, sys.stdout, indent=1)
