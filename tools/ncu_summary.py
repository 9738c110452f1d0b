"""Summarise an ncu --set full report into a JSON list (one entry per profiled launch).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/ncu_xxx.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
           "smsp__issue_active.avg.pct_of_peak_sustained_active"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
res = []
for r in rows[2:]:
    e = {"kernel": r[h.index("Kernel Name")]}
    for m in METRICS:
        if m in h:
            v = r[h.index(m)].replace(",", "")
            try:
                e[m] = float(v)
            except ValueError:
                e[m] = v
            e[m + ".unit"] = units[h.index(m)]
    res.append(e)
json.dump(res, sys.stdout, indent=1)
