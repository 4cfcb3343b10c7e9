"""Summarise an `ncu --set full` report of one kernel into a small JSON file.

    python tools/ncu_summary.py report.ncu-rep out.json [algorithmic_bytes]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
UNIT = {"dram__bytes_read.sum": 1, "dram__bytes_write.sum": 1}

rep, out = sys.argv[1], sys.argv[2]
alg = float(sys.argv[3]) if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
res = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    s = {"kernel": d.get("Kernel Name", "")[:80]}
    for k in KEYS:
        if k in d:
            v = d[k].replace(",", "")
            try:
                v = float(v)
            except ValueError:
                pass
            # normalise byte counts to bytes
            if k.startswith("dram__bytes") and isinstance(v, float):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[k], 1)
                v *= scale
            if k == "gpu__time_duration.sum" and isinstance(v, float):
                v *= {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u[k], 1)
                k = "duration_us"
            s[k] = v
    if "dram__bytes_read.sum" in s:
        s["traffic_bytes"] = s["dram__bytes_read.sum"] + s["dram__bytes_write.sum"]
        if alg:
            s["algorithmic_bytes"] = alg
            s["traffic_over_algorithmic"] = s["traffic_bytes"] / alg
    res.append(s)
json.dump(res if len(res) > 1 else res[0], open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
