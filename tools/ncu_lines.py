"""Per-CUDA-line stall samples / instructions from an ncu report.

    python tools/ncu_lines.py report.ncu-rep [top] [kernel filter, e.g. regex:k_update]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kern = ["-k", sys.argv[3]] if len(sys.argv) > 3 else []  # e.g. regex:k_update
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda", *kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
lines = []
fname = ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "File Path", "Function Name") and len(r) == len(hdr):
        lines.append((fname, r))
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
stall = [(i, k) for i, k in enumerate(hdr) if k.startswith("stall_") and "Not Issued" not in k]
tot_s = sum(int(r[si] or 0) for _, r in lines)
tot_i = sum(int(r[ie] or 0) for _, r in lines)
print(f"samples {tot_s}  instructions {tot_i}")
lines.sort(key=lambda x: -int(x[1][si] or 0))
for f, r in lines[:top]:
    s = int(r[si] or 0)
    reasons = sorted(((int(r[i] or 0), k[6:]) for i, k in stall), reverse=True)[:3]
    rs = " ".join(f"{k}:{v}" for v, k in reasons if v)
    print(f"{f}:{r[0]:>4} {100 * s / tot_s:5.1f}% inst {100 * int(r[ie] or 0) / tot_i:5.1f}%  {r[1].strip()[:60]:<60} {rs}")
