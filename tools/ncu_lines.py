"""Warp-stall samples of one kernel per CUDA source line (innermost inlined line).

  python tools/ncu_lines.py report.ncu-rep <kernel-substring> [top]
"""
import csv
import io
import re
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
fname, func, hdr = None, None, None
out = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or func is None or pat not in func or r[0] == "":
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        n = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    if n == 0:
        continue
    st = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v)}
    out.append((n, f"{fname}:{r[0]}", r[1].strip()[:90], st))
tot = sum(o[0] for o in out)
out.sort(key=lambda o: -o[0])
print(f"total samples {tot}")
for n, loc, src, st in out[:top]:
    s = ", ".join(f"{k} {v * 100 // n}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:4])
    print(f"{n * 100 / tot:5.1f}%  {loc:22s} {s}\n        {src}")
