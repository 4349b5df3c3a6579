"""Warp-stall samples along the SASS of one kernel, in address-ordered chunks.

  python tools/ncu_regions.py report.ncu-rep <kernel-substring> [chunks]
"""
import csv
import io
import re
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
chunks = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
for b in re.split(r'(?m)^"Kernel Name",', txt)[1:]:
    name, rest = b.split("\n", 1)
    if pat not in name:
        continue
    rows = list(csv.reader(io.StringIO(rest)))
    hdr = rows[0]
    st = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    data = [(r[1].strip(), int(r[st] or 0), int(r[ie] or 0)) for r in rows[1:] if len(r) > ie]
    tot = sum(d[1] for d in data) or 1
    print(name[:100], "samples", tot)
    step = max(1, len(data) // chunks)
    for i in range(0, len(data), step):
        seg = data[i:i + step]
        ops = {}
        for d in seg:
            t = d[0].split()
            o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            ops[o] = ops.get(o, 0) + d[1]
        top = sorted(ops.items(), key=lambda kv: -kv[1])[:4]
        print(f"{i:5d} {100 * sum(d[1] for d in seg) / tot:5.1f}%  inst {sum(d[2] for d in seg):9d}  {top}")
    break
