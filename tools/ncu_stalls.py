"""Warp-stall samples of one kernel grouped by the stalled instruction's opcode.

  python tools/ncu_stalls.py report.ncu-rep <kernel-substring> [top]

Each sample is attributed (by ncu) to the instruction the warp was waiting to
issue; the table shows, per opcode, its share of all samples and the dominant
stall reasons.
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
for b in re.split(r'(?m)^"Kernel Name",', txt)[1:]:
    name, rest = b.split("\n", 1)
    if pat not in name:
        continue
    rows = list(csv.reader(io.StringIO(rest)))
    hdr = rows[0]
    si = hdr.index("Source")
    stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    per = collections.defaultdict(collections.Counter)
    tot = collections.Counter()
    for r in rows[1:]:
        if len(r) <= max(stalls):
            continue
        op = r[si].strip().split()
        if not op:
            continue
        o = op[0]
        if o.startswith("@"):
            o = op[1] if len(op) > 1 else o
        o = o.split(".")[0]
        for i in stalls:
            try:
                v = float(r[i] or 0)
            except ValueError:
                continue
            if v:
                per[o][hdr[i][6:]] += v
                tot[hdr[i][6:]] += v
    allv = sum(tot.values())
    print(name[:110], f"samples {allv:.0f}")
    print("  overall:", ", ".join(f"{k} {v / allv:.1%}" for k, v in tot.most_common(8)))
    ranked = sorted(per.items(), key=lambda kv: -sum(kv[1].values()))
    for o, c in ranked[:top]:
        s = sum(c.values())
        print(f"  {o:10s} {s / allv:6.1%}  " + ", ".join(f"{k} {v / s:.0%}" for k, v in c.most_common(4)))
    break
