"""Dynamic SASS opcode mix (warp-level instructions executed) per kernel from an ncu report.

  python tools/ncu_opmix.py gpurun_out/prof.ncu-rep [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = re.split(r'(?m)^"Kernel Name",', txt)
for b in blocks[1:]:
    name, rest = b.split("\n", 1)
    rows = list(csv.reader(io.StringIO(rest)))
    hdr = rows[0]
    ie = hdr.index("Instructions Executed")
    st = hdr.index("Warp Stall Sampling (All Samples)")
    mix = collections.Counter()
    stall = collections.Counter()
    tot = 0
    for r in rows[1:]:
        if len(r) <= ie:
            continue
        op = r[1].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        o = o.split(".")[0]
        n = int(r[ie] or 0)
        mix[o] += n
        stall[o] += int(r[st] or 0)
        tot += n
    print(name[:110])
    print(f"  total warp-instructions {tot:,}")
    for o, n in mix.most_common(top):
        print(f"  {o:10s} {n:14,d} {100*n/tot:5.1f}%   stall-samples {stall[o]}")
