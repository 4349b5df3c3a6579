"""Summarise an ncu --csv launch list: per kernel family, launches / total us / DRAM bytes.

  python tools/launch_summary.py gpurun_out/launches_cfg5.csv
"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
idi = hdr.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[1:]:
    per[r[idi]][r[mi]] = (float(r[vi].replace(",", "")), r[ui])
    names[r[idi]] = r[ki]
agg = collections.OrderedDict()
for i in sorted(per, key=int):
    n = re.sub(r"\(.*", "", names[i].replace("<unnamed>::", "")).replace("void ", "")
    n = re.sub(r"<.*", "", n) + ("<" + ",".join(re.findall(r"(float2|double2|\b\d+\b)", names[i])[:3]) + ">")
    t = per[i].get("gpu__time_duration.sum", (0, ""))
    us = t[0] / 1000.0 if t[1] in ("ns", "nsecond") else (t[0] * 1000 if t[1] in ("ms", "msecond") else t[0])
    rb = per[i].get("dram__bytes_read.sum", (0, "byte"))
    wb = per[i].get("dram__bytes_write.sum", (0, "byte"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    b = rb[0] * scale.get(rb[1], 1) + wb[0] * scale.get(wb[1], 1)
    a = agg.setdefault(n, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += us
    a[2] += b
tot = sum(a[1] for a in agg.values())
for n, (c, us, b) in agg.items():
    print(f"{n[:70]:70s} launches {c:4d}  {us:10.1f} us  {100 * us / tot:5.1f}%  dram {b / 1e6:9.1f} MB  {b / (us * 1e3) if us else 0:7.1f} GB/s")
