"""Summarise an ncu --csv launch list: python scripts/launch_summary.py file.csv [filter]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, data = rows[0], rows[1:]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
flt = sys.argv[2] if len(sys.argv) > 2 else ""
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    name = r[ik].split("(")[0]
    if flt and flt not in name:
        continue
    agg[name][0] += 1
    agg[name][1] += float(r[iv].replace(",", ""))
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v[1] / 1e3:10.1f} us  {v[0]:5d} launches  {v[1] / 1e3 / v[0]:8.1f} us/launch  {100 * v[1] / tot:5.1f}%  {k}")
print(f"total {tot / 1e3:.1f} us")
