"""Summarise an ncu --csv launch list (gpu__time_duration.sum per kernel)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[h], rows[h + 1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in data:
    agg.setdefault(r[ki].split("(")[0][:70], []).append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':70s} {'n':>4s} {'mean_us':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:70s} {len(v):4d} {sum(v)/len(v)/1e3:9.2f} {sum(v)/tot:6.1%}")
print(f"total {tot/1e3:.1f} us")
