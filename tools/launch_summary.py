"""Summarise an ncu --csv launch list (gpu__time_duration.sum per kernel).

Shares are of the solver's device time: the bench's instrumentation kernels (the profiling pass's
host-overlap `spin_kernel` and torch's fill of the L2-flush buffer) are listed separately.
"""
import collections
import csv
import sys

INSTRUMENTATION = ("spin_kernel", "FillFunctor")
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[h], rows[h + 1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in data:
    agg.setdefault(r[ki].split("(")[0][:70], []).append(float(r[vi].replace(",", "")))
inst = {k: v for k, v in agg.items() if any(s in k for s in INSTRUMENTATION)}
work = {k: v for k, v in agg.items() if k not in inst}
tot = sum(sum(v) for v in work.values())
print(f"{'kernel':70s} {'n':>4s} {'mean_us':>9s} {'share':>6s}")
for k, v in sorted(work.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:70s} {len(v):4d} {sum(v)/len(v)/1e3:9.2f} {sum(v)/tot:6.1%}")
print(f"total (solver kernels) {tot/1e3:.1f} us")
for k, v in inst.items():
    print(f"instrumentation, not in the shares: {k} x{len(v)} {sum(v)/1e3:.1f} us")
