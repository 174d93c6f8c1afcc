"""Top SASS lines by warp-stall samples from `ncu -i rep --page source --csv --print-source sass -k <kernel>`."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
data = [(int(r[si]), r[0], r[src]) for r in rows[2:] if len(r) > si and r[si].isdigit()]
tot = sum(d[0] for d in data)
print("total samples", tot)
for i, (s, a, t) in enumerate(data):
    pass
for s, a, t in sorted(data, reverse=True)[:top]:
    print(f"{s:6d} {s/tot:6.1%} {a[-5:]} {t.strip()[:90]}")
