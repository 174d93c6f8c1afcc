"""Top SASS instructions by warp-stall samples for one kernel of an ncu report (source page).

python tools/ncu_hotsass.py <report> <kernel-regex> [top]
"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[h]
si, ni = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = [(int(r[ni] or 0), r[si].strip(), i) for i, r in enumerate(rows[h + 1:]) if len(r) > ni and r[ni].isdigit()]
tot = sum(d[0] for d in data)
print(f"total samples {tot}")
for cnt, src, i in sorted(data, reverse=True)[:top]:
    print(f"{cnt:7d} {100*cnt/tot:5.1f}%  [{i:5d}] {src[:90]}")
# by opcode
agg = {}
for cnt, src, _ in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    agg[op.split(".")[0]] = agg.get(op.split(".")[0], 0) + cnt
print(" ".join(f"{k}={100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:14]))
