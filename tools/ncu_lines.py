"""Warp-stall samples per CUDA source line (ncu --page source --print-source cuda,sass)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg, cur, fname = {}, None, ""
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 5 or r[0] == "Line No":
        continue
    if r[0]:   # a source line row
        cur = (fname, r[0], r[1].strip()[:100])
        try:
            agg[cur] = agg.get(cur, 0) + int(r[4])
        except ValueError:
            pass
tot = sum(agg.values()) or 1
print("total samples", tot)
for (f, ln, src), s in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{s/tot:6.1%} {f}:{ln:>5} {src}")
