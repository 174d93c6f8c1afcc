"""Warp-state breakdown (stall reasons, per issued instruction) of each launch in an ncu report.

python tools/ncu_stalls.py <report.ncu-rep> [kernel-substring]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
pre = "smsp__average_warps_issue_stalled_"
suf = "_per_issue_active.ratio"
for v in rows[2:]:
    name = v[h.index("Kernel Name")].split("(")[0]
    if want and want not in name:
        continue
    st = []
    for i, key in enumerate(h):
        if key.startswith(pre) and key.endswith(suf):
            try:
                x = float(v[i].replace(",", ""))
            except ValueError:
                continue
            if x >= 0.05:
                st.append((x, key[len(pre):-len(suf)]))
    st.sort(reverse=True)
    print(name[:40], " ".join(f"{k}={x:.2f}" for x, k in st[:9]))
