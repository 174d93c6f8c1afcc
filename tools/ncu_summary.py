"""Summarise ncu --set full captures (one launch each) into a markdown table + traffic.json.

python tools/ncu_summary.py <out.md> <traffic.json> <cfg>:<bench-kernel-name>:<report.ncu-rep> ...
"""
import csv
import json
import subprocess
import sys

WANT = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram read"),
        ("dram__bytes_write.sum", "dram write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
        ("launch__block_size", "block")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}, v[h.index("Kernel Name")] if "Kernel Name" in h else "?"


md = ["| config | kernel | " + " | ".join(n for _, n in WANT) + " | traffic (B) |",
      "|---|---|" + "---|" * len(WANT) + "---|"]
traffic = {}
for arg in sys.argv[3:]:
    cfg, bname, rep = arg.split(":", 2)
    m, kname = raw(rep)
    cells = []
    for key, _ in WANT:
        val, unit = m.get(key, ("", ""))
        cells.append(f"{val} {unit}".strip())
    rd = float(m["dram__bytes_read.sum"][0].replace(",", "")) * SCALE.get(m["dram__bytes_read.sum"][1], 1)
    wr = float(m["dram__bytes_write.sum"][0].replace(",", "")) * SCALE.get(m["dram__bytes_write.sum"][1], 1)
    traffic.setdefault(cfg, {})[bname] = int(rd + wr)
    md.append(f"| {cfg} | `{kname.split('(')[0][:48]}` | " + " | ".join(cells) + f" | {int(rd + wr):.3e} |")
open(sys.argv[1], "w").write("\n".join(md) + "\n")
json.dump(traffic, open(sys.argv[2], "w"), indent=1)
print("\n".join(md))
