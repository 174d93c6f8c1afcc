"""One line per captured launch of an ncu report: the counters that decide what binds a kernel.

python tools/ncu_brief.py <report.ncu-rep> [extra-metric ...]
"""
import csv
import subprocess
import sys

KEYS = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "dramR"),
        ("dram__bytes_write.sum", "dramW"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
        ("lts__t_sector_hit_rate.pct", "L2hit%"), ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts%"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
        ("sm__inst_executed.avg.per_cycle_active", "ipc"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
        ("launch__occupancy_limit_registers", "occ_reg"), ("launch__occupancy_limit_shared_mem", "occ_smem")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}

rep = sys.argv[1]
extra = [(m, m.split("__")[-1][:24]) for m in sys.argv[2:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u = rows[0], rows[1]
for v in rows[2:]:
    cells = []
    for key, name in KEYS + extra:
        if key not in h:
            continue
        i = h.index(key)
        val, unit = v[i], u[i]
        if key == "Kernel Name":
            cells.append(val.split("(")[0][:40])
            continue
        try:
            x = float(val.replace(",", ""))
            if unit in SCALE:
                x *= SCALE[unit]
                if "bytes" in key:
                    x /= 1e6   # MB
            cells.append(f"{name}={x:.4g}")
        except ValueError:
            cells.append(f"{name}={val}")
    print("  ".join(cells))
