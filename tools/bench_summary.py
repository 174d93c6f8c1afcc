"""One-screen summary of a bench.py JSON line."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
c = d["config"]
print(f"{c['workload']} {c['mode']}: {d['value']:.1f} {d['unit']}  ms/step {d['ms_per_step']:.4f}  "
      f"exact {d.get('exact_iters_per_s')}  e2e {d['e2e']['value'] if d.get('e2e') else None}")
r = d["roofline"]
print(f"  roofline {r['kernel']}: {r['achieved']} {r['unit']} frac {r['frac']}  share {r['share_of_step']:.2f}")
print("  lvs", d.get("lvs_stats_mean"), "rf_ms", d.get("rangefinder_ms"))
for k, v in sorted(d["kernels"].items(), key=lambda kv: -kv[1]["ms"] * kv[1]["launches_per_step"]):
    print(f"   {k:28s} {v['ms']:9.4f} ms x{v['launches_per_step']}  {v['gbs']} GB/s")
