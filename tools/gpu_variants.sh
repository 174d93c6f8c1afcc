#!/bin/bash
# A/B a kernel source: bash tools/gpu_variants.sh <dst.cu> "<bench cfg:mode[:rule] ...>" <variant.cu>...
dst=$1; specs=$2; shift 2
OUT=gpurun_out/var; mkdir -p $OUT
for v in "$@"; do
  cp $v $dst
  python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo "build fail $v"; tail -5 $OUT/build.log; continue; }
  for spec in $specs; do
    IFS=: read c m r <<< "$spec"
    for rep in 1 2; do
      timeout 600 python bench.py --config $c --mode $m --rule ${r:-hals} --steps 20 --no-cpu-baseline --no-e2e > $OUT/b.json 2> $OUT/b.err
      python - $v $spec <<'PY'
import json, sys
d = json.loads(open("gpurun_out/var/b.json").read().strip().splitlines()[-1])
ks = d.get("kernels", {})
top = sorted(ks.items(), key=lambda kv: -kv[1]["ms"] * kv[1]["launches_per_step"])[:2]
print(f"{sys.argv[1].split('/')[-1]:28s} {sys.argv[2]:10s} {d['value']:10.1f} {d['unit']}  " +
      "  ".join(f"{k} {v['ms']:.4f}" for k, v in top), flush=True)
PY
    done
  done
done
