#!/bin/bash
# build, a test subset, and bench lines: bash tools/gpu_quick.sh "<pytest -k>" "<cfg:mode:rule> ..."
OUT=gpurun_out/q; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -20 $OUT/build.log; exit 1; }
if [ -n "$1" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$1" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log; fi
for spec in $2; do
  IFS=: read c m r <<< "$spec"
  timeout 600 python bench.py --config $c --mode $m --rule ${r:-hals} --steps 20 --no-cpu-baseline --no-e2e > $OUT/b_${c}_$m.json 2> $OUT/b_${c}_$m.err; echo "$spec rc=$?"
  python tools/bench_summary.py $OUT/b_${c}_$m.json 2>/dev/null | head -6
done
