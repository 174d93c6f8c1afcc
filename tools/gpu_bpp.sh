#!/bin/bash
OUT=gpurun_out/bpp; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
for c in c2 c4; do
  timeout 600 python bench.py --config $c --rule bpp --steps 20 --no-cpu-baseline --no-e2e > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bpp $c rc=$?"
  python tools/bench_summary.py $OUT/bench_$c.json 2>/dev/null | head -6
done
timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e > $OUT/bench_c2_hals.json 2>&1; python tools/bench_summary.py $OUT/bench_c2_hals.json 2>/dev/null | head -6
