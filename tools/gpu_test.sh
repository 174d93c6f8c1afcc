#!/bin/bash
# build + GPU tests (optionally a subset via -k) + one bench line
set -u
TAG=${1:-t}; K=${2:-}; CFG=${3:-c2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > $OUT/pytest_gpu.log 2>&1
else timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; fi
echo "pytest rc=$?"; tail -15 $OUT/pytest_gpu.log
for c in $CFG; do
timeout 600 python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench $c rc=$?"
python tools/bench_summary.py $OUT/bench_$c.json; tail -3 $OUT/bench_$c.err
done
