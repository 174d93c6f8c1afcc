#!/bin/bash
# One gpurun call: GPU tests, smoke, bench lines for the configs, ncu launch list.
# usage: gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tag] [configs...]'
set -u
TAG=${1:-r1}
shift || true
CFGS=${@:-c2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $OUT/gpu.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/summary.txt
tail -5 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $OUT/summary.txt
tail -2 $OUT/smoke.log
for c in $CFGS; do
  timeout 900 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench $c rc=$?" | tee -a $OUT/summary.txt
  tail -c 600 $OUT/bench_$c.json; tail -3 $OUT/bench_$c.err
done
