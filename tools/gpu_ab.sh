#!/bin/bash
# A/B of one environment knob on the default bench (c4 LvS) or the config given in the bench args:
# (each value twice, interleaved; prints it/s and the per-kernel ms).  Runs the knob's parity tests first.
set -u
TAG=$1; VAR=$2; VALS=$3; shift 3
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "sampled_csr or csr_lvs_solver_equals" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest.log
for rep in 1 2; do
  for v in $VALS; do
    env $VAR=$v timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e "$@" > $OUT/b_${v}_$rep.json 2>$OUT/b_${v}_$rep.err
    python -c "import json;d=json.load(open('$OUT/b_${v}_$rep.json'));print('$VAR=$v', round(d['value'],1), {k:v['ms'] for k,v in d['kernels'].items() if v['ms']>0.05})"
  done
done
