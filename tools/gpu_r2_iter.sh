#!/bin/bash
# Round-2 iteration: build, targeted GPU tests, c4 benches (variants via env), launch lists.
# usage: bash tools/gpu_r2_iter.sh <tag> "<pytest -k expr>" "<name:cfg:mode:ENV=V,ENV2=V2[|bench args];...>"
set -u
TAG=$1; KEXPR=${2:-}; VARIANTS=${3:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
if [ -n "$KEXPR" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$KEXPR" > $OUT/pytest.log 2>&1
  echo "pytest rc=$?"; tail -15 $OUT/pytest.log
fi
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  [ -z "$v" ] && continue
  NAME=${v%%:*}; REST=${v#*:}; CFG=${REST%%:*}; REST=${REST#*:}; MODE=${REST%%:*}; ENVS=${REST#*:}
  ARGS=""; if [[ "$ENVS" == *"|"* ]]; then ARGS=${ENVS#*|}; ENVS=${ENVS%%|*}; fi
  ENVS=${ENVS//,/ }
  timeout 900 env $ENVS python bench.py --config $CFG --mode $MODE --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $ARGS > $OUT/b_$NAME.json 2> $OUT/b_$NAME.err
  echo "$NAME rc=$? $(python -c "import json;d=json.load(open('$OUT/b_$NAME.json'));print(round(d['value'],1), 'it/s', d.get('exact_iters_per_s') and round(d['exact_iters_per_s'],1), {k:v['ms'] for k,v in d['kernels'].items()})" 2>&1 | tail -1)"
done
