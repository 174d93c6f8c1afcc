#!/bin/bash
# ncu evidence for one config: launch list of the timed loop + one --set full capture of a kernel.
# usage: bash tools/gpu_ncu.sh <tag> <config> <mode> <kernel-regex> [skip]
set -u
TAG=$1; CFG=$2; MODE=$3; KRE=$4; SKIP=${5:-20}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
CMD="python bench.py --config $CFG --mode $MODE --steps 3 --warmup 3 --profile-only --no-cpu-baseline --no-e2e"
$CMD > $OUT/plain_${CFG}_${MODE}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${CFG}_${MODE}.csv $CMD > $OUT/ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c 1 -o $OUT/full_${CFG}_${MODE} $CMD > $OUT/ncu_full.log 2>&1
echo "rc=$?"
python tools/launch_summary.py $OUT/launches_${CFG}_${MODE}.csv | head -30
