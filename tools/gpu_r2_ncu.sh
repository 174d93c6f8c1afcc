#!/bin/bash
# ncu --set full of chosen kernels of one c4 bench configuration (after the plain run exits 0).
# usage: bash tools/gpu_r2_ncu.sh <tag> <name> <cfg> <mode> "<kernel regex>" <count> [ENV=V ...]
set -u
TAG=$1; NAME=$2; CFG=$3; MODE=$4; KRE=$5; CNT=$6; shift 6
OUT=gpurun_out/$TAG; mkdir -p $OUT
[ -f paper_2402_08134_b200/libsymnmf.so ] || python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
CMD="python bench.py --config $CFG --mode $MODE --steps 3 --warmup 3 --profile-only --no-cpu-baseline --no-e2e"
env "$@" $CMD > $OUT/plain_$NAME.log 2>&1 || { echo "$NAME plain failed"; tail -5 $OUT/plain_$NAME.log; exit 1; }
env "$@" ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$NAME.csv $CMD > /dev/null 2>&1
python tools/launch_summary.py $OUT/launches_$NAME.csv > $OUT/launches_$NAME.txt 2>&1
env "$@" ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 4 -c $CNT -o $OUT/full_$NAME $CMD > $OUT/ncu_full_$NAME.log 2>&1
echo "$NAME ncu rc=$?"
head -14 $OUT/launches_$NAME.txt
python tools/ncu_brief.py $OUT/full_$NAME.ncu-rep 2>&1 | head -20
