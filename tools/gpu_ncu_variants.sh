#!/bin/bash
# ncu --set full of one kernel for each variant source: bash tools/gpu_ncu_variants.sh <dst.cu> <cfg> <mode> <kregex> <variant.cu>...
dst=$1; CFG=$2; MODE=$3; KRE=$4; shift 4
OUT=gpurun_out/nv; mkdir -p $OUT
for v in "$@"; do
  b=$(basename $v .cu)
  cp $v $dst
  python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo "build fail $v"; continue; }
  CMD="python bench.py --config $CFG --mode $MODE --steps 3 --warmup 3 --profile-only --no-cpu-baseline --no-e2e"
  $CMD > $OUT/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$KRE -s 4 -c 1 -o $OUT/$b $CMD > $OUT/ncu_$b.log 2>&1
  echo "$b rc=$?"
done
