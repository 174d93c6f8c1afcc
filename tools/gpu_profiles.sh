#!/bin/bash
# Round profiles: per config, the plain bench command, then an ncu launch list and one --set full
# capture of the dominant kernel (same command line, exited 0 just before).
set -u
OUT=gpurun_out/prof; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
prof() {  # cfg mode regex
  local CMD="python bench.py --config $1 --mode $2 --steps 3 --warmup 3 --profile-only --no-cpu-baseline --no-e2e"
  $CMD > $OUT/plain_$1_$2.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$1_$2.csv $CMD > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$3 -s 2 -c 1 -o $OUT/full_$1_$2 $CMD > $OUT/ncu_full_$1_$2.log 2>&1
  echo "$1 $2 rc=$?"
}
ONLY=${1:-all}   # optional: one of c2_lvs c3_lvs c3_exact c4_lvs c5_lai
run() { [ "$ONLY" = all ] || [ "$ONLY" = "$1_$2" ] && prof "$@"; }
run c2 lvs sweep_fused
run c3 lvs sampled_dense
run c3 exact tc_gemm
run c4 lvs sampled_csr
run c5 lai lai_sweep_fused
