#!/bin/bash
# Round-2 ncu evidence for the c4 kernels (LvS and EXACT), before/after changes.
# usage: bash tools/gpu_r2_prof.sh <tag> [what...]   what in: lvs exact exact_spmm
set -u
TAG=$1; shift
WHAT=${@:-lvs exact exact_spmm}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
prof() {  # name env mode regex count
  local NAME=$1 ENVS=$2 MODE=$3 KRE=$4 CNT=$5
  local CMD="python bench.py --config c4 --mode $MODE --steps 3 --warmup 3 --profile-only --no-cpu-baseline --no-e2e"
  env $ENVS $CMD > $OUT/plain_$NAME.log 2>&1 || { echo "$NAME plain failed"; tail -5 $OUT/plain_$NAME.log; return; }
  env $ENVS ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$NAME.csv $CMD > /dev/null 2>&1
  python tools/launch_summary.py $OUT/launches_$NAME.csv > $OUT/launches_$NAME.txt 2>&1
  env $ENVS ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 2 -c $CNT -o $OUT/full_$NAME $CMD > $OUT/ncu_full_$NAME.log 2>&1
  echo "$NAME rc=$?"
  cat $OUT/launches_$NAME.txt | head -14
}
for w in $WHAT; do
  case $w in
    lvs) prof c4_lvs "SYMNMF_X=1" lvs "sweep_fused|leverage_fused|sampled_csr" 3 ;;
    exact) prof c4_exact "SYMNMF_X=1" exact "csr_tile_sweep" 1 ;;
    exact_spmm) prof c4_exact_spmm "SYMNMF_CSR_TILE=never" exact "spmm_csr" 1 ;;
  esac
done
