#!/bin/bash
# Round-2 checkpoint: build, the whole GPU suite, smoke, the default bench line (+ reference arm),
# per-config bench lines, launch lists and ncu --set full captures of the dominant kernels.
set -u
TAG=${1:-ckpt}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 2400 python -m pytest tests -m gpu -q -rA > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed" $OUT/pytest.log | tail -3
  python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
fi
timeout 1800 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "bench rc=$?"; cut -c1-300 $OUT/bench_default.json
if [ "${SKIP_REF:-0}" != 1 ]; then
  timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "ref rc=$?"; cut -c1-200 $OUT/bench_reference.json
fi
for cm in c1:lvs c2:lvs c2:exact c3:lvs c3:exact c4:exact c5:lai; do
  C=${cm%%:*}; M=${cm#*:}
  timeout 900 python bench.py --config $C --mode $M --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/b_${C}_$M.json 2>$OUT/b_${C}_$M.err
  python -c "import json;d=json.load(open('$OUT/b_${C}_$M.json'));print('$C $M', round(d['value'],1), d.get('roofline',{}).get('kernel'), round(d.get('roofline',{}).get('frac',0),3), d.get('rangefinder_ms',''))" 2>&1 | tail -1
done
prof() {  # name cfg mode regex count
  local CMD="python bench.py --config $2 --mode $3 --steps 3 --warmup 3 --profile-only --no-cpu-baseline --no-e2e"
  $CMD > $OUT/plain_$1.log 2>&1 || { echo "$1 plain failed"; return; }
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$1.csv $CMD > /dev/null 2>&1
  python tools/launch_summary.py $OUT/launches_$1.csv > $OUT/launches_$1.txt 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"$4" -s 4 -c $5 -o $OUT/full_$1 $CMD > $OUT/ncu_full_$1.log 2>&1
  echo "$1 ncu rc=$?"
}
prof c4_lvs c4 lvs "sampled_csr|sweep_stream|leverage_fused" 5
prof c4_exact c4 exact "^spmm_nnz$" 1
prof c3_lvs c3 lvs "tc_sampled" 1
prof c3_exact c3 exact "tc_gemm" 1
prof c2_lvs c2 lvs "sweep_fused|leverage_fused|sampled_csr" 3
prof c5_lai c5 lai "lai_sweep_fused" 1
python tools/rf_prof.py > $OUT/rf.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_rf.csv python tools/rf_prof.py > /dev/null 2>&1
python tools/launch_summary.py $OUT/launches_rf.csv > $OUT/launches_rf.txt 2>&1
for f in $OUT/full_*.ncu-rep; do python tools/ncu_brief.py $f; done > $OUT/ncu_brief.txt 2>&1
cat $OUT/ncu_brief.txt | cut -c1-250
