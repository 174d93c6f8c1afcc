set -u
OUT=gpurun_out/r2f; mkdir -p $OUT
python tools/rf_prof.py > $OUT/rf.log 2>&1; tail -3 $OUT/rf.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_rf.csv python tools/rf_prof.py > /dev/null 2>&1
python tools/launch_summary.py $OUT/launches_rf.csv | head -20
for sp in 1 2 3 5; do SYMNMF_SB_SPLITS=$sp timeout 600 python bench.py --config c3 --mode lvs --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c3_sp$sp.json 2>/dev/null; python -c "import json;d=json.load(open('$OUT/c3_sp$sp.json'));print('splits $sp', round(d['value'],1), d['kernels']['sampled_ah_dense'])"; done
CMD="python bench.py --config c3 --mode lvs --steps 3 --warmup 3 --profile-only --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"tc_sampled" -s 2 -c 1 -o $OUT/full_c3_tcs $CMD > $OUT/ncu1.log 2>&1
SYMNMF_SAMPLED_DENSE=simt ncu --set full --clock-control none --import-source on -k regex:"sampled_dense_v3" -s 2 -c 1 -o $OUT/full_c3_simt $CMD > $OUT/ncu2.log 2>&1
python tools/ncu_brief.py $OUT/full_c3_tcs.ncu-rep; python tools/ncu_brief.py $OUT/full_c3_simt.ncu-rep
python tools/ncu_stalls.py $OUT/full_c3_tcs.ncu-rep
