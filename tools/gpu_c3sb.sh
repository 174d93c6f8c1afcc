# c3 LvS with the tensor-core sampled product: correctness spot check + variants
set -u
OUT=gpurun_out/${1:-c3sb}; mkdir -p $OUT
timeout 300 python tools/sb_check.py 2>&1 | grep -v simt | grep -v SWAP | tail -3
for v in "tc:X=1" "tc_sp1:SYMNMF_SB_SPLITS=1" "tc_sp3:SYMNMF_SB_SPLITS=3" "tc_sp8:SYMNMF_SB_SPLITS=8"; do
  NAME=${v%%:*}; E=${v#*:}
  env $E timeout 600 python bench.py --config c3 --mode lvs --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/c3_$NAME.json 2>$OUT/c3_$NAME.err
  python -c "import json;d=json.load(open('$OUT/c3_$NAME.json'));print('$NAME', round(d['value'],1), d['kernels']['sampled_ah_dense'])" 2>&1 | tail -1
done
