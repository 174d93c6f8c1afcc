#!/bin/bash
# Session 5: REDG microbenchmark, sharded-LAI + shuffled-scatter tests, A/B of the shuffled scatter on c4 LvS.
set -u
OUT=gpurun_out/s5b; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/red_bench.cu -o /tmp/red_bench && /tmp/red_bench 1965 > $OUT/red_bench.txt 2>&1
cat $OUT/red_bench.txt
timeout 1200 python -m pytest tests/test_gpu_shard.py tests/test_gpu_parity.py -m gpu -q -k "lai or sampled_csr or csr_lvs_solver_equals" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
for v in 0 1 0 1; do
  SYMNMF_SCATTER_SHFL=$v timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/b_shfl$v.json 2>$OUT/b_shfl$v.err
  python -c "import json;d=json.load(open('$OUT/b_shfl$v.json'));print('shfl=$v', round(d['value'],1), {k:v['ms'] for k,v in d['kernels'].items()})"
done
