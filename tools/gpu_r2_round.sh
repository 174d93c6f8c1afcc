#!/bin/bash
# Round-2 checkpoint: build, the whole GPU suite, smoke, the default bench line (+ reference arm),
# the launch list of the default bench command and one ncu --set full capture of its top kernels.
set -u
TAG=${1:-round}
OUT=gpurun_out/$TAG; mkdir -p $OUT
free -g > $OUT/host.txt 2>&1; nproc >> $OUT/host.txt; lscpu | grep "Model name" >> $OUT/host.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 2400 python -m pytest tests -m gpu -q -rA > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed" $OUT/pytest.log | tail -3
  python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
fi
timeout 1800 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "bench rc=$?"; cut -c1-600 $OUT/bench_default.json
if [ "${SKIP_REF:-0}" != 1 ]; then
  timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "ref rc=$?"; cut -c1-300 $OUT/bench_reference.json
fi
CMD="python bench.py --steps 3 --warmup 3 --profile-only --no-cpu-baseline --no-e2e"
$CMD > $OUT/plain_profile.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_default.csv $CMD > /dev/null 2>&1
python tools/launch_summary.py $OUT/launches_default.csv > $OUT/launches_default.txt 2>&1; head -16 $OUT/launches_default.txt
ncu --set full --clock-control none --import-source on -k regex:"sampled_csr|sweep_stream|leverage_fused" -s 6 -c 5 -o $OUT/full_default $CMD > $OUT/ncu_full.log 2>&1
echo "ncu rc=$?"; python tools/ncu_brief.py $OUT/full_default.ncu-rep 2>&1 | head
