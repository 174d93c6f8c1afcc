#!/bin/bash
mkdir -p gpurun_out/dbg
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for d in ${DBGS:-0 1 2}; do
  SYMNMF_TILE_DBG=$d timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/dbg/c4_$d.json 2>/dev/null
  echo "dbg=$d"; python tools/bench_summary.py gpurun_out/dbg/c4_$d.json | grep -E "csr_tile|lvs:"
done
