#!/bin/bash
# multigrid: parity tests, C5/C4 solve timings (A/B of the stored-level kernels)
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_solve.py -q -x > $OUT/t_solve.log 2>&1; tail -1 $OUT/t_solve.log
for v in "X=1" "TOPO_MG_LANES_MAX=0"; do
  echo "== $v"
  env $v timeout 300 python scripts/solve_bench.py 5 mg,mg 2>&1 | tail -1
  env $v timeout 300 python scripts/solve_bench.py 4 mg,mg 2>&1 | tail -1
done > $OUT/mgab.log
cat $OUT/mgab.log
