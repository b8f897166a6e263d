#!/bin/bash
# coarsest grid for the loop's sharpening designs: size, exact (cuSOLVER / Gauss-Jordan) vs Jacobi
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_solve.py -q -x > $OUT/t_solve.log 2>&1; tail -1 $OUT/t_solve.log
for v in "X=1" "TOPO_MG_MIN_DOFS=2000 TOPO_MG_DENSE_MAX=2048" "TOPO_MG_MIN_DOFS=8000 TOPO_MG_DENSE_MAX=8192"; do
  echo "== $v"
  env $v timeout 600 tests/cpp/_build/test_driver --bench 96 48 48 10 2>&1 | awk '{print $2, $14, $15, $16, $17, $18, $19}' | tail -4
  env $v timeout 300 python scripts/solve_bench.py 5 mg,mg 2>&1 | tail -1
  env $v timeout 300 python scripts/solve_bench.py 4 mg,mg 2>&1 | tail -1
done
