#!/bin/bash
# point-block Jacobi on the H8 operator levels: A/B + tests
set -u
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_solve.py -q -x 2>&1 | tail -1
for v in "TOPO_MG_BLOCK=0" "X=1" "X=1 TOPO_MG_OMEGA=1.0" "X=1 TOPO_MG_OMEGA=1.5"; do
  echo "== $v"
  env $v timeout 300 python scripts/solve_bench.py 5 mg 2>&1 | tail -1
  env $v timeout 300 python scripts/solve_bench.py 4 mg 2>&1 | tail -1
  env $v timeout 600 tests/cpp/_build/test_driver --bench 96 48 48 10 2>&1 | awk '{print $2, $16, $18}' | tail -3 | head -2
done
