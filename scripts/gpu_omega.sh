#!/bin/bash
# damped-Jacobi weight sweep (C5 random field, loop's sharp designs, 2D C3)
set -u
cd "$(dirname "$0")/.."
for v in 0.9 1.2 1.33 1.5 1.7; do
  echo "== omega $v / lambda_max"
  TOPO_MG_OMEGA=$v timeout 300 python scripts/solve_bench.py 5 mg 2>&1 | tail -1
  TOPO_MG_OMEGA=$v timeout 300 python scripts/solve_bench.py 3 mg 2>&1 | tail -1
  TOPO_MG_OMEGA=$v timeout 600 tests/cpp/_build/test_driver --bench 96 48 48 10 2>&1 | awk '{print $2, $16, $18}' | tail -3 | head -2
done
