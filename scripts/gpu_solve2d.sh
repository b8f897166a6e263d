#!/bin/bash
# 2D state solves (C1-C3 grids): exact coarsest solve up to 4096 DOFs
set -u
cd "$(dirname "$0")/.."
for v in "X=1" "TOPO_MG_DENSE_MAX=4096"; do
  echo "== $v"
  for c in 1 2 3; do env $v timeout 300 python scripts/solve_bench.py $c mg,mg 2>&1 | tail -1; done
  env $v timeout 300 python scripts/solve_bench.py 4 mg,mg 2>&1 | tail -1
done
