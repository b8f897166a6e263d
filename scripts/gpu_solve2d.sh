#!/bin/bash
# 2D state solves (C1-C3 grids): node-centric fine level vs colour launches; tests
set -u
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_solve.py -q -x 2>&1 | tail -1
for v in "TOPO_MG_NODE2D=0" "X=1"; do
  echo "== $v"
  for c in 1 2 3; do env $v timeout 300 python scripts/solve_bench.py $c mg,mg 2>&1 | tail -1; done
done
