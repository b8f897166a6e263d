#!/bin/bash
# CUDA graph of the PCG iteration: A/B + tests
set -u
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_adapter.py -q -x 2>&1 | tail -1
for v in "TOPO_MG_GRAPH=0" "X=1"; do
  echo "== $v"
  for c in 5 4 1 2 3; do env $v timeout 300 python scripts/solve_bench.py $c mg,mg 2>&1 | tail -1; done
  env $v timeout 600 tests/cpp/_build/test_driver --bench 96 48 48 10 2>&1 | awk '{print $2, $14, $16, $18}' | tail -3 | head -2
done
