#!/bin/bash
# smoothing sweeps per side on the loop's sharpening designs and C5
set -u
cd "$(dirname "$0")/.."
for v in 1 2 3 4; do
  echo "== nu $v"
  TOPO_MG_NU=$v timeout 600 tests/cpp/_build/test_driver --bench 96 48 48 10 2>&1 | awk '{print $2, $13, $16, $18}' | tail -3
  TOPO_MG_NU=$v timeout 300 python scripts/solve_bench.py 5 mg 2>&1 | tail -1
done
