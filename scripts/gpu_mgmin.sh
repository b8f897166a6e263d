#!/bin/bash
# coarsest-level size sweep (TOPO_MG_MIN_DOFS) on C4 and C5
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
for v in 20000 5000 2000 500 100; do
  echo "== min_dofs $v"
  TOPO_MG_MIN_DOFS=$v timeout 300 python scripts/solve_bench.py 4 mg,mg 2>&1 | tail -1
  TOPO_MG_MIN_DOFS=$v timeout 300 python scripts/solve_bench.py 5 mg,mg 2>&1 | tail -1
done > $OUT/mgmin.log
cat $OUT/mgmin.log
