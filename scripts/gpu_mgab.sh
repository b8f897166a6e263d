#!/bin/bash
# multigrid: parity tests, C5/C4 solve timings, C4 launch list
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_solve.py -q -x > $OUT/t_solve.log 2>&1; tail -1 $OUT/t_solve.log
for v in "X=1" "TOPO_MG_DENSE_COARSE=0"; do
  echo "== $v"
  env $v timeout 300 python scripts/solve_bench.py 5 mg,mg 2>&1 | tail -1
  env $v timeout 300 python scripts/solve_bench.py 4 mg,mg 2>&1 | tail -1
done > $OUT/mgab.log
cat $OUT/mgab.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_mg_c4.csv python scripts/mg_prof.py 4 > $OUT/ncu_mg4.log 2>&1
