#!/bin/bash
# multigrid: parity tests, C5/C4 solve timings (three solves each; buffers persist in the context)
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_solve.py -q -x > $OUT/t_solve.log 2>&1; tail -1 $OUT/t_solve.log
for v in "X=1"; do
  echo "== $v"; env $v timeout 300 python scripts/solve_bench.py 5 mg,mg,mg 2>&1 | tail -3
done > $OUT/mgab.log
timeout 300 python scripts/solve_bench.py 4 mg,mg,mg >> $OUT/mgab.log 2>&1
cat $OUT/mgab.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_mg_c5_v5.csv python scripts/mg_prof.py 5 > $OUT/ncu_mg.log 2>&1
