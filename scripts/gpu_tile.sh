#!/bin/bash
# multigrid operators: parity tests, solve timings (variants), launch list
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_solve.py -q -x > $OUT/t_solve.log 2>&1; tail -3 $OUT/t_solve.log
TOPO_MG_MF1=0 timeout 300 python scripts/solve_bench.py 5 mg,mg > $OUT/solve_c5_nomf1.log 2>&1; tail -1 $OUT/solve_c5_nomf1.log
timeout 300 python scripts/solve_bench.py 5 mg,mg > $OUT/solve_c5_new.log 2>&1; tail -2 $OUT/solve_c5_new.log
timeout 300 python scripts/solve_bench.py 4 mg,mg > $OUT/solve_c4_new.log 2>&1; tail -2 $OUT/solve_c4_new.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_mg_c5_v3.csv python scripts/mg_prof.py 5 > $OUT/ncu_mg.log 2>&1
tail -1 $OUT/ncu_mg.log
