#!/bin/bash
# launch list of a C5 multigrid solve (2 PCG iterations incl. setup)
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python scripts/mg_prof.py 5 > $OUT/mgprof_plain.log 2>&1; tail -2 $OUT/mgprof_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_mg_c5.csv python scripts/mg_prof.py 5 > $OUT/ncu_mg.log 2>&1
tail -2 $OUT/ncu_mg.log
