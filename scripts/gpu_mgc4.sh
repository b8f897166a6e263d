#!/bin/bash
# C4-size multigrid: launch list of 2 PCG iterations
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python scripts/mg_prof.py 4 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_mg_c4.csv python scripts/mg_prof.py 4 > $OUT/ncu_mg4.log 2>&1
tail -1 $OUT/ncu_mg4.log
