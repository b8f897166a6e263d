#!/bin/bash
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mg_apply_tile -s 2 -c 1 -o $OUT/prof_tile3_c5 -f python scripts/mg_prof.py 5 > $OUT/ncu_tile.log 2>&1
tail -2 $OUT/ncu_tile.log
