#!/bin/bash
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python scripts/quick_pass.py 3 --passes=1 > $OUT/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_conv" -c 4 -o $OUT/prof_c3 -f python scripts/quick_pass.py 3 --passes=1 > $OUT/ncu_c3.log 2>&1
tail -2 $OUT/ncu_c3.log
