#!/bin/bash
# ncu --set full of one kernel (regex $2) in a C$1 pass
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
C=${1:-5}; K=${2:-k_elem}; N=${3:-1}
timeout 300 python scripts/quick_pass.py $C --passes=1 > $OUT/plain_prof1.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -c $N -o $OUT/prof1_c$C -f python scripts/quick_pass.py $C --passes=1 > $OUT/ncu_prof1.log 2>&1
tail -2 $OUT/ncu_prof1.log
