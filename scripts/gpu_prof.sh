#!/bin/bash
# ncu --set full of the pass kernels on one config (default C5), one launch each
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
C=${1:-5}
timeout 300 python scripts/quick_pass.py $C --passes=1 > $OUT/plain_prof.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_conv|k_elem|k_eta|k_oc|k_sk" -c 8 -o $OUT/prof_c$C -f python scripts/quick_pass.py $C --passes=1 > $OUT/ncu_prof.log 2>&1
tail -2 $OUT/ncu_prof.log
