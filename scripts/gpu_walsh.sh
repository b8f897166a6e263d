#!/bin/bash
# K3a: Walsh-block quadratic form (default for H8) vs the dense upper-triangle form
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/t_gpu.log 2>&1; tail -2 $OUT/t_gpu.log
( timeout 300 python scripts/quick_pass.py 1 2 3 4 5
echo "--- TOPO_ELEM_WALSH=0"; TOPO_ELEM_WALSH=0 timeout 300 python scripts/quick_pass.py 4 5 ) > $OUT/quick.log 2>&1
timeout 300 python scripts/quick_pass.py 5 --passes=2 > $OUT/plain5.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5.csv python scripts/quick_pass.py 5 --passes=2 > $OUT/ncu_launch5.log 2>&1
echo done
