#!/bin/bash
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/t_gpu.log 2>&1; tail -3 $OUT/t_gpu.log
timeout 300 python scripts/quick_pass.py 1 2 3 4 5 > $OUT/quick.log 2>&1
timeout 300 python scripts/quick_pass.py 3 --passes=2 > $OUT/plain3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3.csv python scripts/quick_pass.py 3 --passes=2 > $OUT/ncu_launch3.log 2>&1
timeout 300 python scripts/quick_pass.py 5 --passes=1 > $OUT/plain_prof.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_conv|k_elem" -c 4 -o $OUT/prof_conv_c5 -f python scripts/quick_pass.py 5 --passes=1 > $OUT/ncu_prof.log 2>&1
echo done
