#!/bin/bash
# sK store overlapped with K3a + K4 (TOPO_SK_OVERLAP=1) at several blocks/SM
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_pass.py -q -m gpu -x > $OUT/t_gpu.log 2>&1; tail -2 $OUT/t_gpu.log
( timeout 300 python scripts/quick_pass.py 4 5
for b in 1 2 3 4 6; do echo "overlap bps=$b"; TOPO_SK_OVERLAP=1 TOPO_SK_BPS=$b timeout 300 python scripts/quick_pass.py 4 5; done ) > $OUT/quick.log 2>&1
TOPO_SK_OVERLAP=1 timeout 300 python scripts/quick_pass.py 5 --passes=2 > $OUT/plain5.log 2>&1 && \
TOPO_SK_OVERLAP=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5.csv python scripts/quick_pass.py 5 --passes=2 > $OUT/ncu_launch5.log 2>&1
echo done
