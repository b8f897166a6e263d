#!/bin/bash
# quick GPU iteration: parity tests, per-config timing, C5 bench both overlap modes, launch list
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/t_gpu.log 2>&1
tail -3 $OUT/t_gpu.log
timeout 300 python scripts/quick_pass.py 1 2 3 4 5 > $OUT/quick.log 2>&1
TOPO_SK_OVERLAP=1 timeout 300 python scripts/quick_pass.py 4 5 > $OUT/quick_ov.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err
TOPO_SK_OVERLAP=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c5_ov.json 2> $OUT/bench_c5_ov.err
timeout 300 python scripts/quick_pass.py 5 --passes=2 > $OUT/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5.csv python scripts/quick_pass.py 5 --passes=2 > $OUT/ncu_launch.log 2>&1
timeout 300 python scripts/quick_pass.py 3 --passes=2 > $OUT/plain3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3.csv python scripts/quick_pass.py 3 --passes=2 > $OUT/ncu_launch3.log 2>&1
echo done
