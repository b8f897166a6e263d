#!/bin/bash
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/t_gpu.log 2>&1; tail -1 $OUT/t_gpu.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err
timeout 300 python bench.py --config 4 --steps 20 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
echo done
