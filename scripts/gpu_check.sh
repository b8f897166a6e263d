#!/bin/bash
# quick HEAD check: GPU tests, smoke, C5 bench line
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x --durations=15 > $OUT/t_gpu.log 2>&1; tail -3 $OUT/t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err; cat $OUT/bench_c5.json | head -c 600
echo done
