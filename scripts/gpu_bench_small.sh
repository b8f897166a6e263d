#!/bin/bash
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
for rep in 1 2 3; do for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bs_c${c}_$rep.json 2>/dev/null
done; done
echo done
