#!/bin/bash
# bench lines (C5 default + C1..C4), the reference arm, and the bench launch list
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err
done
timeout 600 python bench.py --impl reference > $OUT/bench_ref_c5.json 2> $OUT/bench_ref_c5.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
echo done
