#!/bin/bash
# one gpurun session: bench all configs, launch list + ncu capture of the top kernel
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python bench.py --steps 10 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err
done
timeout 300 python scripts/quick_pass.py 5 --passes=2 > $OUT/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5.csv python scripts/quick_pass.py 5 --passes=2 > $OUT/ncu_launch.log 2>&1
timeout 300 python scripts/quick_pass.py 4 --passes=2 > $OUT/plain4.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c4.csv python scripts/quick_pass.py 4 --passes=2 > $OUT/ncu_launch4.log 2>&1
timeout 300 python scripts/quick_pass.py 5 --passes=2 > $OUT/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sk_store -s 1 -c 1 -o $OUT/prof_sk_c5 -f python scripts/quick_pass.py 5 --passes=2 > $OUT/ncu_full.log 2>&1
echo done
