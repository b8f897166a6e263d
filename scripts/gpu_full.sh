#!/bin/bash
# round artefacts: gpu tests, smoke, bench (all configs), launch list + ncu full of the top kernel
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu > $OUT/t_gpu.log 2>&1; tail -3 $OUT/t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -2 $OUT/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref_c5.json 2> $OUT/bench_ref_c5.err
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench_c5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
timeout 300 python scripts/quick_pass.py 5 --passes=1 > $OUT/plain_prof.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_sk_store|k_conv|k_elem|k_eta|k_oc" -c 10 -o $OUT/prof_c5 -f python scripts/quick_pass.py 5 --passes=1 > $OUT/ncu_prof.log 2>&1
echo done
