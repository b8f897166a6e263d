#!/bin/bash
# round evidence: GPU tests, smoke, bench lines (C5 default + C1..C4 + reference
# arm), the bench launch list, ncu --set full of the pass kernels (C5 and C4),
# solve / device-loop timings
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu > $OUT/t_gpu.log 2>&1; tail -1 $OUT/t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err
for c in 1 2 3 4; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err
done
timeout 600 python bench.py --impl reference > $OUT/bench_ref_c5.json 2> $OUT/bench_ref_c5.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench_c5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
timeout 300 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench_c4.csv python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench4.log 2>&1
timeout 300 python scripts/quick_pass.py 5 --passes=1 > $OUT/plain_prof.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_conv3|k_elem|k_eta|k_oc|k_sk" -c 9 -o $OUT/prof_full_c5 -f python scripts/quick_pass.py 5 --passes=1 > $OUT/ncu_full.log 2>&1
timeout 1500 ncu --set full --clock-control none -k regex:"k_conv3|k_elem|k_eta|k_oc|k_sk" -c 9 -o $OUT/prof_full_c4 -f python scripts/quick_pass.py 4 --passes=1 > $OUT/ncu_full4.log 2>&1
python scripts/ncu_summary.py $OUT/prof_full_c5.ncu-rep > $OUT/ncu_full_c5_summary.txt 2>&1
python scripts/ncu_summary.py $OUT/prof_full_c4.ncu-rep > $OUT/ncu_full_c4_summary.txt 2>&1
python scripts/make_ncu_json.py $OUT/prof_full_c5.ncu-rep "ncu --set full of scripts/quick_pass.py 5 (round 2)" $OUT/ncu_summary.json > /dev/null 2>&1
rm -f $OUT/prof_full_c5.ncu-rep $OUT/prof_full_c4.ncu-rep  # (gpurun copies back <= 64 MiB)
for c in 4 5 1 3; do timeout 300 python scripts/solve_bench.py $c mg; done > $OUT/solve.txt 2>&1
timeout 600 tests/cpp/_build/test_driver --bench 96 48 48 30 > $OUT/device_loop_96x48x48.txt 2>&1
echo done
