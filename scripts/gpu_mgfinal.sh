#!/bin/bash
# solve + device loop numbers at the current defaults; solve/adapter tests
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_adapter.py -q -x > $OUT/t_solve.log 2>&1; tail -1 $OUT/t_solve.log
{ timeout 300 python scripts/solve_bench.py 5 mg,mg 2>&1 | tail -2; timeout 300 python scripts/solve_bench.py 4 mg,mg 2>&1 | tail -2; for c in 1 2 3; do timeout 300 python scripts/solve_bench.py $c mg 2>&1 | tail -1; done; } > $OUT/mgab.log; cat $OUT/mgab.log
timeout 600 tests/cpp/_build/test_driver --bench 96 48 48 10 > $OUT/device_loop_96x48x48.txt 2>&1; tail -2 $OUT/device_loop_96x48x48.txt
timeout 600 tests/cpp/_build/test_driver --bench 192 96 96 5 > $OUT/device_loop_192x96x96.txt 2>&1; tail -2 $OUT/device_loop_192x96x96.txt
