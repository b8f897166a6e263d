#!/bin/bash
# device redesign loop (gpu::run_optimization) on the top3D125 cantilever; adapter parity tests
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_adapter.py -q -x > $OUT/t_adapter.log 2>&1; tail -1 $OUT/t_adapter.log
TOPO_LOOP_DEVICE=0 timeout 600 tests/cpp/_build/test_driver --bench 96 48 48 10 > $OUT/device_loop_96x48x48_stages.txt 2>&1; tail -1 $OUT/device_loop_96x48x48_stages.txt
timeout 600 tests/cpp/_build/test_driver --bench 96 48 48 10 > $OUT/device_loop_96x48x48.txt 2>&1; tail -3 $OUT/device_loop_96x48x48.txt
TOPO_LOOP_DEVICE=0 timeout 600 tests/cpp/_build/test_driver --bench 192 96 96 5 > $OUT/device_loop_192x96x96_stages.txt 2>&1; tail -1 $OUT/device_loop_192x96x96_stages.txt
timeout 600 tests/cpp/_build/test_driver --bench 192 96 96 5 > $OUT/device_loop_192x96x96.txt 2>&1; tail -3 $OUT/device_loop_192x96x96.txt
