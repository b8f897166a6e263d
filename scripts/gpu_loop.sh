#!/bin/bash
# device redesign loop (gpu::run_optimization) on the top3D125 cantilever
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 600 tests/cpp/_build/test_driver --bench 96 48 48 10 > $OUT/device_loop_96x48x48.txt 2>&1; tail -3 $OUT/device_loop_96x48x48.txt
timeout 600 tests/cpp/_build/test_driver --bench 192 96 96 5 > $OUT/device_loop_192x96x96.txt 2>&1; tail -3 $OUT/device_loop_192x96x96.txt
