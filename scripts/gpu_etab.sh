#!/bin/bash
# eta cooperative grid sizing: all configs + eta/pass parity tests
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_pass.py tests/test_gpu_stages.py tests/test_gpu_multirank.py -q -x 2>&1 | tail -1
for c in 5 4 3 2 1; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $OUT/eb.json 2>$OUT/eb.err
  python -c "
import json;d=json.load(open('$OUT/eb.json'));print($c,round(d['value'],1),round(d['ms_per_step'],4),round(d['stages_ms']['eta'],4),round(d['stages_ms']['pass'],4))" || tail -3 $OUT/eb.err
done
