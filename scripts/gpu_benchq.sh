#!/bin/bash
# quick bench lines (all configs)
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
for c in 5 4 3 2 1; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bq_c$c.json 2> $OUT/bq_c$c.err
  python -c "
import json;d=json.load(open('$OUT/bq_c$c.json'));print($c,round(d['value'],1),round(d['ms_per_step'],4),round(d['e2e']['value'],1),d['stages_ms']['pass'],d['gpu_launches'])" || tail -3 $OUT/bq_c$c.err
done
