#!/bin/bash
# GPU tests + bench lines of every config (quick round check)
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/t_gpu.log 2>&1; tail -3 $OUT/t_gpu.log
for c in 4 1 2 3; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err
  python - <<PY
import json
try:
    d=json.loads(open("$OUT/bench_c$c.json").read().strip().splitlines()[-1])
    print("C$c", round(d["ms_per_step"],4), "ms", round(d["value"],1), "Melem/s e2e", round(d["e2e"]["value"],1), {k:round(v,4) for k,v in d["stages_ms"].items()})
except Exception as e:
    print("C$c failed", e, open("$OUT/bench_c$c.err").read()[-500:])
PY
done
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err
python - <<PY
import json
d=json.loads(open("$OUT/bench_c5.json").read().strip().splitlines()[-1])
print("C5", round(d["ms_per_step"],4), "ms", round(d["value"],1), "Melem/s e2e", round(d["e2e"]["value"],1), {k:round(v,4) for k,v in d["stages_ms"].items()})
PY
