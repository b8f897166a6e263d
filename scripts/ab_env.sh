#!/bin/bash
# A/B of environment switches on one config: bash scripts/ab_env.sh CONFIG STEPS "A=1 B=2" "A=3" ...
# (each quoted argument is one variant's environment; "-" is the default build)
c=$1; n=$2; shift 2
for rep in 1 2; do for v in "$@"; do
  e="$v"; [ "$v" = "-" ] && e=""
  env $e python bench.py --config $c --steps $n --warmup 4 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$v]', round(d['ms_per_step'],4), round(d['value'],1), 'e2e_ms', round(d['e2e']['ms_per_step'],3), {k:round(v,4) for k,v in d['stages_ms'].items()}, flush=True)"
done; done
