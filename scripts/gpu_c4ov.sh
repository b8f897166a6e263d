#!/bin/bash
# sK overlap on the mid-size configs (C4 3D, C3 2D)
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
run() { # name, config, env...
  local n=$1 c=$2; shift 2
  env "$@" timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > $OUT/ov_$n.json 2> $OUT/ov_$n.err
  python -c "
import json,sys;d=json.load(open('$OUT/ov_$n.json'));print('$n',round(d['value'],1),round(d['ms_per_step'],4),round(d['e2e']['value']),{k:round(v,3) for k,v in d['stages_ms'].items()})" || tail -3 $OUT/ov_$n.err
}
for c in 4 3 2; do
run c${c}_base $c TOPO_SK_OVERLAP=0
run c${c}_ov $c TOPO_SK_OVERLAP=1
run c${c}_ov_bps4 $c TOPO_SK_OVERLAP=1 TOPO_SK_BPS=4
run c${c}_base2 $c TOPO_SK_OVERLAP=0
done
