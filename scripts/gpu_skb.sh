#!/bin/bash
# overlapped sK store (C5), repeated; plus the serial store alone
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
for v in "X=1" "X=1" "X=1" "TOPO_SK_OVERLAP=0" "TOPO_SK_OVERLAP=0 TOPO_SK_BPS=2"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $OUT/skb.json 2>$OUT/skb.err
  python -c "
import json;d=json.load(open('$OUT/skb.json'));print('$v',round(d['value'],1),round(d['ms_per_step'],4),round(d['stages_ms']['sk_store'],3),round(d['stages_ms']['pass'],3))" || tail -3 $OUT/skb.err
done
