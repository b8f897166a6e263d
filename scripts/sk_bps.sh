#!/bin/bash
cd "$(dirname "$0")/.."
for b in 1 2 3 4 6 8; do
  TOPO_SK_FUSE=0 TOPO_SK_BPS=$b timeout 300 python scripts/quick_pass.py 5 --passes=2 > gpurun_out/plain_bps.log 2>&1 && \
  TOPO_SK_FUSE=0 TOPO_SK_BPS=$b timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_sk_store --csv --log-file gpurun_out/bps_$b.csv python scripts/quick_pass.py 5 --passes=2 > /dev/null 2>&1
done
