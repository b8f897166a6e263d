#!/bin/bash
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/t_gpu.log 2>&1; tail -1 $OUT/t_gpu.log
( TAG=default python scripts/overlap_stages.py 5
TAG=oc_late TOPO_OC_EARLY=0 python scripts/overlap_stages.py 5
TAG=oc_late_nonsk TOPO_OC_EARLY=0 python scripts/overlap_stages.py 5
timeout 300 python scripts/quick_pass.py 4 5 ) > $OUT/ov2.log 2>&1
echo done
