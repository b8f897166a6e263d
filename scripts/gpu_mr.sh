#!/bin/bash
# multi-rank paths (threads on one GPU through host exchange; NCCL one-rank clique) + MG variants
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_variants.py tests/test_gpu_pass.py -q -x > $OUT/t_mr.log 2>&1; tail -3 $OUT/t_mr.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/torchrun1.json 2> $OUT/torchrun1.err; head -c 300 $OUT/torchrun1.json; echo
