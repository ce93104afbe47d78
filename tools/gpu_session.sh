#!/bin/bash
# Scratch GPU session driven through gpurun during development (rewritten per experiment):
#   /usr/local/graft/bin/gpurun --gpus N -- "bash tools/gpu_session.sh"
set -x
export PYTHONUNBUFFERED=1
for t in 1 2 4; do export CARAMEL_TILE_DIV=$t; unset CARAMEL_TILE_MULT;
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --no-exposed --no-cpu-baseline --no-nccl --no-zero-copy --steps 10 > gpurun_out/tile$t.json 2> gpurun_out/tile$t.err
done
echo done
