#!/bin/bash
# Scratch GPU session driven through gpurun during development (rewritten per experiment):
#   /usr/local/graft/bin/gpurun --gpus N -- "bash tools/gpu_session.sh"
set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests4.txt 2>&1
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --no-exposed --no-cpu-baseline > gpurun_out/sw2.json 2> gpurun_out/sw2.err
echo done
