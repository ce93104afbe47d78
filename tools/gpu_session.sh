#!/bin/bash
# Scratch GPU session driven through gpurun during development (rewritten per experiment):
#   /usr/local/graft/bin/gpurun --gpus N -- "bash tools/gpu_session.sh"
set -x
export PYTHONUNBUFFERED=1
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611"
ITERS=30 MODEL=vgg16 BATCH=32 ENGINE=ce $T tools/exposed_timeline.py > gpurun_out/tl2_vgg_ce.txt 2>&1
echo done
