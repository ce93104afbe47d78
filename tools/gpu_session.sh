#!/bin/bash
# Scratch GPU session driven through gpurun during development (rewritten per experiment):
#   /usr/local/graft/bin/gpurun --gpus N -- "bash tools/gpu_session.sh"
set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.txt 2>&1
for m in alexnet vgg16 inception_v3; do
  B=64; [ $m = vgg16 ] && B=32
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --model $m --batch $B --no-cpu-baseline --no-sweep > gpurun_out/final_m_${m}_n4.json 2> gpurun_out/final_m_${m}_n4.err
done
echo done
