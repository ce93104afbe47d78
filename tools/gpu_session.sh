#!/bin/bash
# Scratch GPU session driven through gpurun during development (rewritten per experiment):
#   /usr/local/graft/bin/gpurun --gpus N -- "bash tools/gpu_session.sh"
set -x
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/mg4.txt 2>&1
for m in alexnet vgg16; do
  B=64; [ $m = vgg16 ] && B=32
  timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --model $m --batch $B --no-cpu-baseline --no-sweep > gpurun_out/m_${m}_n4.json 2> gpurun_out/m_${m}_n4.err
done
echo done
