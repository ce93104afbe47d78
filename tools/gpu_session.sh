#!/bin/bash
# Scratch GPU session driven through gpurun during development (rewritten per experiment):
#   /usr/local/graft/bin/gpurun --gpus N -- "bash tools/gpu_session.sh"
set -x
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/mg4.txt 2>&1
for pc in 1 0; do
for m in vgg16 alexnet; do
  B=64; [ $m = vgg16 ] && B=32
  CARAMEL_CE_PACED=$pc timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --model $m --batch $B --no-cpu-baseline --no-sweep --exposed-engine ce --no-nccl > gpurun_out/pace${pc}_${m}.json 2> gpurun_out/pace${pc}_${m}.err
done
done
echo done
