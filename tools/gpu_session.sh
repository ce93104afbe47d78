#!/bin/bash
# Scratch GPU session driven through gpurun during development (rewritten per experiment):
#   /usr/local/graft/bin/gpurun --gpus N -- "bash tools/gpu_session.sh"
set -x
export PYTHONUNBUFFERED=1
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611"
for v in "A TAIL_US=0 TAIL_FRAC=0" "B CE_MIN=1048576" "C CE_MIN=8388608" "D TAIL_US=500 TAIL_FRAC=0.05" "E"; do
  set -- $v; tag=$1; shift
  env ITERS=40 MODEL=vgg16 BATCH=32 ENGINE=ce "$@" $T tools/exposed_timeline.py > gpurun_out/tlv_$tag.txt 2>&1
done
echo done
