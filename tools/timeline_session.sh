#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for m in alexnet vgg16; do
 for e in gated ce sm; do
  echo "== $m $e"
  MODEL=$m ENGINE=$e PRIO=-1 BATCH=$([ $m = vgg16 ] && echo 32 || echo 64) timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port $((29700+RANDOM%200)) tools/exposed_timeline.py 2>&1 | grep -v "plan \|launch \|Warn\|\*\*\*" 
 done
done
