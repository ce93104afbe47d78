#!/bin/bash
# bench every BASELINE model config on all GPUs of the box
export CARAMEL_WATCHDOG_MS=3000
NG=$(nvidia-smi -L | wc -l)
for M in ${MODELS:-inception_v3 alexnet vgg16}; do
  B=64; [ $M = vgg16 ] && B=32
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr 127.0.0.1 --master-port 2959$NG bench.py --gpus $NG --steps 30 --warmup 3 --model $M --batch $B --no-sweep > gpurun_out/m_${M}_n$NG.json 2> gpurun_out/m_${M}_n$NG.err; echo "$M rc=$?"
done
