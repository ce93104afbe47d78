#!/bin/bash
export CARAMEL_WATCHDOG_MS=3000
NG=$(nvidia-smi -L | wc -l)
timeout 500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 50 --warmup 3 > gpurun_out/b1.json 2> gpurun_out/b1.err; echo "resnet n1 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $NG --steps 50 --warmup 3 > gpurun_out/b$NG.json 2> gpurun_out/b$NG.err; echo "resnet n$NG rc=$?"
MODELS="inception_v3 alexnet vgg16" bash tools/run_models.sh
