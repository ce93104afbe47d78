#!/bin/bash
# One GPU session: tests, N=1 bench, N=2 bench (if 2 GPUs), reference arm.
export CARAMEL_WATCHDOG_MS=3000
NG=$(nvidia-smi -L | wc -l)
timeout 400 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps ${STEPS:-50} --warmup 3 > gpurun_out/b1.json 2> gpurun_out/b1.err; echo "n1 rc=$?"; tail -2 gpurun_out/b1.err
if [ "$NG" -ge 2 ]; then
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $NG --steps ${STEPS:-50} --warmup 3 > gpurun_out/b$NG.json 2> gpurun_out/b$NG.err; echo "n$NG rc=$?"; grep -v Warning gpurun_out/b$NG.err | tail -3
fi
