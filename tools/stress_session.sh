#!/bin/bash
# closing-build stress: 10,000 fused steps at N=2 and N=4 (ResNet-50) + 2,000 at N=4 (VGG-16), bit-exact
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
  tools/stress.py --steps 10000 --check 1000 > gpurun_out/stress_n2.jsonl 2> gpurun_out/stress_n2.err; echo "n2 rc=$?"; tail -1 gpurun_out/stress_n2.jsonl
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 \
  tools/stress.py --steps 10000 --check 1000 > gpurun_out/stress_n4.jsonl 2> gpurun_out/stress_n4.err; echo "n4 rc=$?"; tail -1 gpurun_out/stress_n4.jsonl
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29613 \
  tools/stress.py --steps 2000 --check 500 --model vgg16 > gpurun_out/stress_vgg_n4.jsonl 2> gpurun_out/stress_vgg_n4.err; echo "vgg n4 rc=$?"; tail -1 gpurun_out/stress_vgg_n4.jsonl
