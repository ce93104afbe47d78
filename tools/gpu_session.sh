#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "ll128" > gpurun_out/gputest_ll128.txt 2>&1; echo "ll128 rc=$?"
tail -3 gpurun_out/gputest_ll128.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/gputest.txt 2>&1; echo "gputest rc=$?"
tail -2 gpurun_out/gputest.txt
SWEEP_MAX=$((64<<20)) SWEEP_ENGINES=single,fused timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29512 tools/sweep.py > gpurun_out/sweep_ll128.jsonl 2> gpurun_out/sweep_ll128.err
echo "sweep rc=$?"
CARAMEL_LL128_MAX=0 SWEEP_MAX=$((64<<20)) SWEEP_ENGINES=single timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29512 tools/sweep.py > gpurun_out/sweep_noll128.jsonl 2> gpurun_out/sweep_noll128.err
echo "sweep2 rc=$?"
echo done
