#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_baseline_sizes.py -m gpu -q -x > gpurun_out/gputest.txt 2>&1; echo "gputest rc=$?"
tail -1 gpurun_out/gputest.txt
SWEEP_MAX=$((1<<30)) SWEEP_ENGINES=single SWEEP_DEPTHS=1,3,8 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29512 tools/sweep.py > gpurun_out/sweep_depth2.jsonl 2> gpurun_out/sweep_depth2.err
echo "sweep rc=$?"
NCCL_ALGO="allreduce:nvls" SWEEP_MAX=$((1<<30)) SWEEP_ENGINES=single timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29513 tools/sweep.py > gpurun_out/sweep_ncclnvls.jsonl 2> gpurun_out/sweep_ncclnvls.err
echo "sweep nccl-nvls rc=$?"
echo done
