#!/bin/bash
# Scratch GPU session driven through gpurun during development (rewritten per experiment):
#   /usr/local/graft/bin/gpurun --gpus N -- "bash tools/gpu_session.sh"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/gputest.txt 2>&1; echo "gputest rc=$?"
tail -3 gpurun_out/gputest.txt
CARAMEL_FUSED_PUSH=64 timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py tests/test_gpu_kernels.py -m gpu -q -x -k "fused or many" > gpurun_out/gputest_fp.txt 2>&1; echo "gputest fused-push rc=$?"
tail -3 gpurun_out/gputest_fp.txt
for fp in 0 32 148; do
CARAMEL_FUSED_PUSH=$fp SWEEP_MAX=$((1<<30)) SWEEP_ENGINES=single,fused timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29512 tools/sweep.py > gpurun_out/sweep_fp$fp.jsonl 2> gpurun_out/sweep_fp$fp.err
echo "sweep $fp rc=$?"
done
echo done
