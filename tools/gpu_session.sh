#!/bin/bash
# Scratch GPU session driven through gpurun during development (rewritten per experiment):
#   /usr/local/graft/bin/gpurun --gpus N -- "bash tools/gpu_session.sh"
set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_executor.py -x -q > gpurun_out/tk.txt 2>&1
timeout 300 python tools/prof_pack.py > gpurun_out/pack.txt 2>&1
timeout 300 python tools/prof_pack.py >> gpurun_out/pack.txt 2>&1
echo done
