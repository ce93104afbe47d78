#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
CARAMEL_LL_MAX=0 timeout 300 python tools/debug_push.py resnet50 inception_v3 > gpurun_out/debug_list_noll.txt 2>&1; echo "debug rc=$?"
timeout 900 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/gputest.txt 2>&1; echo "gputest rc=$?"
tail -3 gpurun_out/gputest.txt
CARAMEL_FUSED_PUSH=64 timeout 900 python -m pytest tests/test_gpu_baseline_sizes.py tests/test_gpu_kernels.py -m gpu -q -x -k "fused or many" > gpurun_out/gputest_fp.txt 2>&1; echo "gputest fused-push rc=$?"
tail -3 gpurun_out/gputest_fp.txt
echo done
