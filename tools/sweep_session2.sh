#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_baseline_sizes.py tests/test_multigpu.py -x -q > gpurun_out/sw2_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/sw2_tests.txt
bash tools/sweep_session.sh
