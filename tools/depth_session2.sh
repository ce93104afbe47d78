#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python tools/depth_probe.py; echo "probe rc=$?"
BYTES=67108864 timeout 300 python tools/depth_probe.py; echo "probe64 rc=$?"
P=4 timeout 300 python tools/depth_probe.py; echo "probe p4 rc=$?"
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_baseline_sizes.py tests/test_gpu_executor.py -x -q > gpurun_out/d2_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/d2_tests.txt
