set -x
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_executor.py -x -q > gpurun_out/tk.txt 2>&1
timeout 300 python tools/prof_pack.py > gpurun_out/pack.txt 2>&1
echo done
