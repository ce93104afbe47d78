#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "pack" > gpurun_out/gputest_pack.txt 2>&1; echo "pack tests rc=$?"; tail -1 gpurun_out/gputest_pack.txt
timeout 1200 python tools/stress_local.py > gpurun_out/stress_local2.jsonl 2> gpurun_out/stress_local2.err; echo "stress_local rc=$?"; cat gpurun_out/stress_local2.jsonl
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-exposed --no-zero-copy > gpurun_out/pack2.json 2> gpurun_out/pack2.err; echo "bench rc=$?"
echo done
