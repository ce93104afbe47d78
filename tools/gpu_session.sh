#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python tools/stress_local.py > gpurun_out/stress_local.jsonl 2> gpurun_out/stress_local.err; echo "stress_local rc=$?"
tail -3 gpurun_out/stress_local.jsonl gpurun_out/stress_local.err
echo done
