#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python tools/depth_probe.py; echo "probe rc=$?"
BYTES=67108864 timeout 300 python tools/depth_probe.py; echo "probe64 rc=$?"
DEPTHS=1,8 ITERS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_collective -s 6 -c 2 \
   -o gpurun_out/depth_k_collective python tools/depth_probe.py > gpurun_out/depth_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/depth_ncu.log
