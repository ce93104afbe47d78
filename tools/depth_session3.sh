#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
DEPTHS=1,2 ITERS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_collective -s 6 -c 2 \
   -o gpurun_out/depth12_k_collective python tools/depth_probe.py > gpurun_out/depth12_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/depth12_ncu.log
