#!/bin/bash
# Scratch GPU session driven through gpurun during development (rewritten per experiment):
#   /usr/local/graft/bin/gpurun --gpus N -- "bash tools/gpu_session.sh"
set -x
export PYTHONUNBUFFERED=1
for i in 1 2 3; do
timeout 600 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/mg_rep$i.txt 2>&1; echo "rep $i rc=$?"
done
echo done
