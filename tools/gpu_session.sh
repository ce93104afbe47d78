#!/bin/bash
# Scratch GPU session driven through gpurun during development (rewritten per experiment):
#   /usr/local/graft/bin/gpurun --gpus N -- "bash tools/gpu_session.sh"
set -x
export PYTHONUNBUFFERED=1
for g in 6 8 12 16 24 32; do
CARAMEL_E2E_GROUP_MB=$g timeout 300 python bench.py --no-exposed --no-cpu-baseline --steps 10 > gpurun_out/e2e_$g.json 2>/dev/null
done
echo done
