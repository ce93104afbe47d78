#!/bin/bash
# Scratch GPU session driven through gpurun during development (rewritten per experiment):
#   /usr/local/graft/bin/gpurun --gpus N -- "bash tools/gpu_session.sh"
set -x
export PYTHONUNBUFFERED=1
for v in 8192x3 4096x3x2 8192x3 4096x3x2; do
CARAMEL_TMA=$v timeout 300 python bench.py --no-exposed --no-cpu-baseline --no-zero-copy --steps 50 > gpurun_out/tma_$v.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/tma_$v.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])" >> gpurun_out/tma_sweep.txt
done
echo done
