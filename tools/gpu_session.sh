#!/bin/bash
# Scratch GPU session driven through gpurun during development (rewritten per experiment):
#   /usr/local/graft/bin/gpurun --gpus N -- "bash tools/gpu_session.sh"
set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests1.txt 2>&1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/b1.json 2> gpurun_out/b1.err
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-exposed --no-zero-copy"
timeout 600 $CMD > gpurun_out/n1_plain.json 2> gpurun_out/n1_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n1_launches.csv $CMD > gpurun_out/n1_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_local_flat_tma -s 3 -c 1 -o gpurun_out/n1_full -f $CMD > gpurun_out/n1_ncu2.log 2>&1
echo done
