#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
nproc; cat /proc/loadavg
timeout 300 python tools/pcie_probe.py
for i in 1 2; do
timeout 900 python bench.py --steps 20 --warmup 5 --no-exposed > gpurun_out/e2c.json 2> gpurun_out/e2c.err
python -c "
import json; d=json.loads(open('gpurun_out/e2c.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e']['ms_per_step'], d['cpu_baseline']['value'])"
done
cat /proc/loadavg
