#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for g in 4 8 16 32; do
CARAMEL_E2E_GROUP_MB=$g timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-exposed > gpurun_out/e2e_g$g.json 2>gpurun_out/e2e_g$g.err; echo "g=$g rc=$?"
done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"
echo done
