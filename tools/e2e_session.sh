#!/bin/bash
# e2e host-buffer pipeline: tapered first/last groups vs flat 16 MiB groups (N=1)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_executor.py -x -q > gpurun_out/e2e_tests.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/e2e_tests.txt
for rep in 1 2; do
 for t in 0 1 2 4; do
  CARAMEL_E2E_TAPER_MB=$t timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/e2e_t$t.json 2> gpurun_out/e2e.err
  python - $t <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/e2e_t{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("taper", sys.argv[1], "MiB:", d["e2e"]["value"], "GB/s", d["e2e"]["ms_per_step"], "ms", d["e2e"]["groups"], "groups; value", d["value"])
PY
 done
done
