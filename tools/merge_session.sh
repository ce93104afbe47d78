#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py tests/test_gpu_executor.py -x -q > gpurun_out/mg_tests.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/mg_tests.txt
bash tools/run_models.sh
python - <<'PY'
import json
for m in ["inception_v3","alexnet","vgg16"]:
    d=json.loads(open(f"gpurun_out/m_{m}_n4.json").read().strip().splitlines()[-1])
    e=d["exposed_comm"]
    print(m, d["ms_per_step"], "C", e["compute_ms"], {k:(v["exposed_ms"], v["exposed_spread_ms"]) for k,v in e["engines"].items()}, "ddp", e.get("nccl_ddp_exposed_ms"))
PY
