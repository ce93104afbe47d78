#!/bin/bash
# balanced per-CTA ranges in the pull loop: parity, then the p=2 sweep (adaptive vs fixed depth)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_baseline_sizes.py tests/test_multigpu.py -x -q > gpurun_out/bal_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/bal_tests.txt
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29911 \
   bench.py --gpus 2 --steps 20 --warmup 5 --no-cpu-baseline --no-exposed --no-zero-copy > gpurun_out/bal_n2.json 2> gpurun_out/bal_n2.err; echo "n2 rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bal_n2.json").read().strip().splitlines()[-1])
print("step", d["ms_per_step"], d["roofline"]["frac"])
for r in d.get("bucket_sweep", []):
    print(r["bytes"], r["depth"], r["caramel_us"], r.get("fixed_depth_us"), r.get("gated_us"), r["nccl_us"])
PY
echo done
