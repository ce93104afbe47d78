#!/bin/bash
# gated SM engine: parity at 2 GPUs, then exposed communication (sm / gated / ce) and the bucket sweep
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/gated_mgpu.txt 2>&1; echo "mgpu rc=$?"; tail -3 gpurun_out/gated_mgpu.txt
for m in alexnet vgg16; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700+RANDOM%200)) \
   bench.py --gpus 2 --steps 10 --warmup 3 --model $m --no-sweep --no-cpu-baseline --no-zero-copy > gpurun_out/gated_$m.json 2> gpurun_out/gated_$m.err; echo "$m rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/gated_$m.json").read().strip().splitlines()[-1])
e=d.get("exposed") or d.get("exposed_comm") or {}
print("$m", json.dumps({k: e.get(k) for k in ("compute_ms","engines","engine_errors","nccl_ddp_exposed_ms")}))
PY
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29911 \
   bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/gated_resnet50.json 2> gpurun_out/gated_resnet50.err; echo "resnet rc=$?"
python - <<PY
import json
d=json.loads(open("gpurun_out/gated_resnet50.json").read().strip().splitlines()[-1])
e=d.get("exposed") or d.get("exposed_comm") or {}
print("resnet50", json.dumps({k: e.get(k) for k in ("compute_ms","engines","engine_errors","nccl_ddp_exposed_ms")}))
for r in d.get("bucket_sweep", []):
    print({k: r.get(k) for k in ("bytes","caramel_us","ce_us","gated_us","nccl_us")})
PY
echo done
