#!/bin/bash
# gated push vs gated pull vs copy engines: parity at 2 GPUs, exposed comm (priority -1), sweep rows
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/gpush_mgpu.txt 2>&1; echo "mgpu rc=$?"; tail -3 gpurun_out/gpush_mgpu.txt
grep -i "mismatch\|failures" gpurun_out/gpush_mgpu.txt | head
run() {  # model engines gpush_ctas
  CARAMEL_GPUSH_CTAS=$3 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700+RANDOM%200)) bench.py --gpus 2 --steps 10 --warmup 3 --model $1 --no-sweep --no-cpu-baseline \
    --no-zero-copy --no-nccl --exposed-engine $2 --comm-priority -1 > gpurun_out/gp.json 2> gpurun_out/gp.err
  python - "$@" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/gp.json").read().strip().splitlines()[-1])
e = d["exposed_comm"]
print(json.dumps({"model": sys.argv[1], "gpush_ctas": sys.argv[3], "compute_ms": e["compute_ms"],
                  "engines": e["engines"], "errors": e.get("engine_errors")}), flush=True)
PY
}
for m in alexnet vgg16 resnet50; do
  run $m gated_push 16
  run $m gated_push 32
  run $m gated 16
  run $m ce 16
done
CARAMEL_GPUSH_CTAS=16 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29911 \
   bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-exposed --no-zero-copy > gpurun_out/gp_sweep.json 2> gpurun_out/gp_sweep.err; echo "sweep rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/gp_sweep.json").read().strip().splitlines()[-1])
for r in d.get("bucket_sweep", []):
    print({k: r.get(k) for k in ("bytes","caramel_us","ce_us","gated_us","gated_push_us","nccl_us")})
PY
echo done
