#!/bin/bash
# every overlapped engine (sm / gated / ce) in one process per model, comm-stream priority 0 vs -1
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/prio_mgpu.txt 2>&1; echo "mgpu rc=$?"; tail -1 gpurun_out/prio_mgpu.txt
for m in alexnet vgg16 resnet50; do
 for pr in 0 -1; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700+RANDOM%200)) bench.py --gpus 2 --steps 10 --warmup 3 --model $m --no-sweep --no-cpu-baseline \
    --no-zero-copy --no-nccl --comm-priority $pr > gpurun_out/pr_${m}_${pr}.json 2> gpurun_out/pr.err
  python - $m $pr <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/pr_{sys.argv[1]}_{sys.argv[2]}.json").read().strip().splitlines()[-1])
e = d["exposed_comm"]
print(json.dumps({"model": sys.argv[1], "prio": sys.argv[2], "compute_ms": e["compute_ms"],
                  "exposed": {k: [v["exposed_ms"]] + v["exposed_spread_ms"] for k, v in e["engines"].items()},
                  "errors": e.get("engine_errors")}), flush=True)
PY
 done
done
echo done
