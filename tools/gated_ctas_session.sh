#!/bin/bash
# gated engine: exposed comm vs grid cap (CARAMEL_GATED_CTAS) and comm-stream priority
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
run() {  # model engine ctas prio
  CARAMEL_GATED_CTAS=$3 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700+RANDOM%200)) bench.py --gpus 2 --steps 10 --warmup 3 --model $1 --no-sweep --no-cpu-baseline \
    --no-zero-copy --no-nccl --exposed-engine $2 --comm-priority $4 > gpurun_out/gc.json 2> gpurun_out/gc.err
  python - "$@" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/gc.json").read().strip().splitlines()[-1])
e = d["exposed_comm"]
print(json.dumps({"model": sys.argv[1], "engine": sys.argv[2], "ctas": sys.argv[3], "prio": sys.argv[4],
                  "compute_ms": e["compute_ms"], "engines": e["engines"]}), flush=True)
PY
}
for m in alexnet vgg16; do
  for c in 8 16 32 64 148; do run $m gated $c 0; done
  run $m gated 32 -1
  run $m sm 32 -1
  run $m ce 32 0
done
echo done
