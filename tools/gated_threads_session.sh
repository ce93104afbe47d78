#!/bin/bash
# gated engine: exposed comm vs CTA size (library variants) x grid cap, priority -1
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
run() {  # model lib ctas tag
  CARAMEL_LIB=$2 CARAMEL_GATED_CTAS=$3 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700+RANDOM%200)) bench.py --gpus 2 --steps 10 --warmup 3 --model $1 --no-sweep --no-cpu-baseline \
    --no-zero-copy --no-nccl --exposed-engine gated --comm-priority -1 > gpurun_out/gt.json 2> gpurun_out/gt.err
  python - "$@" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/gt.json").read().strip().splitlines()[-1])
e = d["exposed_comm"]
print(json.dumps({"model": sys.argv[1], "threads": sys.argv[4], "ctas": sys.argv[3],
                  "compute_ms": e["compute_ms"], "gated": e["engines"]["gated"]}), flush=True)
PY
}
DEF=paper_2004_14020_b200/csrc/libcaramel_b200.so
for m in alexnet vgg16; do
  run $m tools/lib_gt128.so 64 128
  run $m tools/lib_gt128.so 128 128
  run $m $DEF 32 256
  run $m $DEF 64 256
  run $m $DEF 128 256
  run $m tools/lib_gt512.so 32 512
done
echo done
