#!/bin/bash
# gated engine: 8 float4s in flight per thread and rank (GATED_U=8) at 16/32 CTAs vs the default (4, 32 CTAs)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
run() {  # model lib ctas tag
  CARAMEL_LIB=$2 CARAMEL_GATED_CTAS=$3 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700+RANDOM%200)) bench.py --gpus 2 --steps 10 --warmup 3 --model $1 --no-sweep --no-cpu-baseline \
    --no-zero-copy --no-nccl --exposed-engine gated > gpurun_out/gu.json 2> gpurun_out/gu.err
  python - "$@" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/gu.json").read().strip().splitlines()[-1])
e = d["exposed_comm"]
print(json.dumps({"model": sys.argv[1], "variant": sys.argv[4], "ctas": sys.argv[3],
                  "compute_ms": e["compute_ms"], "gated": e["engines"]["gated"]}), flush=True)
PY
}
DEF=paper_2004_14020_b200/csrc/libcaramel_b200.so
for rep in 1 2; do
for m in alexnet vgg16; do
  run $m $DEF 32 u4
  run $m tools/lib_gu8.so 16 u8
  run $m tools/lib_gu8.so 32 u8
done
done
echo done
