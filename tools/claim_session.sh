#!/bin/bash
# fused step: claim granularity of the dynamic item split (CARAMEL_FUSED_CLAIM; 0 = static) at p=2 and 4
export PYTHONUNBUFFERED=1
for n in 2 4; do
 for c in 0 1 2 4; do
  echo "p=$n claim=$c"
  CARAMEL_FUSED_CLAIM=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29700+RANDOM%200)) tools/fused_breakdown.py 2>&1 | grep "world"
 done
done
