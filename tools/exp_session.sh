#!/bin/bash
# A/B session: K1/K4 tile/occupancy variant and fused-step V at p=2 (CARAMEL_LIB swaps the library)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
DEF=paper_2004_14020_b200/csrc/libcaramel_b200.so
for rep in 1 2; do
 for L in $DEF tools/lib_kt2.so; do
  echo "pack lib=$L rep=$rep"
  CARAMEL_LIB=$L timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch, bench
from paper_2004_14020_b200 import gradsets
r = bench.pack_unpack_bw(torch, gradsets.gradient_set('resnet50'), torch.device('cuda',0), 6524.0, reps=50)
print({k: r[k] for k in ('pack_ms','pack_frac','unpack_ms','unpack_frac','round_trip_exact')})
" 2>&1 | tail -1
 done
done
for rep in 1 2; do
 for L in $DEF tools/lib_v6.so tools/lib_v8.so; do
  echo "fused2 lib=$L rep=$rep"
  CARAMEL_LIB=$L timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600+RANDOM%300)) tools/fused_breakdown.py 2>&1 | grep -v Warn | tail -3
 done
done
echo done
