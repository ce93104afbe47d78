#!/bin/bash
# Scratch GPU session driven through gpurun during development (rewritten per experiment):
#   /usr/local/graft/bin/gpurun --gpus N -- "bash tools/gpu_session.sh"
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
run_sweep() {  # $1 = tag, $2 = library
  CARAMEL_LIB=$2 SWEEP_MAX=$((1<<30)) SWEEP_ENGINES=single timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29512 tools/sweep.py > gpurun_out/ab_$1.jsonl 2> gpurun_out/ab_$1.err
  echo "sweep $1 rc=$?"
}
for v in NONE NO_EXIT NO_ENTER r01; do run_sweep $v tools/libcaramel_$v.so; done
./tools/mb_nvlink > gpurun_out/mb_nvlink.jsonl 2>&1; echo "mb rc=$?"
echo done
