#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for probe in 0 1 2; do
CARAMEL_NVLS_PROBE=$probe SWEEP_MAX=$((1<<30)) SWEEP_ENGINES=nvls timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 2951$probe tools/sweep.py > gpurun_out/sweep_nvls_probe$probe.jsonl 2> gpurun_out/sweep_nvls_probe$probe.err
echo "probe $probe rc=$?"
done
echo done
