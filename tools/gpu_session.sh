#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_multigpu.py -q -x -s > gpurun_out/mgpu.txt 2>&1; echo "mgpu rc=$?"
grep -i "nvls\|parity" gpurun_out/mgpu.txt | head
CARAMEL_WATCHDOG_MS=2000 SWEEP_MAX=$((16<<20)) SWEEP_ENGINES=nvls timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29512 tools/sweep.py > gpurun_out/sweep_nvls_only.jsonl 2> gpurun_out/sweep_nvls_only.err
echo "sweep nvls rc=$?"
cat gpurun_out/sweep_nvls_only.jsonl | head -20
CARAMEL_WATCHDOG_MS=2000 SWEEP_MAX=$((16<<20)) SWEEP_ENGINES=single,fused timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29512 tools/sweep.py > gpurun_out/sweep_sf.jsonl 2> gpurun_out/sweep_sf.err
echo "sweep sf rc=$?"
echo done
