#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_baseline_sizes.py -m gpu -q -x > gpurun_out/gputest.txt 2>&1; echo "gputest rc=$?"
tail -1 gpurun_out/gputest.txt
for mc in 64 128; do
CARAMEL_MAX_CTAS=$mc SWEEP_MAX=$((1<<30)) SWEEP_ENGINES=single,fused SWEEP_DEPTHS=1,8 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 2951${mc:0:1} tools/sweep.py > gpurun_out/sweep_u4_mc$mc.jsonl 2> gpurun_out/sweep_u4_mc$mc.err
echo "sweep $mc rc=$?"
done
echo done
