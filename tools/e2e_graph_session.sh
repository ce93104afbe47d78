#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_executor.py -x -q > gpurun_out/eg_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/eg_tests.txt
for i in 1 2; do
 for gr in 0 1; do
  CARAMEL_E2E_GRAPH=$gr timeout 900 python bench.py --steps 20 --warmup 5 --no-exposed --no-cpu-baseline > gpurun_out/eg.json 2> gpurun_out/eg_$gr.err; echo "bench rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/eg.json').read().strip().splitlines()[-1]); print('graph=$gr', d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['api'][:40])"
 done
done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 \
   bench.py --gpus 2 --steps 20 --warmup 5 --no-exposed --no-sweep --no-cpu-baseline > gpurun_out/eg2.json 2> gpurun_out/eg2.err; echo "bench2 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/eg2.json').read().strip().splitlines()[-1]); print('n2', d['value'], d['e2e'])"
