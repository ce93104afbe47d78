#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/chk_gputest.txt 2>&1; echo "gputest rc=$?"; tail -1 gpurun_out/chk_gputest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/chk_n1.json 2> gpurun_out/chk_n1.err; echo "bench1 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/chk_n1.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'], d['clocks'])"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
   bench.py --gpus 2 --steps 20 --warmup 5 --no-exposed --no-sweep > gpurun_out/chk_n2.json 2> gpurun_out/chk_n2.err; echo "bench2 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/chk_n2.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"
