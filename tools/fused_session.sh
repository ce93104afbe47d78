#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_baseline_sizes.py tests/test_multigpu.py tests/test_gpu_robustness.py -x -q > gpurun_out/fu_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/fu_tests.txt
for n in 2 4; do
 for rep in 1 2; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29800+n+rep)) \
   bench.py --gpus $n --steps 20 --warmup 5 --no-cpu-baseline --no-exposed --no-zero-copy --no-sweep --no-nccl > gpurun_out/fu_n$n.json 2> gpurun_out/fu_n$n.err; echo "n$n rc=$?"
python - $n <<'PY'
import json, sys
d=json.loads(open(f"gpurun_out/fu_n{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("n", sys.argv[1], "step", d["ms_per_step"], d["roofline"]["achieved"], d["roofline"]["frac"])
PY
 done
done
for m in vgg16 alexnet; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29877 \
   bench.py --gpus 4 --steps 20 --warmup 5 --model $m --no-cpu-baseline --no-exposed --no-zero-copy --no-sweep --no-nccl > gpurun_out/fu_$m.json 2> gpurun_out/fu_$m.err; echo "$m rc=$?"
python - $m <<'PY'
import json, sys
d=json.loads(open(f"gpurun_out/fu_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print(sys.argv[1], "n4 step", d["ms_per_step"], d["roofline"]["achieved"], d["roofline"]["frac"])
PY
done
