#!/bin/bash
# 4-GPU session: full GPU suite, 10k-step stress at 2 and 4, bench N=2 (resnet50) and per-model N=4 lines
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/gputest4.txt 2>&1; echo "gputest rc=$?"
tail -2 gpurun_out/gputest4.txt
for n in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n \
   tools/stress.py --steps 10000 --check 1000 > gpurun_out/stress_n$n.jsonl 2> gpurun_out/stress_n$n.err; echo "stress$n rc=$?"
tail -1 gpurun_out/stress_n$n.jsonl
done
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29520 \
   bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench2 rc=$?"
for m in vgg16 alexnet inception_v3; do
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 \
   bench.py --gpus 4 --steps 20 --warmup 5 --model $m --no-sweep > gpurun_out/bench_n4_$m.json 2> gpurun_out/bench_n4_$m.err; echo "bench4 $m rc=$?"
done
echo done
