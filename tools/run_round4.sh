#!/bin/bash
# 4-GPU session: tests, N=1 bench (+ ncu launch list and full capture), N=4 bench.
export CARAMEL_WATCHDOG_MS=3000
NG=$(nvidia-smi -L | wc -l)
timeout 500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 50 --warmup 3 > gpurun_out/b1.json 2> gpurun_out/b1.err; echo "n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $NG --steps 50 --warmup 3 > gpurun_out/b$NG.json 2> gpurun_out/b$NG.err; echo "n$NG rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-exposed --no-zero-copy > gpurun_out/ncu_plain.log 2>&1 && \
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_n1.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-exposed --no-zero-copy > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-exposed --no-zero-copy > gpurun_out/ncu_plain2.log 2>&1 && \
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_local_flat_tma -s 3 -c 1 -o gpurun_out/bench_n1_full python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-exposed --no-zero-copy > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
