#!/bin/bash
# r02 closing session (4 GPUs): GPU suite, smoke, bench N=1/2/4 + reference arms, PCIe probe
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/final_gputest.txt 2>&1; echo "gputest rc=$?"
tail -2 gpurun_out/final_gputest.txt; grep -E "FAILED|Error" gpurun_out/final_gputest.txt | head
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err; echo "bench1 rc=$?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/final_ref_n1.json 2> gpurun_out/final_ref_n1.err; echo "ref1 rc=$?"
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29520 \
   bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/final_bench_n2.json 2> gpurun_out/final_bench_n2.err; echo "bench2 rc=$?"
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 \
   bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/final_bench_n4.json 2> gpurun_out/final_bench_n4.err; echo "bench4 rc=$?"
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 \
   bench.py --impl reference --gpus 4 --steps 20 --warmup 5 > gpurun_out/final_ref_n4.json 2> gpurun_out/final_ref_n4.err; echo "ref4 rc=$?"
timeout 300 python tools/pcie_probe.py > gpurun_out/pcie_probe.txt 2>&1; echo "pcie rc=$?"; cat gpurun_out/pcie_probe.txt
echo done
