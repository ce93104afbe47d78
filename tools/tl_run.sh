set -x
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/tk.txt 2>&1
CARAMEL_FUSED_CLAIM=2 timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/tk2.txt 2>&1
for c in 0 1 2 4; do
CARAMEL_FUSED_CLAIM=$c CUDA_VISIBLE_DEVICES=0,1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 tools/fused_breakdown.py > gpurun_out/fb2_c$c.txt 2>&1
CARAMEL_FUSED_CLAIM=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 tools/fused_breakdown.py > gpurun_out/fb4_c$c.txt 2>&1
done
echo done
