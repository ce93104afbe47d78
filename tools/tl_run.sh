set -x
export PYTHONUNBUFFERED=1
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-exposed > gpurun_out/b1.json 2> gpurun_out/b1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --no-exposed --no-sweep > gpurun_out/b2.json 2> gpurun_out/b2.err
echo done
