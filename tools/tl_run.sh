set -x
export PYTHONUNBUFFERED=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 > gpurun_out/b2.json 2> gpurun_out/b2.err
for m in alexnet vgg16 inception_v3; do
  B=64; [ $m = vgg16 ] && B=32
  timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --model $m --batch $B --no-cpu-baseline --no-sweep > gpurun_out/m_${m}_n2.json 2> gpurun_out/m_${m}_n2.err
done
echo done
