set -x
export PYTHONUNBUFFERED=1
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611"
ITERS=60 MODEL=vgg16 BATCH=32 ENGINE=ce $T tools/exposed_timeline.py > gpurun_out/tl4_vgg_ce.txt 2>&1
ITERS=60 MODEL=vgg16 BATCH=32 ENGINE=sm $T tools/exposed_timeline.py > gpurun_out/tl4_vgg_sm.txt 2>&1
echo done
