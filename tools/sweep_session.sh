#!/bin/bash
# config-5 sweeps at p=2 and p=4 (adaptive vs fixed depth), no exposed-comm runs
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for n in 2 4; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29800+n)) \
   bench.py --gpus $n --steps 20 --warmup 5 --no-cpu-baseline --no-exposed --no-zero-copy > gpurun_out/sw_n$n.json 2> gpurun_out/sw_n$n.err; echo "n$n rc=$?"
python - $n <<'PY'
import json, sys
d=json.loads(open(f"gpurun_out/sw_n{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("step", d["ms_per_step"], d["roofline"]["frac"])
for r in d.get("bucket_sweep", []):
    f = r.get("fixed_depth_us") or {}
    best = min(f.values()) if f else None
    print(r["bytes"], r["depth"], r["caramel_us"], f, "adaptive/best %.3f" % (r["caramel_us"] / best) if best else "", r.get("gated_us"), r["nccl_us"])
PY
done
