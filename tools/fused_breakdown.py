"""N>1 fused step breakdown: full step vs the same launch without the pack
phase (buckets taken as already packed) vs an empty list cost (barriers)."""
import ctypes, os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch, torch.distributed as dist
import bench
from paper_2004_14020_b200 import gradsets, _native as N
from paper_2004_14020_b200.executor import Aggregator

rank, world, local = bench.env_rank()
torch.cuda.set_device(local); dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
tensors, art, plan, _ = bench.build_plan("resnet50", world, "shuffle")
ids = [gradsets.param_id(i, len(tensors)) for i in range(len(tensors))]
params = {pid: torch.randn(t.shape, device=dev) * 0.01 for pid, t in zip(ids, tensors)}
agg = Aggregator(plan, params, rank=rank, lr=0.1)
for p in params.values(): p.grad.normal_()

def timed(fn, iters=30):
    for _ in range(5): fn()
    torch.cuda.synchronize(); dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); e.synchronize()
    t = torch.tensor([s.elapsed_time(e) / iters * 1e3], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()

full = timed(lambda: agg.step())
# same list without the pack phase
nopack = (N.Bucket * len(agg._live))(*[lv.desc for lv in agg._live])
for b in nopack: b.flags &= ~N.F_PACK
dl = torch.frombuffer(bytearray(bytes(nopack)), dtype=torch.uint8).to(dev)
s = torch.cuda.current_stream().cuda_stream
def step_nopack():
    N.check(N.lib().caramel_allreduce_many(agg.ctx._ctx, nopack, len(agg._live), dl.data_ptr(),
            agg._dev_prefix.data_ptr(), agg._dev_segprefix.data_ptr(), 0, N.MANY_FUSED, 0, ctypes.c_void_p(s)))
np_us = timed(step_nopack)
# one tiny bucket: barrier + launch overhead
one = (N.Bucket * 1)(agg._live[0].desc)
one[0].flags &= ~N.F_PACK
d1 = torch.frombuffer(bytearray(bytes(one)), dtype=torch.uint8).to(dev)
def step_one():
    N.check(N.lib().caramel_allreduce_many(agg.ctx._ctx, one, 1, d1.data_ptr(), agg._dev_prefix.data_ptr(),
            agg._dev_segprefix.data_ptr(), 0, N.MANY_FUSED, 0, ctypes.c_void_p(s)))
one_us = timed(step_one)
if rank == 0:
    print(f"world {world}: full step {full:.1f} us, without pack {np_us:.1f} us, single tiny bucket {one_us:.1f} us; "
          f"bus bytes {plan.bus_bytes()/1e6:.1f} MB -> {plan.bus_bytes()/(np_us*1e-6)/1e9:.0f} GB/s w/o pack")
agg.close(); dist.destroy_process_group()
