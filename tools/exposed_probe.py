"""Timeline of the overlapped (hooks) aggregation during a real backward:
per-bucket start/end on the comm stream relative to the end of backward."""
import os, sys, json
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch, torch.distributed as dist, torchvision
import bench
from paper_2004_14020_b200 import gradsets, _native as N
from paper_2004_14020_b200.executor import Aggregator

rank, world, local = bench.env_rank()
torch.cuda.set_device(local); dev = torch.device("cuda", local)
if world > 1: dist.init_process_group("nccl", device_id=dev)
model_name = os.environ.get("MODEL", "resnet50")
tensors, art, plan, _ = bench.build_plan(model_name, world, "shuffle")
ids = [gradsets.param_id(i, len(tensors)) for i in range(len(tensors))]
torch.manual_seed(7)
model = getattr(torchvision.models, model_name)().to(dev)
for p in model.parameters(): p.grad = torch.zeros_like(p)
x = torch.randn(64, 3, 224, 224, device=dev); y = torch.randint(0, 1000, (64,), device=dev)
agg = Aggregator(plan, dict(zip(ids, model.parameters())), rank=rank, lr=0.1)
agg.attach_hooks()
marks = []
orig = agg._launch
def launch(lv, stream):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(agg.comm_stream); orig(lv, stream); b.record(agg.comm_stream)
    marks.append((lv.spec.group_id, lv.spec.numel, lv.spec.ctas, a, b))
agg._launch = launch
def it():
    model.zero_grad(set_to_none=False); agg.begin_iteration()
    s = torch.cuda.Event(enable_timing=True); s.record()
    with torch.autocast("cuda", dtype=torch.bfloat16):
        loss = torch.nn.functional.cross_entropy(model(x).float(), y)
    f = torch.cuda.Event(enable_timing=True); f.record()
    loss.backward()
    e = torch.cuda.Event(enable_timing=True); e.record()
    agg.finish_iteration()
    z = torch.cuda.Event(enable_timing=True); z.record()
    return s, f, e, z
for _ in range(3): it()
marks.clear(); torch.cuda.synchronize()
s, f, e, z = it(); torch.cuda.synchronize()
if rank == 0:
    print(f"fwd {s.elapsed_time(f):.2f} ms  bwd {f.elapsed_time(e):.2f} ms  tail(after bwd) {e.elapsed_time(z):.3f} ms  buckets {len(marks)}")
    busy = sum(a.elapsed_time(b) for _, _, _, a, b in marks)
    print(f"sum of bucket kernel spans {busy:.3f} ms")
    for gid, n, c, a, b in marks[-12:]:
        print(f"{gid} numel={n:>9} ctas={c:>3} start {e.elapsed_time(a):+8.3f} ms end {e.elapsed_time(b):+8.3f} ms  dur {a.elapsed_time(b)*1e3:7.1f} us")
    first = marks[0][3]
    print(f"first bucket starts {f.elapsed_time(first):.3f} ms after backward start")
agg.close()
if world > 1: dist.destroy_process_group()
