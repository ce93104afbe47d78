"""Small driver for ncu: the N=1 fused aggregation step (k_local_many) on the
resnet50 plan, a few launches."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch
import bench
torch.cuda.set_device(0)
tensors, art, plan, _ = bench.build_plan(sys.argv[1] if len(sys.argv) > 1 else "resnet50", 1, "shuffle")
from paper_2004_14020_b200.executor import Aggregator
from paper_2004_14020_b200 import gradsets
ids = [gradsets.param_id(i, len(tensors)) for i in range(len(tensors))]
params = {pid: torch.randn(t.shape, device="cuda") * 0.01 for pid, t in zip(ids, tensors)}
agg = Aggregator(plan, params, lr=0.1)
for p in params.values():
    p.grad.normal_()
for _ in range(8):
    agg.step()
torch.cuda.synchronize()
agg.status()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    agg.step()
e.record(); e.synchronize()
print(f"eager step {s.elapsed_time(e)/20*1e3:.1f} us")
agg.close()
