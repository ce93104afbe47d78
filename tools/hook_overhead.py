"""Cost of the gradient hooks alone: per-iteration time of a model's
forward+backward with a no-op post-accumulate-grad hook on every parameter
(and with a hook that records one CUDA event, like the Aggregator's drain)
versus no hooks.  One GPU.

    MODEL=vgg16 BATCH=32 python tools/hook_overhead.py
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import torchvision  # noqa: E402

name = os.environ.get("MODEL", "vgg16")
B = int(os.environ.get("BATCH", "32"))
K = 30
dev = torch.device("cuda", 0)
model = getattr(torchvision.models, name)().to(dev)
for p in model.parameters():
    p.grad = torch.zeros_like(p)
x = torch.randn(B, 3, 224, 224, device=dev)
y = torch.randint(0, 1000, (B,), device=dev)


def it():
    model.zero_grad(set_to_none=False)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        loss = torch.nn.functional.cross_entropy(model(x).float(), y)
    loss.backward()


def timed():
    for _ in range(3):
        it()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K):
        it()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / K


side = torch.cuda.Stream()
res = {}
for mode in ("none", "noop", "event", "none"):
    hs = []
    if mode == "noop":
        hs = [p.register_post_accumulate_grad_hook(lambda _p: None) for p in model.parameters()]
    elif mode == "event":
        def h(_p):
            side.wait_stream(torch.cuda.current_stream())
            e = torch.cuda.Event()
            e.record(side)
        hs = [p.register_post_accumulate_grad_hook(h) for p in model.parameters()]
    res.setdefault(mode, []).append(timed())
    for hh in hs:
        hh.remove()
print(name, {k: [round(v, 3) for v in vs] for k, vs in res.items()})
