"""Timeline of the overlapped aggregation on a real model, with the same
ingested plan bench.py's exposed-communication measurement uses.

  MODEL=alexnet BATCH=64 GRADS=bucket HOOK_CTAS=0 torchrun --nproc-per-node 2 \
      --master-addr 127.0.0.1 tools/exposed_timeline.py

Prints, on rank 0: compute-only forward/backward times, the plan (bucket size,
placement, planned begin/finish), every launch on the comm stream relative to
the start of backward, and the per-iteration time with aggregation."""
import os
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before any CUDA context: one hardware queue per stream
import sys
from pathlib import Path
from types import SimpleNamespace

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torchvision  # noqa: E402

import bench  # noqa: E402
from paper_2004_14020_b200.executor import Aggregator, calibrate_network_model  # noqa: E402

rank, world, local = bench.env_rank()
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
D = dist if world > 1 else None
name = os.environ.get("MODEL", "alexnet")
B = int(os.environ.get("BATCH", "64"))
args = SimpleNamespace(model=name, pattern="shuffle")
torch.manual_seed(7)
model = getattr(torchvision.models, name)().to(dev)
for p in model.parameters():
    p.grad = torch.zeros_like(p)
gen = torch.Generator(device=dev).manual_seed(11 + rank)
x = torch.randn(B, 3, 224, 224, device=dev, generator=gen)
y = torch.randint(0, 1000, (B,), device=dev, generator=gen)


host_bwd = []


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


host_fwd = []


def fwd_bwd(marks):
    marks.append(ev())
    t = time.perf_counter()
    with torch.autocast("cuda", dtype=torch.bfloat16):
        loss = torch.nn.functional.cross_entropy(model(x).float(), y)
    host_fwd.append(time.perf_counter() - t)
    marks.append(ev())
    t = time.perf_counter()
    loss.backward()
    host_bwd.append(time.perf_counter() - t)
    marks.append(ev())


def compute_only():
    model.zero_grad(set_to_none=False)
    fwd_bwd([])


net = calibrate_network_model(world, rank)[0] if world > 1 else None
ing, art, plan, net = bench.ingested_plan(args, model, compute_only, world, D, dev, net, example_inputs=(x,))
if "PRIO" in os.environ:
    Aggregator.comm_priority = int(os.environ["PRIO"])
agg = Aggregator(plan, dict(ing.params), rank=rank, lr=0.01, epilogue="sgd", grads=os.environ.get("GRADS", "bucket"),
                 engine=os.environ.get("ENGINE", "sm"))
gated = agg.gate_forward(ing.modules)
cap = int(os.environ.get("HOOK_CTAS", "0"))
if "CE_MIN" in os.environ:
    agg.ce_min_bytes = int(os.environ["CE_MIN"])
if "TAIL_US" in os.environ:
    agg.ce_tail_us = float(os.environ["TAIL_US"])
    agg.ce_tail_frac = float(os.environ.get("TAIL_FRAC", "0"))
if cap:
    agg.coalesce_ctas = cap
launches = []
orig_one, orig_range = agg._launch, agg._launch_range


def one(lv, stream):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(agg.comm_stream)
    if cap:
        i = agg._live.index(lv)
        orig_range(i, i + 1, stream, 1, max(cap, 1))
    else:
        orig_one(lv, stream)
    b.record(agg.comm_stream)
    launches.append((lv.spec.group_id, 1, 4 * lv.spec.numel, cap or lv.spec.ctas, a, b))


def rng(i, j, stream, mode, ctas):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(agg.comm_stream)
    orig_range(i, j, stream, mode, ctas)
    b.record(agg.comm_stream)
    launches.append((agg._live[i].spec.group_id, j - i, 4 * sum(lv.spec.numel for lv in agg._live[i:j]), ctas, a, b))


if os.environ.get("COMM") == "ce":
    # experiment: move the same NVLink bytes with copy engines instead of SMs
    # (pull (p-1)/p of the bucket from peers twice, as reduce-scatter + all-gather)
    from cuda.bindings import runtime as rt

    maxb = max(4 * b.numel for b in plan.buckets)
    err, buf = rt.cudaMalloc(maxb)
    err, stage = rt.cudaMalloc(maxb)
    err, h = rt.cudaIpcGetMemHandle(buf)
    blobs = [None] * world
    dist.all_gather_object(blobs, bytes(h.reserved))
    peers = {}
    for q in range(world):
        if q != rank:
            hh = rt.cudaIpcMemHandle_t()
            hh.reserved = blobs[q]
            err, peers[q] = rt.cudaIpcOpenMemHandle(hh, rt.cudaIpcMemLazyEnablePeerAccess)
    dist.barrier()

    def ce(nbytes):
        part = nbytes // world
        for _ in range(2):
            for q, ptr in peers.items():
                rt.cudaMemcpyAsync(stage + q * part, ptr + rank * part, part, rt.cudaMemcpyKind.cudaMemcpyDefault,
                                   agg.comm_stream.cuda_stream)

    def one(lv, stream):  # noqa: F811
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(agg.comm_stream)
        ce(4 * lv.spec.numel)
        b.record(agg.comm_stream)
        launches.append((lv.spec.group_id, 1, 4 * lv.spec.numel, 0, a, b))

    def rng(i, j, stream, mode, ctas):  # noqa: F811
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(agg.comm_stream)
        nb = 4 * sum(lv.spec.numel for lv in agg._live[i:j])
        ce(nb)
        b.record(agg.comm_stream)
        launches.append((agg._live[i].spec.group_id, j - i, nb, 0, a, b))
agg._launch, agg._launch_range = one, rng
orig_ce = agg._launch_ce


def ce_timed(i, j, stream, grad_stream=None):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(agg.comm_stream)
    orig_ce(i, j, stream, grad_stream)
    b.record(agg.comm_stream)
    launches.append((agg._live[i].spec.group_id, j - i, 4 * sum(lv.spec.numel for lv in agg._live[i:j]), -1, a, b))


agg._launch_ce = ce_timed
drain_t = []
orig_drain_ce = agg._drain_ce


def drain_ce_timed(j):
    t = time.perf_counter()
    orig_drain_ce(j)
    drain_t.append(time.perf_counter() - t)


agg._drain_ce = drain_ce_timed
hook_t = []
orig_drain = agg._drain


def drain_timed(force=False):
    t = time.perf_counter()
    orig_drain(force)
    hook_t.append(time.perf_counter() - t)


agg._drain = drain_timed
agg.attach_hooks()


def caramel_iter(marks):
    agg.zero_grad()
    agg.begin_iteration()
    fwd_bwd(marks)
    agg.finish_iteration(postpone=True)
    marks.append(ev())


for _ in range(5):
    caramel_iter([])
torch.cuda.synchronize()
K = int(os.environ.get("ITERS", "20"))


def clk(cs):
    sm = sorted(float(l.split(",")[1]) for l in cs.lines if len(l.split(",")) >= 9)
    pw = sorted(float(l.split(",")[3]) for l in cs.lines if len(l.split(",")) >= 9)
    rs = sorted({l.split(",")[4].strip() for l in cs.lines if len(l.split(",")) >= 9})
    return (sm[len(sm) // 2] if sm else None, pw[len(pw) // 2] if pw else None, rs)


with bench.ClockSampler(local) as cs_k:
    s = ev()
    for _ in range(K):
        caramel_iter([])
    e = ev()
    torch.cuda.synchronize()
host_k = sorted(host_bwd[-K:])[K // 2]
host_fk = sorted(host_fwd[-K:])[K // 2]


def fwd_only():
    with torch.no_grad(), torch.autocast("cuda", dtype=torch.bfloat16):
        model(x)


def time_fwd():
    for _ in range(3):
        fwd_only()
    torch.cuda.synchronize()
    a = ev()
    for _ in range(K):
        fwd_only()
    b = ev()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K


caramel_iter([])
torch.cuda.synchronize()
fwd_after = time_fwd()
drain_per_it = sum(drain_t[-K * 40:]) / K if drain_t else 0.0
hooks_per_it = sum(hook_t) / (K + 5)
launches.clear()
m0, m1 = [], []
caramel_iter(m0)
caramel_iter(m1)
torch.cuda.synchronize()
k_ms = s.elapsed_time(e) / K
agg.detach_hooks()
host_bwd.clear()
host_fwd.clear()
for _ in range(3):
    compute_only()
c = []
fwd_bwd(c)
torch.cuda.synchronize()
with bench.ClockSampler(local) as cs_c:
    s = ev()
    for _ in range(K):
        compute_only()
    e = ev()
    torch.cuda.synchronize()
c_ms = s.elapsed_time(e) / K
fwd_plain = time_fwd()
if rank == 0:
    print(f"clocks (sm MHz, power W, reasons): aggregation {clk(cs_k)}, compute only {clk(cs_c)}")
    print(f"no-grad forward: after aggregation iterations {fwd_after:.3f} ms, after compute-only {fwd_plain:.3f} ms; "
          f"host time in forward: aggregation iterations {1e3 * host_fk:.3f} ms, compute only "
          f"{1e3 * sorted(host_fwd)[len(host_fwd) // 2]:.3f} ms")
    print(f"{name} p={world} batch {B}: compute fwd {c[0].elapsed_time(c[1]):.3f} bwd {c[1].elapsed_time(c[2]):.3f}"
          f" ms; per-iteration compute {c_ms:.3f} caramel {k_ms:.3f} exposed {k_ms - c_ms:.3f} ms; gated {gated}")
    print(f"host time in backward(): with aggregation {1e3 * host_k:.3f} ms, compute only "
          f"{1e3 * sorted(host_bwd)[len(host_bwd) // 2]:.3f} ms; _drain per iteration {1e3 * hooks_per_it:.3f} ms "
          f"(_drain_ce {1e3 * sum(drain_t) / (K + 7):.3f} ms)")
    print(f"network model {net.latency_us:.2f} us + {net.per_byte_us:.3e} us/B;"
          f" modelled exposed {art.transfer_schedule.added_iteration_time_us:.1f} us")
    for b in plan.buckets:
        print(f"  plan {b.group_id:>8} {4 * b.numel / 1e6:9.3f} MB depth {b.depth} ctas {b.ctas:>3} {b.placement}")
    print(f"iteration 1: fwd {m0[0].elapsed_time(m0[1]):.3f} bwd {m0[1].elapsed_time(m0[2]):.3f}"
          f" finish->{m0[2].elapsed_time(m0[3]):.3f}; next fwd {m1[0].elapsed_time(m1[1]):.3f}")
    t0 = m0[1]
    for gid, cnt, nbytes, ctas, a, b in launches:
        print(f"  launch {gid:>8} x{cnt:<2} {nbytes / 1e6:9.3f} MB ctas {ctas:>3}  start {t0.elapsed_time(a):8.3f}"
              f"  end {t0.elapsed_time(b):8.3f} ms (bwd end {t0.elapsed_time(m0[2]):.3f}, next bwd start"
              f" {t0.elapsed_time(m1[1]):.3f})  {nbytes / 1e6 / max(1e-6, a.elapsed_time(b)):8.1f} GB/s")
agg.sync()
agg.close()
if world > 1:
    dist.destroy_process_group()
