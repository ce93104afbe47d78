"""Watchdog and lifetime behaviour on one GPU (rank emulation, cooperative
launch): a flag wait that times out poisons the context and stores nothing;
Aggregator.close() hands the model torch-owned storage back."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def test_timeout_poisons_context_and_stores_nothing():
    """A ring bucket launched at epoch 3 on a fresh context waits for the
    neighbours' epoch-2 'buffer free' flags, which never come: every rank's
    wait times out.  The parameters must be untouched (no epilogue store
    from inputs that never arrived), status()/poll() must raise, and a later,
    well-formed launch must be a no-op (the context stays poisoned)."""
    from paper_2004_14020_b200 import _native as N
    from paper_2004_14020_b200 import comm

    dev = torch.device("cuda:0")
    p, n = 2, 50_000
    ctas, bbytes, _ = N.bucket_layout(n, 1, N.RING, p)
    fbytes = N.flag_bytes_for(1, ctas, N.RING, p)
    foff = (bbytes + 255) // 256 * 256
    ctx = comm.Context(0, p, arena_bytes=foff + fbytes, param_bytes=4 * n, nlocal=p)
    ctx.set_timeout_ms(200)
    theta = torch.randn(n, device=dev)
    for r in range(p):
        ctx.arena_view(r, 0, n, param=True).copy_(theta)
        ctx.arena_view(r, 0, n).normal_()
    b = comm.make_bucket(n, 0, foff, depth=1, pattern=N.RING, epilogue=N.EPI_SGD, flags=N.F_PARAM_ARENA,
                         ctas=ctas, lr=0.5, scale=0.5)
    stream = torch.cuda.current_stream().cuda_stream
    ctx.allreduce(b, 3, stream)
    torch.cuda.synchronize()
    with pytest.raises(N.CaramelError, match="poisoned"):
        ctx.poll()
    with pytest.raises(N.CaramelError, match="watchdog"):
        ctx.status()
    for r in range(p):
        assert torch.equal(ctx.arena_view(r, 0, n, param=True), theta), f"rank {r} parameters were written"
    # a valid launch on the poisoned context exits at entry
    b2 = comm.make_bucket(n, 0, foff, depth=1, pattern=N.SHUFFLE, epilogue=N.EPI_SGD, flags=N.F_PARAM_ARENA,
                          ctas=ctas, lr=0.5, scale=0.5)
    ctx.allreduce(b2, 1, stream)
    torch.cuda.synchronize()
    for r in range(p):
        assert torch.equal(ctx.arena_view(r, 0, n, param=True), theta)
    with pytest.raises(N.CaramelError):
        ctx.status()
    ctx.close()


def test_timeout_in_list_launch_stores_nothing():
    """Same through a CARAMEL_MANY_FLAGS list (k_collective_many) whose second
    bucket is a ring bucket at an unreachable epoch: buckets before it may
    complete, nothing after the failed wait is stored."""
    import ctypes

    from paper_2004_14020_b200 import _native as N
    from paper_2004_14020_b200 import comm

    dev = torch.device("cuda:0")
    p, n = 4, 4096
    ctas, bbytes, _ = N.bucket_layout(n, 1, N.RING, p)
    fbytes = N.flag_bytes_for(1, ctas, N.RING, p)
    foff = (bbytes + 255) // 256 * 256
    ctx = comm.Context(0, p, arena_bytes=foff + fbytes, param_bytes=4 * n, nlocal=p)
    ctx.set_timeout_ms(200)
    theta = torch.randn(n, device=dev)
    for r in range(p):
        ctx.arena_view(r, 0, n, param=True).copy_(theta)
    b = comm.make_bucket(n, 0, foff, depth=1, pattern=N.RING, epilogue=N.EPI_SGD, flags=N.F_PARAM_ARENA,
                         ctas=ctas, lr=0.5, scale=0.25)
    host = (N.Bucket * 1)(b)
    dl = torch.frombuffer(bytearray(bytes(host)), dtype=torch.uint8).to(dev)
    pre = torch.tensor([0, n], dtype=torch.int64, device=dev)
    spre = torch.tensor([0, 0], dtype=torch.int64, device=dev)
    N.check(N.lib().caramel_allreduce_many(ctx._ctx, host, 1, dl.data_ptr(), pre.data_ptr(), spre.data_ptr(), 0,
                                           N.MANY_FLAGS, 5, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    with pytest.raises(N.CaramelError):
        ctx.status()
    for r in range(p):
        assert torch.equal(ctx.arena_view(r, 0, n, param=True), theta)
    ctx.close()


def test_close_returns_torch_owned_storage():
    """After close() the model's parameters and gradients no longer point into
    the (freed) arenas: values kept, state_dict() and a forward work."""
    from paper_2004_14020_b200 import gradsets
    from paper_2004_14020_b200.collective import Pattern, ReduceModel
    from paper_2004_14020_b200.costmodel import NetworkModel
    from paper_2004_14020_b200.executor import Aggregator, lower
    from paper_2004_14020_b200.pipeline import run_pipeline
    from paper_2004_14020_b200.sim import SimConfig

    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(33, 65), torch.nn.ReLU(), torch.nn.Linear(65, 7)).cuda()
    tensors = tuple(gradsets.Tensor(n, tuple(q.shape)) for n, q in model.named_parameters())
    art = run_pipeline(gradsets.layered_chain_dag(tensors),
                       SimConfig(workers=2, network=NetworkModel(10.0, 1e-4), reduce=ReduceModel(400.0, 10.0)))
    ids = [gradsets.param_id(i, len(tensors)) for i in range(len(tensors))]
    plan = lower(art, {pid: t.numel for pid, t in zip(ids, tensors)}, 1, Pattern.SHUFFLE)
    for grads in ("bucket", "flat"):
        agg = Aggregator(plan, dict(zip(ids, model.parameters())), lr=0.1, epilogue="sgd", grads=grads)
        arena = agg.ctx.arena_ptrs(0)
        x = torch.randn(8, 33, device="cuda")
        model(x).square().mean().backward()
        agg.step()
        torch.cuda.synchronize()
        before = [q.detach().clone() for q in model.parameters()]
        gbefore = [q.grad.detach().clone() for q in model.parameters()]
        agg.close()
        spans = [(arena[0], arena[0] + plan.arena_bytes), (arena[1], arena[1] + plan.param_bytes)]
        for q, b, g in zip(model.parameters(), before, gbefore):
            assert torch.equal(q, b) and torch.equal(q.grad, g)
            for t in (q, q.grad):
                assert not any(a <= t.data_ptr() < e for a, e in spans), "tensor still points into an arena"
        sd = {k: v.clone() for k, v in model.state_dict().items()}
        assert all(np.isfinite(v.cpu().numpy()).all() for v in sd.values())
        model(x).sum().item()
        model.zero_grad(set_to_none=True)


def test_push_engine_parity_in_its_own_process():
    """The TMA push engine (one-shot / two-shot push, CARAMEL_PUSH=1) over
    single buckets, synthetic lists and full ResNet-50 / Inception-v3 plans,
    FLAGS and FUSED lists, emulated p = 2..8: bit-exact, no watchdog."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    here = Path(__file__).resolve().parent
    r = subprocess.run([sys.executable, str(here / "_push_engine_check.py")], capture_output=True, text=True,
                       timeout=900, env={**os.environ, "CARAMEL_PUSH": "1", "CARAMEL_FUSED_PUSH": "64"})
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "MISMATCH" not in out and "TIMEOUT" not in out, out[-4000:]
    assert out.count(": ok") >= 40, out[-4000:]
