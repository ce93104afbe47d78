"""The N > 1 host logic on the CPU: two processes, torch.distributed over gloo
(world_size 2).  Every rank plans and lowers independently; the plans must be
rank-invariant (identical digests), and the agreement check that guards the
flag protocols must pass on identical plans and raise DeadlockDetected on both
ranks when one rank plans from a different network model or engine knobs."""

from __future__ import annotations

import os
import socket
import sys
import traceback
from pathlib import Path

import pytest

torch = pytest.importorskip("torch")

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _plan(model: str, world: int, net):
    from paper_2004_14020_b200 import gradsets
    from paper_2004_14020_b200.collective import Pattern, ReduceModel
    from paper_2004_14020_b200.costmodel import NetworkModel
    from paper_2004_14020_b200.executor import lower
    from paper_2004_14020_b200.pipeline import run_pipeline
    from paper_2004_14020_b200.sim import SimConfig

    tensors = gradsets.gradient_set(model)
    art = run_pipeline(gradsets.layered_chain_dag(model),
                       SimConfig(workers=world, network=NetworkModel(*net), reduce=ReduceModel(400.0, 10.0)))
    return lower(art, {gradsets.param_id(i, len(tensors)): t.numel for i, t in enumerate(tensors)}, world,
                 Pattern.SHUFFLE)


def _worker(rank: int, world: int, port: int, outq) -> None:
    try:
        sys.path.insert(0, str(ROOT))
        import torch.distributed as dist

        from paper_2004_14020_b200.executor import agree
        from paper_2004_14020_b200.sim import DeadlockDetected

        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        res = {}
        # 1. identical inputs -> identical plans on every rank, agreement passes
        plan = _plan("resnet50", world, (10.0, 1.0 / 460e3))
        digests: list = [None] * world
        dist.all_gather_object(digests, plan.digest())
        res["rank_invariant"] = len(set(digests)) == 1
        agree("execution plan", plan.digest(), world)
        res["agree_ok"] = True
        # 2. rank 1 plans with another network model -> both ranks raise
        net = (10.0, 1.0 / 460e3) if rank == 0 else (12.0, 1.0 / 400e3)
        other = _plan("resnet50", world, net)
        try:
            agree("execution plan", other.digest(), world)
            res["mismatch_raised"] = False
        except DeadlockDetected as exc:
            res["mismatch_raised"] = "ranks [1]" in str(exc)
        # 3. same plan, different engine knobs (e.g. ce_min_bytes) -> both ranks raise
        knobs = '{"engine": "ce", "ce_min_bytes": %d}' % (0 if rank == 0 else 4096)
        try:
            agree("engine of some bucket", knobs, world)
            res["knob_mismatch_raised"] = False
        except DeadlockDetected:
            res["knob_mismatch_raised"] = True
        dist.barrier()
        dist.destroy_process_group()
        outq.put((rank, res))
    except Exception:  # pragma: no cover - surfaced by the parent
        outq.put((rank, {"error": traceback.format_exc()}))


def test_two_process_plan_agreement_over_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert "error" not in results[r], results[r].get("error")
        assert results[r] == {"rank_invariant": True, "agree_ok": True, "mismatch_raised": True,
                              "knob_mismatch_raised": True}, results[r]
