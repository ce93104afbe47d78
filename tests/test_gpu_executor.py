"""Executor on one GPU: plan -> lowering -> Aggregator, both the one-launch
pass (step, also captured in a CUDA graph) and the overlapped mode (gradient
hooks launching buckets in the enforced order during backward)."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _tiny_model(seed=0):
    torch.manual_seed(seed)
    return torch.nn.Sequential(torch.nn.Linear(37, 64), torch.nn.ReLU(), torch.nn.Linear(64, 129),
                               torch.nn.ReLU(), torch.nn.Linear(129, 10)).cuda()


def _plan_for(model, world=1, max_ctas=None):
    from paper_2004_14020_b200 import gradsets
    from paper_2004_14020_b200.collective import Pattern, ReduceModel
    from paper_2004_14020_b200.costmodel import NetworkModel
    from paper_2004_14020_b200.executor import lower
    from paper_2004_14020_b200.pipeline import run_pipeline
    from paper_2004_14020_b200.sim import SimConfig

    tensors = tuple(gradsets.Tensor(n, tuple(p.shape)) for n, p in model.named_parameters())
    dag = gradsets.layered_chain_dag(tensors)
    art = run_pipeline(dag, SimConfig(workers=max(2, world), network=NetworkModel(10.0, 1e-4),
                                      reduce=ReduceModel(400.0, 10.0)))
    ids = [gradsets.param_id(i, len(tensors)) for i in range(len(tensors))]
    plan = lower(art, {pid: t.numel for pid, t in zip(ids, tensors)}, world, Pattern.SHUFFLE, max_ctas=max_ctas)
    return plan, dict(zip(ids, model.parameters()))


def test_hooks_overlapped_update_matches_sgd():
    from paper_2004_14020_b200.executor import Aggregator

    lr = 0.05
    model = _tiny_model()
    ref = _tiny_model()
    plan, params = _plan_for(model)
    assert len(plan.buckets) >= 2
    agg = Aggregator(plan, params, lr=lr, epilogue="sgd")
    agg.attach_hooks()
    x = torch.randn(16, 37, device="cuda")
    for it in range(3):
        # reference: plain backward + theta - lr * g (separate roundings)
        ref.zero_grad(set_to_none=False)
        ref(x * (it + 1)).square().mean().backward()
        with torch.no_grad():
            for p in ref.parameters():
                p.copy_(p - lr * p.grad)
        model.zero_grad(set_to_none=False)
        agg.begin_iteration()
        model(x * (it + 1)).square().mean().backward()
        agg.finish_iteration()
        torch.cuda.synchronize()
        agg.status()
        for (n, a), b in zip(model.named_parameters(), ref.parameters()):
            assert torch.equal(a, b), f"iteration {it}: {n} differs"
    agg.close()


def test_step_and_graph_replay_match_sgd():
    from paper_2004_14020_b200.executor import Aggregator

    lr = 0.1
    model = _tiny_model(1)
    plan, params = _plan_for(model)
    agg = Aggregator(plan, params, lr=lr, epilogue="sgd")
    for p in params.values():
        p.grad.normal_()
    theta0 = {k: v.detach().clone() for k, v in params.items()}
    agg.step()
    torch.cuda.synchronize()
    for k, p in params.items():
        assert torch.equal(p, theta0[k] - lr * p.grad)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        agg.step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    theta1 = {k: v.detach().clone() for k, v in params.items()}  # capture does not execute
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    for k, p in params.items():
        assert torch.equal(p, (theta1[k] - lr * p.grad) - lr * p.grad)
    agg.close()


def test_gradient_mean_mode_writes_back_grads():
    from paper_2004_14020_b200.executor import Aggregator

    model = _tiny_model(2)
    plan, params = _plan_for(model)
    agg = Aggregator(plan, params, epilogue="mean")
    for p in params.values():
        p.grad.normal_()
    want = {k: p.grad.clone() for k, p in params.items()}  # world = 1: mean == identity
    agg.step(fused=False)
    torch.cuda.synchronize()
    for k, p in params.items():
        assert torch.equal(p.grad, want[k])
    agg.close()


def test_step_host_pipelined_matches_sgd():
    from paper_2004_14020_b200.executor import Aggregator

    lr = 0.1
    model = _tiny_model(3)
    plan, params = _plan_for(model)
    agg = Aggregator(plan, params, lr=lr, epilogue="sgd")
    theta0 = {k: v.detach().cpu().clone() for k, v in params.items()}
    host_g = {k: torch.randn(v.numel()).pin_memory() for k, v in params.items()}
    host_p = {k: torch.empty(v.numel()).pin_memory() for k, v in params.items()}
    n = agg.step_host(host_g, host_p, group_bytes=4096)  # several groups, one launch each
    torch.cuda.synchronize()
    assert n >= 2
    for k in params:
        want = theta0[k].view(-1) - lr * host_g[k]
        assert torch.equal(host_p[k], want), k
        assert torch.equal(params[k].detach().cpu().view(-1), want)
    agg.close()


@pytest.mark.parametrize("grads", ["bucket", "flat"])
def test_step_host_flat_matches_sgd(grads):
    from paper_2004_14020_b200.executor import Aggregator

    lr = 0.1
    model = _tiny_model(4)
    plan, params = _plan_for(model)
    agg = Aggregator(plan, params, lr=lr, epilogue="sgd", grads=grads)
    theta0 = {k: v.detach().cpu().clone().view(-1) for k, v in params.items()}
    hg = torch.zeros(plan.param_bytes // 4).pin_memory()
    hp = torch.zeros(plan.param_bytes // 4).pin_memory()
    layout = agg.flat_layout()
    for pid, off, n in layout:
        hg[off:off + n].normal_()
    agg.step_host_flat(hg, hp, group_bytes=4096)
    torch.cuda.synchronize()
    for pid, off, n in layout:
        assert torch.equal(hp[off:off + n], theta0[pid] - lr * hg[off:off + n]), pid
    agg.close()


def test_tables_track_gradient_storage():
    from paper_2004_14020_b200.executor import Aggregator

    model = _tiny_model(5)
    plan, params = _plan_for(model)
    agg = Aggregator(plan, params, lr=0.1, epilogue="sgd")
    assert agg.check_tables()
    # coalesced: with the flat gradient buffer every bucket is one contiguous piece
    assert all(lv.desc.nseg == 1 for lv in agg._live)
    next(iter(params.values())).grad = torch.zeros_like(next(iter(params.values())))
    assert not agg.check_tables()
    agg.refresh_tables()
    assert agg.check_tables()
    agg.close()


@pytest.mark.parametrize("grads", ["bucket", "flat", "own"])
def test_gradient_storage_modes_match_sgd(grads):
    from paper_2004_14020_b200.executor import Aggregator

    lr = 0.05
    model = _tiny_model(6)
    ref = _tiny_model(6)
    plan, params = _plan_for(model)
    agg = Aggregator(plan, params, lr=lr, epilogue="sgd", grads=grads)
    agg.attach_hooks()
    x = torch.randn(16, 37, device="cuda")
    for it in range(2):
        ref.zero_grad(set_to_none=False)
        ref(x * (it + 1)).square().mean().backward()
        with torch.no_grad():
            for p in ref.parameters():
                p.copy_(p - lr * p.grad)
        model.zero_grad(set_to_none=False)
        agg.begin_iteration()
        model(x * (it + 1)).square().mean().backward()
        agg.finish_iteration()
        torch.cuda.synchronize()
        for a, b in zip(model.parameters(), ref.parameters()):
            assert torch.equal(a, b)
    # the one-launch pass too
    for p in params.values():
        p.grad.normal_()
    theta0 = {k: v.detach().clone() for k, v in params.items()}
    agg.step()
    torch.cuda.synchronize()
    for k, p in params.items():
        assert torch.equal(p, theta0[k] - lr * p.grad)
    agg.close()


def test_postponed_update_gated_by_next_forward():
    """Buckets placed into the next forward (FP_OVERLAP) are not waited for at
    the end of backward but by the forward gate of the module that reads them;
    every iteration's loss and the final parameters must equal plain SGD."""
    import dataclasses

    from paper_2004_14020_b200.executor import Aggregator, ExecPlan

    lr = 0.05
    model = _tiny_model(7)
    ref = _tiny_model(7)
    plan, params = _plan_for(model)
    # postpone the buckets launched last (first layers' parameters: read first
    # in the next forward) -- the hardest case for the gate
    n = len(plan.buckets)
    bks = tuple(dataclasses.replace(b, placement="fp_overlap") if b.index >= n - 2 else b for b in plan.buckets)
    plan = dataclasses.replace(plan, buckets=bks)
    owner = {}
    for m in model.modules():
        for p in m.parameters(recurse=False):
            owner[id(p)] = m
    agg = Aggregator(plan, params, lr=lr, epilogue="sgd")
    agg.attach_hooks()
    assert agg.gate_forward({pid: owner[id(p)] for pid, p in params.items()}) >= 1
    x = torch.randn(16, 37, device="cuda")
    for it in range(4):
        ref.zero_grad(set_to_none=False)
        lr_ = ref(x * (it + 1)).square().mean()
        lr_.backward()
        with torch.no_grad():
            for p in ref.parameters():
                p.copy_(p - lr * p.grad)
        agg.zero_grad()
        agg.begin_iteration()
        lm = model(x * (it + 1)).square().mean()
        lm.backward()
        agg.finish_iteration(postpone=True)
        assert torch.equal(lm.detach(), lr_.detach()), f"iteration {it}: forward saw stale parameters"
    agg.sync()
    torch.cuda.synchronize()
    for a, b in zip(model.parameters(), ref.parameters()):
        assert torch.equal(a, b)
    agg.close()


def test_ingest_model_dag_and_plan():
    from paper_2004_14020_b200.dag import validate_dag
    from paper_2004_14020_b200.ingest import ingest_model

    model = _tiny_model(8)
    x = torch.randn(64, 37, device="cuda")

    def step():
        model.zero_grad(set_to_none=False)
        model(x).square().mean().backward()

    ing = ingest_model(model, step, runs=3, example_inputs=(x,))
    rep = validate_dag(ing.dag)
    assert rep.ok, rep.errors
    assert len(ing.dag.params) == len(list(model.parameters()))
    assert all(op.duration_us >= 1 for op in ing.dag.ops.values() if op.kind.value == "compute")
    from paper_2004_14020_b200.collective import ReduceModel
    from paper_2004_14020_b200.costmodel import NetworkModel
    from paper_2004_14020_b200.pipeline import run_pipeline
    from paper_2004_14020_b200.sim import SimConfig

    art = run_pipeline(ing.dag, SimConfig(workers=2, network=NetworkModel(10.0, 1e-5), reduce=ReduceModel(5e6, 0.5)))
    assert sum(len(g.param_ids) for g in art.batch_plan.groups) == len(ing.dag.params)


@pytest.mark.parametrize("case", ["resnet50_p4_nvlink", "vgg16_p2_nvlink"])
def test_persisted_reference_plan_drives_the_executor(case):
    """The reference CLI's own optimize output (tests/golden/optimize) lowered
    by planio and executed: one fused pass over the full gradient set, every
    parameter bit-exact with theta - lr * (g * 1) (world = 1 layout)."""
    import json
    from pathlib import Path

    from paper_2004_14020_b200 import gradsets, planio
    from paper_2004_14020_b200.executor import Aggregator

    d = Path(__file__).resolve().parent / "golden" / "optimize" / case
    meta = json.loads((d / "case.json").read_text())
    tensors = gradsets.gradient_set(meta["model"])
    ids = [gradsets.param_id(i, len(tensors)) for i in range(len(tensors))]
    numels = {pid: t.numel for pid, t in zip(ids, tensors)}
    plan = planio.load_exec_plan(d, numels, 1, meta["pattern"], depth=meta["depth"])
    assert [b.group_id for b in plan.buckets] == \
        [t["group_id"] for t in json.loads((d / "transfer_schedule.json").read_text())["transfers"]]
    g = torch.Generator(device="cuda").manual_seed(3)
    params = {pid: (torch.randn(t.shape, device="cuda", generator=g) * 0.01) for pid, t in zip(ids, tensors)}
    lr = 0.1
    agg = Aggregator(plan, params, lr=lr, epilogue="sgd")
    for p in params.values():
        p.grad.normal_(generator=g)
    theta0 = {k: v.detach().clone() for k, v in params.items()}
    agg.step()
    torch.cuda.synchronize()
    agg.status()
    for k, p in params.items():
        want = (theta0[k].cpu().numpy() - np.float32(lr) * p.grad.cpu().numpy()).astype(np.float32)
        assert np.array_equal(p.detach().cpu().numpy().view(np.uint32), want.view(np.uint32)), k
    agg.close()


def test_captured_host_step_replays_full_steps():
    """capture_step_host_flat: every replay is a whole step -- new host
    gradients in, SGD applied, parameters out -- bit-exact, twice in a row."""
    from paper_2004_14020_b200.executor import Aggregator

    lr = 0.1
    model = _tiny_model(5)
    plan, params = _plan_for(model)
    agg = Aggregator(plan, params, lr=lr, epilogue="sgd", grads="flat")
    hg = torch.zeros(plan.param_bytes // 4).pin_memory()
    hp = torch.zeros(plan.param_bytes // 4).pin_memory()
    layout = agg.flat_layout()
    theta = {pid: params[pid].detach().cpu().clone().view(-1) for pid, _, _ in layout}
    for pid, off, n in layout:
        hg[off:off + n].normal_()
    g = agg.capture_step_host_flat(hg, hp, group_bytes=4096)  # runs one eager step first
    torch.cuda.synchronize()
    for pid, off, n in layout:
        theta[pid] = theta[pid] - lr * hg[off:off + n]
    for _ in range(2):
        for pid, off, n in layout:
            hg[off:off + n].normal_()
        g.replay()
        torch.cuda.synchronize()
        for pid, off, n in layout:
            theta[pid] = theta[pid] - lr * hg[off:off + n]
            assert torch.equal(hp[off:off + n], theta[pid]), pid
    agg.close()
