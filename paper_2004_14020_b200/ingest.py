"""DAG ingestion from a PyTorch model.

Builds the planner's DataflowDag (dag.py; JSON wire format dag.py:267-365)
from a real model instead of the synthetic layered chain:

* ops are the model's parameterised leaf modules in the order their forward
  pass actually runs (forward hooks), each with a forward compute op f{k} and a
  backward compute op b{k} (backward visits them in reverse);
* every parameter gets a read marker feeding the forward op of its module and
  an update marker fed by that module's backward op (a module's weight and bias
  become ready together -- their gradients come from the same backward node);
* durations are measured on the device: CUDA events at the boundaries of every
  module's forward and backward, over several runs, each op's duration the
  minimum across runs (estimate_op_times, costmodel.py:74-81);
  the time between two parameterised modules (activations, pooling, residual
  adds) is charged to the later one, so the ops partition the iteration;
  backward boundaries are the moments a module's parameter gradients are
  accumulated (post-accumulate-grad hooks), i.e. the update times the batcher
  works from.

Parameter ids are gradsets.param_id(i) over named_parameters() order, the ids
the gradient inventories and the executor use.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .costmodel import OpProfile, estimate_op_times
from .dag import DataflowDag, Op, OpKind, Parameter, Phase
from .gradsets import param_id


@dataclass
class IngestedModel:
    dag: DataflowDag
    params: dict[str, torch.nn.Parameter]       # param id -> parameter
    modules: dict[str, torch.nn.Module]          # param id -> owning module
    forward_us: dict[str, int]                   # op id -> duration
    runs: int


def _param_modules(model: torch.nn.Module):
    owner = {}
    for mod in model.modules():
        for p in mod.parameters(recurse=False):
            owner[id(p)] = mod
    return owner


def ingest_model(model: torch.nn.Module, step_fn, runs: int = 5) -> IngestedModel:
    """Run `step_fn()` (one forward + backward of `model`) `runs` times with
    timing hooks and return the measured iteration DAG."""
    named = list(model.named_parameters())
    n = len(named)
    pids = {id(p): param_id(i, n) for i, (_, p) in enumerate(named)}
    owner = _param_modules(model)
    mods = []
    for _, p in named:
        m = owner[id(p)]
        if all(m is not x for x in mods):
            mods.append(m)
    fwd_events: list[list] = []
    bwd_events: list[list] = []
    order: list = []   # modules in forward execution order (first run)
    handles = []

    def f_hook(m, *_):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        fwd_events[-1].append((m, ev))

    # backward boundaries: the moment each module's parameter gradients are
    # accumulated (post-accumulate-grad hooks; module backward hooks would wrap
    # outputs and break in-place activations)
    def make_b_hook(m):
        def b_hook(_p):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            bwd_events[-1].append((m, ev))
        return b_hook

    for m in mods:
        handles.append(m.register_forward_hook(f_hook))
        for p in m.parameters(recurse=False):
            handles.append(p.register_post_accumulate_grad_hook(make_b_hook(m)))
    samples: dict[str, list[int]] = {}
    try:
        for r in range(runs + 1):  # the first run warms up
            fwd_events.append([])
            bwd_events.append([])
            start = torch.cuda.Event(enable_timing=True)
            start.record()
            step_fn()
            torch.cuda.synchronize()
            if r == 0:
                seen = []
                for m, _ in fwd_events[-1]:
                    if all(m is not x for x in seen):
                        seen.append(m)
                order = seen
                continue
            # forward: boundary-to-boundary times in execution order
            prev = start
            t_f = {}
            for m, ev in fwd_events[-1]:
                t_f[id(m)] = t_f.get(id(m), 0.0) + prev.elapsed_time(ev)
                prev = ev
            # backward: a module's boundary is its last parameter's accumulation
            last = {}
            for m, ev in bwd_events[-1]:
                last[id(m)] = ev
            seq = sorted(last.items(), key=lambda kv: prev.elapsed_time(kv[1]))
            t_b = {}
            for mid, ev in seq:
                t_b[mid] = max(0.0, prev.elapsed_time(ev))
                prev = ev
            for k, m in enumerate(order):
                for kind, t in (("f", t_f), ("b", t_b)):
                    us = max(1, int(round(1000.0 * t.get(id(m), 0.0))))
                    samples.setdefault(f"{kind}{k:04d}", []).append(us)
    finally:
        for h in handles:
            h.remove()
    dur = estimate_op_times([OpProfile(op, tuple(v)) for op, v in sorted(samples.items())])
    K = len(order)
    ops: dict[str, Op] = {}
    params: dict[str, Parameter] = {}
    param_map: dict[str, torch.nn.Parameter] = {}
    module_map: dict[str, torch.nn.Module] = {}
    for k, m in enumerate(order):
        fid, bid = f"f{k:04d}", f"b{K - 1 - k:04d}"
        reads = []
        for p in m.parameters(recurse=False):
            pid = pids[id(p)]
            params[pid] = Parameter(pid, 4 * p.numel())
            param_map[pid] = p
            module_map[pid] = m
            rid = f"r_{pid}"
            ops[rid] = Op(rid, OpKind.PARAM_READ, 0, frozenset(), Phase.FORWARD, pid)
            reads.append(rid)
            uid = f"u_{pid}"
            ops[uid] = Op(uid, OpKind.PARAM_UPDATE, 0, frozenset({bid}), Phase.BACKPROP, pid)
        deps = set(reads) | ({f"f{k - 1:04d}"} if k else set())
        ops[fid] = Op(fid, OpKind.COMPUTE, dur.get(f"f{k:04d}", 1), frozenset(deps), Phase.FORWARD)
        # backward op of module k runs after the backward of module k+1
        bdeps = {f"b{K - 2 - k:04d}"} if k < K - 1 else {f"f{K - 1:04d}"}
        ops[bid] = Op(bid, OpKind.COMPUTE, dur.get(f"b{k:04d}", 1), frozenset(bdeps), Phase.BACKPROP)
    missing = [pid for pid in pids.values() if pid not in params]
    if missing:
        raise RuntimeError(f"parameters whose module never ran forward: {missing[:5]}")
    return IngestedModel(dag=DataflowDag(ops=ops, params=params), params=param_map, modules=module_map,
                         forward_us=dur, runs=runs)
