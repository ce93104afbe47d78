"""DAG ingestion from a PyTorch model.

Builds the planner's DataflowDag (dag.py; JSON wire format dag.py:267-365)
from a real model instead of the synthetic layered chain, in two parts.

Structure -- `trace_units`.  A "unit" is a module that owns parameters
directly (a conv, a batch norm, a linear layer).  One forward pass runs under
a TorchDispatchMode that sees every aten op: each tensor carries the set of
units whose outputs flowed into it; an op inside a unit's forward makes its
outputs that unit's and records, as the unit's inputs, the units behind the
tensors it consumed; any other op (relu, add, cat, pooling, views, in-place
updates) passes the union of its inputs' sets on.  The result is the real
branch structure: a ResNet block's convolutions form a chain while its
identity/downsample path joins at the add; Inception's towers run side by
side from one input and meet at the concatenation; the auxiliary classifier
is a second sink.  The trace runs on a meta-device copy of the model (no
memory, no compute), so it is cheap and has no side effects.

Graph -- `build_dag`.  Per unit U (ids follow the forward execution order k):
  * read marker r_<pid> per parameter -> forward op f<k>;
  * f<k> depends on the forward ops of U's input units;
  * backward op b<K-1-k> depends on the backward ops of the units that
    consumed U's output (the gradient arrives from them); a unit nothing
    consumes (a loss input) waits for the forward pass to finish;
  * update marker u_<pid> per parameter fed by b<K-1-k>.
Lexicographic op ids make the planner's priority the execution order
(forward) and its reverse (backward), as in the survey's layered chain.

Durations -- `ingest_model`.  CUDA events at the boundaries of every unit's
forward and at the moment its parameter gradients are accumulated, over
several runs, each op's duration the minimum across runs (estimate_op_times,
costmodel.py:74-81); the time between two units is charged to
the later one, so the ops partition the iteration.

Parameter ids are gradsets.param_id(i) over named_parameters() order, the ids
the gradient inventories and the executor use.
"""

from __future__ import annotations

import copy
from dataclasses import dataclass

import torch
from torch.utils._python_dispatch import TorchDispatchMode
from torch.utils._pytree import tree_leaves

from .costmodel import OpProfile, estimate_op_times
from .dag import DataflowDag, Op, OpKind, Parameter, Phase
from .gradsets import param_id


@dataclass(frozen=True)
class UnitGraph:
    """Parameter-owning modules in forward execution order and their dataflow."""

    names: tuple[str, ...]                          # qualified module names, execution order
    inputs: tuple[frozenset[int], ...]              # unit k <- units feeding its forward
    params: tuple[tuple[tuple[str, int], ...], ...]  # unit k -> ((param id, bytes), ...)

    def consumers(self) -> list[set[int]]:
        out: list[set[int]] = [set() for _ in self.names]
        for k, ins in enumerate(self.inputs):
            for v in ins:
                out[v].add(k)
        return out


class _Provenance(TorchDispatchMode):
    """Tracks, per tensor, which units' outputs it was computed from."""

    def __init__(self):
        super().__init__()
        self.origin: dict[int, frozenset[int]] = {}
        self.keep: list = []          # keeps traced tensors alive: ids stay unique
        self.stack: list[int] = []    # units whose forward is running (innermost last)
        self.inputs: dict[int, set[int]] = {}

    def __torch_dispatch__(self, func, types, args=(), kwargs=None):
        out = func(*args, **(kwargs or {}))
        src: set[int] = set()
        for t in tree_leaves((args, kwargs)):
            if isinstance(t, torch.Tensor):
                src |= self.origin.get(id(t), frozenset())
        if self.stack:
            unit = self.stack[-1]
            self.inputs.setdefault(unit, set()).update(src - {unit})
            tag = frozenset((unit,))
        else:
            tag = frozenset(src)
        for t in tree_leaves(out):
            if isinstance(t, torch.Tensor):
                self.origin[id(t)] = tag
                self.keep.append(t)
        return out


def _units(model: torch.nn.Module) -> dict[str, torch.nn.Module]:
    return {name: m for name, m in model.named_modules() if any(True for _ in m.parameters(recurse=False))}


def trace_units(model: torch.nn.Module, example_inputs: tuple) -> UnitGraph:
    """Unit dataflow of one forward pass of `model` on `example_inputs`
    (traced on a meta-device copy; `model` itself is not run)."""
    named = list(model.named_parameters())
    pids = {id(p): param_id(i, len(named)) for i, (_, p) in enumerate(named)}
    owner_name = {}
    for name, m in _units(model).items():
        for p in m.parameters(recurse=False):
            owner_name[id(p)] = name
    by_name: dict[str, list[tuple[str, int]]] = {}
    for _, p in named:
        by_name.setdefault(owner_name[id(p)], []).append((pids[id(p)], 4 * p.numel()))
    ghost = copy.deepcopy(model).to("meta")
    units = _units(ghost)
    index: dict[str, int] = {}   # name -> execution position
    mode = _Provenance()
    handles = []

    def pre(name):
        def hook(_m, _args):
            k = index.setdefault(name, len(index))
            mode.stack.append(k)
        return hook

    def post(_m, _args, _out):
        mode.stack.pop()

    for name, m in units.items():
        handles.append(m.register_forward_pre_hook(pre(name)))
        handles.append(m.register_forward_hook(post))
    meta_in = tuple(torch.empty_like(x, device="meta") if isinstance(x, torch.Tensor) else x for x in example_inputs)
    try:
        with torch.no_grad(), mode:
            ghost(*meta_in)
    finally:
        for h in handles:
            h.remove()
    missing = [n for n in by_name if n not in index]
    if missing:
        raise RuntimeError(f"modules with parameters that never ran forward: {missing[:5]}")
    names = tuple(sorted(index, key=index.get))
    return UnitGraph(names=names, inputs=tuple(frozenset(mode.inputs.get(k, ())) for k in range(len(names))),
                     params=tuple(tuple(by_name[n]) for n in names))


def build_dag(graph: UnitGraph, fwd_us: dict[int, int], bwd_us: dict[int, int]) -> DataflowDag:
    """DataflowDag of a traced unit graph with per-unit forward/backward
    durations (see the module docstring for the op naming and edges)."""
    K = len(graph.names)
    cons = graph.consumers()
    sinks = [k for k in range(K) if not cons[k]]
    fid = [f"f{k:04d}" for k in range(K)]
    bid = [f"b{K - 1 - k:04d}" for k in range(K)]
    ops: dict[str, Op] = {}
    params: dict[str, Parameter] = {}
    for k in range(K):
        reads = set()
        for pid, nbytes in graph.params[k]:
            params[pid] = Parameter(pid, nbytes)
            ops[f"r_{pid}"] = Op(f"r_{pid}", OpKind.PARAM_READ, 0, frozenset(), Phase.FORWARD, pid)
            ops[f"u_{pid}"] = Op(f"u_{pid}", OpKind.PARAM_UPDATE, 0, frozenset({bid[k]}), Phase.BACKPROP, pid)
            reads.add(f"r_{pid}")
        fdeps = reads | {fid[v] for v in graph.inputs[k]}
        ops[fid[k]] = Op(fid[k], OpKind.COMPUTE, max(1, int(fwd_us.get(k, 1))), frozenset(fdeps), Phase.FORWARD)
        bdeps = {bid[w] for w in cons[k]} if cons[k] else {fid[s] for s in sinks}
        ops[bid[k]] = Op(bid[k], OpKind.COMPUTE, max(1, int(bwd_us.get(k, 1))), frozenset(bdeps), Phase.BACKPROP)
    return DataflowDag(ops=ops, params=params)


def synthetic_durations(graph: UnitGraph) -> tuple[dict[int, int], dict[int, int]]:
    """The survey's stand-in timing: forward max(1, int(numel /
    1e6 * 100)) us per unit, backward twice that -- for planning a traced
    graph without a device."""
    fwd = {k: max(1, int(sum(b for _, b in ps) / 4 / 1e6 * 100)) for k, ps in enumerate(graph.params)}
    return fwd, {k: 2 * v for k, v in fwd.items()}


@dataclass
class IngestedModel:
    dag: DataflowDag
    params: dict[str, torch.nn.Parameter]       # param id -> parameter
    modules: dict[str, torch.nn.Module]          # param id -> owning module
    forward_us: dict[str, int]                   # op id -> duration
    runs: int
    graph: UnitGraph | None = None


def _measure(model: torch.nn.Module, step_fn, names: tuple[str, ...], runs: int) -> tuple[dict, dict]:
    """Per-unit forward / backward device time (us), minimum over `runs`."""
    mods = dict(model.named_modules())
    pos = {id(mods[n]): k for k, n in enumerate(names)}
    fwd_events: list[list] = []
    bwd_events: list[list] = []
    handles = []

    def f_hook(m, *_):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        fwd_events[-1].append((pos[id(m)], ev))

    def make_b_hook(k):
        def b_hook(_p):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            bwd_events[-1].append((k, ev))
        return b_hook

    for k, n in enumerate(names):
        handles.append(mods[n].register_forward_hook(f_hook))
        for p in mods[n].parameters(recurse=False):
            handles.append(p.register_post_accumulate_grad_hook(make_b_hook(k)))
    samples: dict[tuple[str, int], list[int]] = {}
    try:
        for r in range(runs + 1):  # the first run warms up
            fwd_events.append([])
            bwd_events.append([])
            start = torch.cuda.Event(enable_timing=True)
            start.record()
            step_fn()
            torch.cuda.synchronize()
            if r == 0:
                continue
            prev, t_f = start, {}
            for k, ev in fwd_events[-1]:
                t_f[k] = t_f.get(k, 0.0) + prev.elapsed_time(ev)
                prev = ev
            last = {}
            for k, ev in bwd_events[-1]:  # a unit's boundary: its last gradient's accumulation
                last[k] = ev
            t_b = {}
            for k, ev in sorted(last.items(), key=lambda kv: prev.elapsed_time(kv[1])):
                t_b[k] = max(0.0, prev.elapsed_time(ev))
                prev = ev
            for k in range(len(names)):
                for kind, t in (("f", t_f), ("b", t_b)):
                    samples.setdefault((kind, k), []).append(max(1, int(round(1000.0 * t.get(k, 0.0)))))
    finally:
        for h in handles:
            h.remove()
    est = estimate_op_times([OpProfile(f"{kind}{k}", tuple(v)) for (kind, k), v in samples.items()])
    return ({k: est[f"f{k}"] for k in range(len(names))}, {k: est[f"b{k}"] for k in range(len(names))})


def ingest_model(model: torch.nn.Module, step_fn, runs: int = 5, example_inputs: tuple | None = None) -> IngestedModel:
    """Measured iteration DAG of `model`: structure traced from one forward on
    `example_inputs` (the units' real dataflow), durations from `runs` timed
    executions of `step_fn()` (one forward + backward)."""
    if example_inputs is None:
        raise ValueError("ingest_model needs example_inputs to trace the model's dataflow")
    graph = trace_units(model, example_inputs)
    fwd, bwd = _measure(model, step_fn, graph.names, runs)
    dag = build_dag(graph, fwd, bwd)
    named = list(model.named_parameters())
    mods = dict(model.named_modules())
    by_pid = {param_id(i, len(named)): p for i, (_, p) in enumerate(named)}
    owner = {pid: mods[graph.names[k]] for k in range(len(graph.names)) for pid, _ in graph.params[k]}
    durs = {f"f{k:04d}": v for k, v in fwd.items()}
    return IngestedModel(dag=dag, params=by_pid, modules=owner, forward_us=durs, runs=runs, graph=graph)
