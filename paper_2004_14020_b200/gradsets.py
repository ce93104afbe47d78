"""Gradient inventories of the BASELINE.json configs and their iteration graphs.

The four model configs use the exact parameter shapes of the
torchvision models, recorded once from `named_parameters()` on the meta device
into data/gradsets.json (so nothing here needs torchvision at run time):

  vgg16          32 tensors  138,357,544 elements
  resnet50      161 tensors   25,557,032 elements
  inception_v3  292 tensors   27,161,264 elements (aux logits on)
  alexnet        16 tensors   61,100,840 elements

`layered_chain_dag` is the survey's stand-in DAG for a model:
read marker r_p{i} -> forward f{i} (after f{i-1}, duration
max(1, int(numel/1e6*100)) us); a backward chain b{j} visits tensors in
reverse at twice the forward duration and b{j} feeds update marker u_p{i}.
Ids are zero-padded so lexicographic priority is the intended order.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from functools import lru_cache
from pathlib import Path

from .dag import DataflowDag, Op, OpKind, Parameter, Phase

DATA = Path(__file__).resolve().parent / "data" / "gradsets.json"
MODELS = ("vgg16", "resnet50", "inception_v3", "alexnet")


@dataclass(frozen=True)
class Tensor:
    name: str
    shape: tuple[int, ...]

    @property
    def numel(self) -> int:
        return math.prod(self.shape) if self.shape else 1

    @property
    def nbytes(self) -> int:
        return 4 * self.numel


@lru_cache(maxsize=None)
def gradient_set(model: str) -> tuple[Tensor, ...]:
    """Parameter tensors of `model` in named_parameters() order."""
    doc = json.loads(DATA.read_text())
    if model not in doc:
        raise KeyError(f"unknown model {model!r}; choose from {sorted(doc)}")
    return tuple(Tensor(n, tuple(s)) for n, s in doc[model]["tensors"])


def param_id(i: int, count: int) -> str:
    return f"p{i:0{len(str(count))}d}"


def layered_chain_dag(model: str | tuple[Tensor, ...]) -> DataflowDag:
    tensors = gradient_set(model) if isinstance(model, str) else tuple(model)
    n = len(tensors)
    w = len(str(n))
    ops: dict[str, Op] = {}
    params: dict[str, Parameter] = {}
    fwd = [max(1, int(t.numel / 1e6 * 100)) for t in tensors]
    for i, t in enumerate(tensors):
        pid = f"p{i:0{w}d}"
        params[pid] = Parameter(pid, t.nbytes)
        rid, fid = f"r_{pid}", f"f{i:0{w}d}"
        ops[rid] = Op(rid, OpKind.PARAM_READ, 0, frozenset(), Phase.FORWARD, pid)
        deps = {rid} | ({f"f{i - 1:0{w}d}"} if i else set())
        ops[fid] = Op(fid, OpKind.COMPUTE, fwd[i], frozenset(deps), Phase.FORWARD)
    for j in range(n):
        i = n - 1 - j
        bid = f"b{j:0{w}d}"
        dep = f"b{j - 1:0{w}d}" if j else f"f{n - 1:0{w}d}"
        ops[bid] = Op(bid, OpKind.COMPUTE, 2 * fwd[i], frozenset({dep}), Phase.BACKPROP)
        pid = f"p{i:0{w}d}"
        uid = f"u_{pid}"
        ops[uid] = Op(uid, OpKind.PARAM_UPDATE, 0, frozenset({bid}), Phase.BACKPROP, pid)
    return DataflowDag(ops=ops, params=params)


def shapes_by_param(model: str) -> dict[str, tuple[int, ...]]:
    """param id (as in layered_chain_dag) -> tensor shape."""
    ts = gradient_set(model)
    return {param_id(i, len(ts)): t.shape for i, t in enumerate(ts)}
