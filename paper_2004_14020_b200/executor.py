"""From a plan to real launches: lowering, arenas, schedule enforcement.

`lower()` turns the planner's PipelineArtifacts (pipeline.py) into a
rank-invariant ExecPlan:

* launch order = TransferSchedule.transfers order (transfer.py:193) -- the
  order every rank enqueues bucket collectives on its comm stream, so cross-
  rank flag waits can never cross (schedule enforcement);
* per bucket: members in BatchGroup.param_ids order (batching.py:76,122),
  depth from the plan (pipeline.py:83-86, adaptive_depth), CTA count and flag
  block size from caramel_bucket_layout, byte offsets into the symmetric
  bucket arena and parameter arena (identical on every rank);
* trigger = the bucket's last member gradient (BatchGroup.ready_time_us is
  the max member start, batching.py:84-91); placement BP vs FP (postponed
  update, transfer.py:156-160);
* a digest all-gathered at init so mismatched plans fail loudly instead of
  deadlocking.

`Aggregator` owns the CUDA context (comm.Context), moves the parameters into
the symmetric parameter arena (bucket order, so each bucket's parameters are
contiguous and the owner's fused SGD epilogue stores them straight into every
replica), keeps persistent gradient tensors, and launches buckets either all
at once (`step`, graph-capturable) or as their gradients become ready
(`attach_hooks`, register_post_accumulate_grad_hook) on a dedicated comm
stream in the enforced order.
"""

from __future__ import annotations

import ctypes
import hashlib
import json
import os
from dataclasses import dataclass, field

import torch

from . import _native as N
from . import comm
from .collective import Pattern
from .pipeline import PipelineArtifacts
from .transfer import PlacementKind

PATTERN_CODE = {Pattern.RING: N.RING, Pattern.HALVING_DOUBLING: N.HD, Pattern.SHUFFLE: N.SHUFFLE}
ALIGN = 256
#: overlapped-mode engines whose waits are stream memory operations
STREAM_ENGINES = ("ce", "gated")
#: their stream-memory-op waits stall the stream's hardware queue; with fewer
#: queues than streams a wait can stall the backward pass too
CE_MIN_CONNECTIONS = 16


def agree(what: str, payload: str, world: int, group=None) -> None:
    """All-gather a rank's view of `what` (its hash) and raise DeadlockDetected
    if any two ranks differ: the flag protocols are only deadlock-free when
    every rank launches the same buckets, in the same order, the same way."""
    import torch.distributed as dist

    from .sim import DeadlockDetected

    mine = hashlib.sha256(payload.encode()).hexdigest()
    allv: list = [None] * world
    dist.all_gather_object(allv, mine, group=group)
    if len(set(allv)) != 1:
        bad = [r for r, v in enumerate(allv) if v != allv[0]]
        raise DeadlockDetected(f"ranks disagree on the {what} (ranks {bad} differ from rank 0): "
                               "the flag protocols would deadlock")


def ce_connections_ok() -> bool:
    """True if CUDA_DEVICE_MAX_CONNECTIONS gives every stream its own queue."""
    try:
        return int(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8")) >= CE_MIN_CONNECTIONS
    except ValueError:
        return False


def _align(x: int, a: int = ALIGN) -> int:
    return (x + a - 1) // a * a


@dataclass(frozen=True)
class ExecBucket:
    index: int                    # launch position
    group_id: str
    param_ids: tuple[str, ...]    # member order inside the bucket
    numels: tuple[int, ...]
    numel: int
    depth: int
    ctas: int
    bucket_off: int
    flag_off: int
    param_off: int
    placement: str                # PlacementKind value
    ready_time_us: float


@dataclass(frozen=True)
class ExecPlan:
    world: int
    pattern: int
    buckets: tuple[ExecBucket, ...]
    arena_bytes: int
    param_bytes: int
    total_numel: int

    def digest(self) -> str:
        doc = {"world": self.world, "pattern": self.pattern, "arena": self.arena_bytes,
               "param": self.param_bytes,
               "buckets": [[b.group_id, list(b.param_ids), list(b.numels), b.depth, b.ctas, b.bucket_off,
                            b.flag_off, b.param_off] for b in self.buckets]}
        return hashlib.sha256(json.dumps(doc, sort_keys=True).encode()).hexdigest()

    def bus_bytes(self) -> int:
        """Per-GPU NVLink bytes of one aggregation pass: sum of 2(p-1)/p * S
        (StagePlan.total_transfer_bytes, collective.py:15-16)."""
        p = self.world
        return sum(2 * (p - 1) * 4 * b.numel // p for b in self.buckets) if p > 1 else 0


def lower(art: PipelineArtifacts, numels: dict[str, int], world: int, pattern: Pattern = Pattern.SHUFFLE,
          max_ctas: int | None = None) -> ExecPlan:
    """Rank-invariant launch plan of a pipeline run (see module docstring)."""
    groups = {g.group_id: g for g in art.batch_plan.groups}
    launch = [t for t in art.transfer_schedule.transfers]
    if {t.group_id for t in launch} != set(groups):
        raise ValueError("transfer schedule and batch plan disagree")
    rows = [(t.group_id, tuple(groups[t.group_id].param_ids), groups[t.group_id].total_bytes,
             int(art.depths[t.group_id]), t.placement.value, groups[t.group_id].ready_time_us) for t in launch]
    return lower_groups(rows, numels, world, pattern, max_ctas)


def lower_groups(rows, numels: dict[str, int], world: int, pattern: Pattern = Pattern.SHUFFLE,
                 max_ctas: int | None = None) -> ExecPlan:
    """ExecPlan from buckets in launch order: rows of (group_id, param_ids,
    total_bytes, depth, placement, ready_time_us) -- from a pipeline run
    (lower) or from persisted plan files (planio.load_exec_plan)."""
    code = PATTERN_CODE[pattern]
    buckets = []
    off = 0
    poff = 0
    for idx, (gid, pids, total_bytes, depth, placement, ready) in enumerate(rows):
        ns = tuple(int(numels[p]) for p in pids)
        n = sum(ns)
        if 4 * n != total_bytes:
            raise ValueError(f"{gid}: fp32 member sizes {4 * n} B != planned {total_bytes} B")
        depth = int(depth)
        ctas, bbytes, _ = N.bucket_layout(n, depth, code, world)
        if max_ctas:
            ctas = max(1, min(ctas, max_ctas))
        fbytes = N.flag_bytes_for(depth, ctas, code, world)
        boff = off
        foff = _align(boff + bbytes)
        off = _align(foff + fbytes)
        buckets.append(ExecBucket(index=idx, group_id=gid, param_ids=tuple(pids), numels=ns,
                                  numel=n, depth=depth, ctas=ctas, bucket_off=boff, flag_off=foff,
                                  param_off=poff, placement=placement, ready_time_us=float(ready)))
        poff = _align(poff + 4 * n)
    return ExecPlan(world=world, pattern=code, buckets=tuple(buckets), arena_bytes=max(off, ALIGN),
                    param_bytes=max(poff, ALIGN), total_numel=sum(b.numel for b in buckets))


@dataclass
class _Live:
    """Per-bucket runtime state."""

    spec: ExecBucket
    desc: N.Bucket
    table: torch.Tensor
    members: list[str]
    remaining: int = 0
    done: torch.cuda.Event | None = None
    ce_done: torch.cuda.Event | None = None  # engine="ce": recorded by the library's worker
    gate_modules: list = field(default_factory=list)


def host_groups(sizes: list[int], group_bytes: int, taper_bytes: int = 0) -> list[tuple[int, int]]:
    """Consecutive ranges [i, j) of `sizes` (bytes, launch order) of about
    `group_bytes` each, every range non-empty; taper_bytes > 0 caps a range
    at min(group_bytes, max(taper_bytes, min(bytes before it, half the bytes
    from its start))) -- see Aggregator.host_groups."""
    total = sum(sizes)
    out, i, done = [], 0, 0
    while i < len(sizes):
        target = group_bytes
        if taper_bytes:
            target = min(group_bytes, max(taper_bytes, min(done, (total - done) // 2)))
        j, acc = i, 0
        while j < len(sizes) and (j == i or acc + sizes[j] <= target):
            acc += sizes[j]
            j += 1
        out.append((i, j))
        done += acc
        i = j
    return out


class Aggregator:
    """Runs an ExecPlan's bucket collectives on this rank.

    params   : param id -> fp32 CUDA tensor (the model's parameters); with
               `param_arena=True` their storage is moved into the symmetric
               parameter arena (values kept) so the fused SGD epilogue writes
               every replica directly.
    epilogue : "sgd" (fused postponed update), "mean" or "sum" (gradient
               all-reduce, result written back into .grad).
    engine   : overlapped-mode (hooks) engine; "auto" picks "ce" where it
               applies (zero-copy gradients, world > 1, SHUFFLE), else "sm".
               "sm": the NVLink kernels
               (caramel_allreduce / _many).  "ce": the copy-engine two-shot
               (caramel_allreduce_ce) -- bytes move on the copy engines and
               ranks wait on stream memory operations, so the backward kernels
               keep every SM; buckets under `ce_min_bytes` still take the SM
               kernels.  Needs grads="bucket", world > 1, SHUFFLE.
               "gated": the NVLink SM kernels with every wait on the stream
               front end (caramel_allreduce_gated): the kernel is scheduled
               only once every peer's gradients are ready, so it never holds
               an SM while waiting; same requirements as "ce".
               step() / step_host*() always use the SM kernels.
    """

    def __init__(self, plan: ExecPlan, params: dict[str, torch.Tensor], *, rank: int = 0, lr: float = 0.01,
                 epilogue: str = "sgd", param_arena: bool = True, grads: str = "bucket", group=None,
                 bootstrap: bool = True, engine: str = "auto"):
        if engine not in ("auto", "sm") + STREAM_ENGINES:
            raise ValueError("engine must be 'auto', 'sm', 'ce' or 'gated'")
        if engine in STREAM_ENGINES and (grads != "bucket" or plan.world < 2 or plan.pattern != N.SHUFFLE):
            raise ValueError(f"engine={engine!r} needs grads='bucket', world > 1 and the SHUFFLE pattern")
        self.engine = engine
        self.plan = plan
        self.rank, self.world = rank, plan.world
        self.lr = float(lr)
        self.epi = {"sum": N.EPI_SUM, "mean": N.EPI_SCALE, "sgd": N.EPI_SGD}[epilogue]
        self.param_arena = bool(param_arena) and self.epi == N.EPI_SGD
        self.params = params
        dev = next(iter(params.values())).device
        if dev.type != "cuda":
            raise ValueError("parameters must live on a CUDA device")
        self.device = dev
        self.ctx = comm.Context(rank, self.world, plan.arena_bytes,
                                plan.param_bytes if self.param_arena else 0)
        if self.world > 1 and bootstrap:
            agree("execution plan", plan.digest(), self.world, group)
            self.ctx.bootstrap(group)
        if engine in STREAM_ENGINES and not N.lib().caramel_ce_available(self.ctx._ctx):
            raise RuntimeError(f"engine={engine!r}: this device lacks 64-bit stream memory operations")
        if engine in STREAM_ENGINES and not ce_connections_ok():
            raise RuntimeError(f"engine={engine!r} needs CUDA_DEVICE_MAX_CONNECTIONS >= {CE_MIN_CONNECTIONS} in the "
                               "environment before CUDA initialises: a stream-memory-op wait stalls its hardware "
                               "queue, and with shared queues it can stall the backward pass behind a peer")
        if engine == "auto":
            ok = grads == "bucket" and self.world > 1 and plan.pattern == N.SHUFFLE and ce_connections_ok()
            engine = "ce" if ok and N.lib().caramel_ce_available(self.ctx._ctx) else "sm"
        self.engine = engine
        self._group = group
        self._engines_checked = not (self.world > 1 and bootstrap)
        if self.param_arena:
            self._adopt_params()
        # Gradient storage:
        #   "bucket" (default) zero-copy, see below
        #   "flat"   views into one flat buffer with the parameter arena's layout
        #            (bucket order, gradient_as_bucket_view style): the pack kernel
        #            gathers contiguous runs, host staging is one copy per group
        #   "bucket" zero-copy: views into the symmetric bucket arena itself --
        #            autograd writes every bucket in place, peers read it over
        #            NVLink, no pack at all
        #   "own"    keep the caller's gradient tensors (arbitrary addresses)
        if grads not in ("flat", "bucket", "own"):
            raise ValueError("grads must be 'flat', 'bucket' or 'own'")
        self.grads = grads
        self.grad_flat = None
        if grads == "flat":
            self.grad_flat = torch.zeros(plan.param_bytes // 4, device=dev)
            for b in plan.buckets:
                off = b.param_off // 4
                for pid, n in zip(b.param_ids, b.numels):
                    params[pid].grad = self.grad_flat[off:off + n].view(params[pid].shape)
                    off += n
        elif grads == "bucket":
            for b in plan.buckets:
                region = self.ctx.arena_view(0, b.bucket_off, b.numel)
                region.zero_()
                off = 0
                for pid, n in zip(b.param_ids, b.numels):
                    params[pid].grad = region[off:off + n].view(params[pid].shape)
                    off += n
        for p in params.values():
            if p.grad is None:
                p.grad = torch.zeros_like(p)
        self.comm_stream = torch.cuda.Stream(device=dev, priority=self.comm_priority)
        self._live = [self._make_live(b) for b in plan.buckets]
        self._by_param = {}
        for lv in self._live:
            for pid in lv.members:
                self._by_param[pid] = lv
        if self.engine in STREAM_ENGINES:
            for lv in self._live:  # materialised now, recorded by the worker thread later
                lv.ce_done = torch.cuda.Event()
                lv.ce_done.record(self.comm_stream)
        self._next = 0
        self._hooks = []
        self.epoch = 0
        self._ce_epoch = 0
        self.launches = 0
        self._last_done = None
        self._fp_pending = set()
        self._gated = False
        self._build_list()

    # -- setup -----------------------------------------------------------------
    def _adopt_params(self) -> None:
        """Move every parameter into the symmetric arena in bucket order."""
        for b in self.plan.buckets:
            off = b.param_off
            for pid, n in zip(b.param_ids, b.numels):
                p = self.params[pid]
                view = self.ctx.arena_view(0, off, n, param=True).view(p.shape)
                view.copy_(p.detach())
                p.data = view
                off += 4 * n

    def _make_live(self, b: ExecBucket) -> _Live:
        segs = comm.coalesce(comm.segments_for([self.params[p].grad for p in b.param_ids],
                                               None if self.param_arena else [self.params[p] for p in b.param_ids]))
        table = comm.segment_table([segs], self.device)
        if self.grads == "bucket":
            # zero-copy: the bucket IS the gradient storage; results land in the
            # parameter arena (SGD) or in place (mean / sum; ring/hd unpack)
            flags = N.F_PARAM_ARENA if self.param_arena else N.F_UNPACK
            if self.engine in STREAM_ENGINES and not self.param_arena:
                flags = 0  # the copy-engine all-gather lands in the bucket = the gradients
        else:
            flags = N.F_PACK | (N.F_PARAM_ARENA if self.param_arena else N.F_UNPACK)
            if len(segs) == 1 and segs[0].grad % 16 == 0:
                flags |= N.F_FLAT  # one contiguous aligned gradient run: TMA streaming path
        scale = 1.0 / self.world
        desc = comm.make_bucket(b.numel, b.bucket_off, b.flag_off, depth=b.depth, pattern=self.plan.pattern,
                                epilogue=self.epi, flags=flags, ctas=b.ctas, segs=table, nseg=len(segs),
                                param_off=b.param_off, lr=self.lr, scale=scale)
        return _Live(spec=b, desc=desc, table=table, members=list(b.param_ids))

    def _build_list(self) -> None:
        """Host + device copies of every bucket descriptor (launch order) and
        the element prefix sums, for the one-launch pass (caramel_allreduce_many)."""
        n = len(self._live)
        self._host_list = (N.Bucket * n)(*[lv.desc for lv in self._live])
        raw = bytes(self._host_list)
        self._dev_list = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(self.device)
        prefix, segpre = [0], [0]
        for lv in self._live:
            prefix.append(prefix[-1] + lv.spec.numel)
            segpre.append(segpre[-1] + lv.desc.nseg)
        self._prefix = prefix
        self._dev_prefix = torch.tensor(prefix, dtype=torch.int64, device=self.device)
        self._dev_segprefix = torch.tensor(segpre, dtype=torch.int64, device=self.device)

    def refresh_tables(self) -> None:
        """Rebuild segment tables (after gradients were reallocated)."""
        old = self._live
        self._live = [self._make_live(lv.spec) for lv in old]
        for a, b in zip(old, self._live):
            b.ce_done = a.ce_done
        self._by_param = {pid: lv for lv in self._live for pid in lv.members}
        self._build_list()

    def check_tables(self) -> bool:
        """True if every gradient still lives where the segment tables point."""
        for lv in self._live:
            segs = comm.coalesce(comm.segments_for([self.params[p].grad for p in lv.members],
                                                   None if self.param_arena else
                                                   [self.params[p] for p in lv.members]))
            rows = lv.table.view(-1, 4).cpu().tolist()[:len(segs)]
            if len(segs) != lv.desc.nseg or [list(map(int, r)) for r in rows] != \
                    [[s_.grad, s_.param, s_.offset, s_.numel] for s_ in segs]:
                return False
        return True

    # -- launches --------------------------------------------------------------
    def _launch(self, lv: _Live, stream: int) -> None:
        self.ctx.allreduce(lv.desc, 0, stream)
        self.launches += 1

    def step(self, stream: torch.cuda.Stream | None = None, fused: bool = True) -> None:
        """Aggregate every bucket now, in launch order, on `stream` (default:
        the current stream): one launch for the whole list (fused=True) or one
        launch per bucket.  Graph-capturable: epochs come from the device
        counter advanced first on the same stream -- except where the launch
        needs none: the world = 1 update and the fused two-shot (its grid
        barriers count launches themselves), one kernel per step instead of two."""
        s = (stream or torch.cuda.current_stream(self.device)).cuda_stream
        if self._step_needs_epoch(fused):
            N.check(N.lib().caramel_epoch_advance(self.ctx._ctx, ctypes.c_void_p(s)))
        if fused:
            self._launch_range(0, len(self._live), s, N.MANY_FUSED, 0)
        else:
            for lv in self._live:
                self._launch(lv, s)

    def _launch_range(self, i: int, j: int, stream: int, mode: int, ctas: int) -> None:
        """Buckets [i, j) of the launch order as one caramel_allreduce_many launch."""
        bsz = ctypes.sizeof(N.Bucket)
        host = ctypes.cast(ctypes.byref(self._host_list, i * bsz), ctypes.POINTER(N.Bucket))
        N.check(N.lib().caramel_allreduce_many(self.ctx._ctx, host, j - i, self._dev_list.data_ptr() + i * bsz,
                                               self._dev_prefix.data_ptr() + 8 * i,
                                               self._dev_segprefix.data_ptr() + 8 * i, ctas, mode, 0,
                                               ctypes.c_void_p(stream)))
        self.launches += 1

    def _launch_ce(self, i: int, j: int, stream: int, grad_stream: int | None = None) -> None:
        """Buckets [i, j) of the launch order on the copy engines
        (caramel_allreduce_ce); READY is signalled on `grad_stream` (default:
        the current stream, where autograd produced the gradients)."""
        bsz = ctypes.sizeof(N.Bucket)
        host = ctypes.cast(ctypes.byref(self._host_list, i * bsz), ctypes.POINTER(N.Bucket))
        gs = grad_stream if grad_stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        N.check(N.lib().caramel_allreduce_ce(self.ctx._ctx, host, j - i, i, self._ce_epoch, ctypes.c_void_p(gs),
                                             ctypes.c_void_p(stream)))
        self.launches += 1

    def host_groups(self, group_bytes: int = 16 << 20, taper_bytes: int = 0) -> list[tuple[int, int]]:
        """Consecutive launch-order bucket ranges of about `group_bytes` each
        (identical on every rank).  taper_bytes > 0: the groups grow from
        about taper_bytes (doubling: at most the bytes already grouped) and
        shrink the same way towards the end (at most half of what is left),
        so the upload of the first group and the download of the last -- the
        two transfers a two-stream pipeline cannot overlap -- are short."""
        return host_groups([4 * lv.spec.numel for lv in self._live], group_bytes, taper_bytes)

    def flat_layout(self) -> list[tuple[str, int, int]]:
        """(param id, element offset, numel) of every parameter in the flat
        arena layout used by step_host_flat (bucket order, 256 B aligned buckets)."""
        out = []
        for b in self.plan.buckets:
            off = b.param_off // 4
            for pid, n in zip(b.param_ids, b.numels):
                out.append((pid, off, n))
                off += n
        return out

    def step_host_flat(self, host_grads: torch.Tensor, host_params: torch.Tensor | None = None,
                       group_bytes: int = 16 << 20, taper_bytes: int = 2 << 20) -> int:
        """step_host for flat pinned buffers in the parameter-arena layout
        (flat_layout()): per group of buckets one H2D (grads="flat"; one per
        bucket with grads="bucket") and one D2H cudaMemcpyAsync, overlapped with
        the group's aggregation kernel; groups tapered at both ends
        (host_groups)."""
        if self.grads not in ("flat", "bucket") or not self.param_arena:
            raise RuntimeError("step_host_flat needs grads='flat' or 'bucket' and the parameter arena")
        cur = torch.cuda.current_stream(self.device)
        if not hasattr(self, "_h2d"):
            self._h2d = torch.cuda.Stream(device=self.device)
            self._d2h = torch.cuda.Stream(device=self.device)
        h2d, d2h = self._h2d, self._d2h
        pflat = self.ctx.arena_view(0, 0, self.plan.param_bytes // 4, param=True)
        h2d.wait_stream(cur)
        launches = 0
        if self._step_needs_epoch(True):
            N.check(N.lib().caramel_epoch_advance(self.ctx._ctx, ctypes.c_void_p(cur.cuda_stream)))
            launches = 1
        for i, j in self.host_groups(group_bytes, taper_bytes):
            a = self._live[i].spec.param_off // 4
            last = self._live[j - 1].spec
            b = last.param_off // 4 + last.numel
            with torch.cuda.stream(h2d):
                if self.grad_flat is not None:
                    self.grad_flat[a:b].copy_(host_grads[a:b], non_blocking=True)
                else:  # zero-copy: each bucket's gradients sit in its arena region
                    for lv in self._live[i:j]:
                        o = lv.spec.param_off // 4
                        self._bucket_view(lv).copy_(host_grads[o:o + lv.spec.numel], non_blocking=True)
            cur.wait_stream(h2d)
            self._launch_range(i, j, cur.cuda_stream, N.MANY_FUSED, 0)
            launches += 1
            if host_params is not None:
                d2h.wait_stream(cur)
                with torch.cuda.stream(d2h):
                    host_params[a:b].copy_(pflat[a:b], non_blocking=True)
        cur.wait_stream(d2h)
        return launches

    def capture_step_host_flat(self, host_grads: torch.Tensor, host_params: torch.Tensor | None = None,
                               group_bytes: int = 16 << 20, taper_bytes: int = 2 << 20) -> torch.cuda.CUDAGraph:
        """step_host_flat captured in a CUDA graph: every replay() is one full
        step -- the H2D copies from `host_grads`, the aggregation launches and
        the D2H copies into `host_params` (fixed pinned buffers; write the next
        step's gradients into host_grads between replays) -- with no per-step
        host issue cost, so a busy host does not stall the copy pipeline."""
        self.step_host_flat(host_grads, host_params, group_bytes, taper_bytes)  # lazy streams / views
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
            self.step_host_flat(host_grads, host_params, group_bytes, taper_bytes)
        torch.cuda.current_stream(self.device).wait_stream(side)
        return g

    def _bucket_view(self, lv: _Live) -> torch.Tensor:
        v = getattr(lv, "_view", None)
        if v is None:
            v = lv._view = self.ctx.arena_view(0, lv.spec.bucket_off, lv.spec.numel)
        return v

    def step_host(self, host_grads: dict, host_params: dict | None = None, group_bytes: int = 16 << 20,
                  taper_bytes: int = 2 << 20) -> int:
        """The plugin path with HOST buffers: pinned host gradients -> device,
        aggregation + fused update, updated parameters -> pinned host, pipelined
        per group of buckets on two copy streams so H2D of group i+1, the
        collective of group i and D2H of group i-1 overlap (PCIe is full
        duplex).  Returns the number of kernels launched."""
        cur = torch.cuda.current_stream(self.device)
        if not hasattr(self, "_h2d"):
            self._h2d = torch.cuda.Stream(device=self.device)
            self._d2h = torch.cuda.Stream(device=self.device)
        h2d, d2h = self._h2d, self._d2h
        h2d.wait_stream(cur)
        launches = 0
        if self._step_needs_epoch(True):
            N.check(N.lib().caramel_epoch_advance(self.ctx._ctx, ctypes.c_void_p(cur.cuda_stream)))
            launches = 1
        for i, j in self.host_groups(group_bytes, taper_bytes):
            members = [pid for lv in self._live[i:j] for pid in lv.members]
            with torch.cuda.stream(h2d):
                for pid in members:
                    self.params[pid].grad.view(-1).copy_(host_grads[pid], non_blocking=True)
            cur.wait_stream(h2d)
            self._launch_range(i, j, cur.cuda_stream, N.MANY_FUSED, 0)
            launches += 1
            if host_params is not None:
                d2h.wait_stream(cur)
                with torch.cuda.stream(d2h):
                    for pid in members:
                        host_params[pid].copy_(self.params[pid].view(-1), non_blocking=True)
        cur.wait_stream(d2h)
        return launches

    def step_kernel(self) -> str:
        """Name of the kernel step() launches (mirrors caramel_allreduce_many's dispatch)."""
        if self.world > 1:
            return "k_shuffle_fused" if self.plan.pattern == N.SHUFFLE else "k_collective_many"
        tma = len(self._live) <= 256 and not os.environ.get("CARAMEL_NO_TMA")
        for lv in self._live:
            d = lv.desc
            flat_ok = (d.flags & N.F_FLAT and d.flags & N.F_PACK and d.nseg == 1) or not d.flags & N.F_PACK
            tma = tma and bool(flat_ok) and bool(d.flags & N.F_PARAM_ARENA) and d.epilogue == N.EPI_SGD
        return "k_local_flat_tma" if tma else "k_local_many"

    def _step_needs_epoch(self, fused: bool) -> bool:
        if not fused:
            return True
        if self.world == 1:
            return False
        # CARAMEL_FUSED_PUSH routes fused lists to the push engine, whose flags carry epochs
        return not (self.plan.pattern == N.SHUFFLE and not os.environ.get("CARAMEL_FUSED_PUSH"))

    def kernels_per_step(self, fused: bool = True) -> int:
        if fused:
            return 1 + int(self._step_needs_epoch(True))
        return 1 + len(self._live)

    # -- overlapped mode: launch when the last gradient of a bucket is ready ----
    def attach_hooks(self) -> None:
        """Launch each bucket on the comm stream as soon as its last member's
        gradient is accumulated, never out of the planned launch order.  Call
        begin_iteration() before every backward and finish_iteration() after."""
        for pid, p in self.params.items():
            self._hooks.append(p.register_post_accumulate_grad_hook(self._make_hook(pid)))

    def _make_hook(self, pid):
        def hook(_p):
            lv = self._by_param[pid]
            lv.remaining -= 1
            if lv.remaining == 0:
                self._drain()
        return hook

    def begin_iteration(self) -> None:
        """Arm every bucket for one backward pass (gradients must be zeroed in
        place -- Aggregator.zero_grad(), or zero_grad(set_to_none=False) -- so
        the segment tables stay valid)."""
        if not self._engines_checked:
            self._check_engines()
        for lv in self._live:
            lv.remaining = len(lv.members)
        self._next = 0
        self._last_done = None
        cur = torch.cuda.current_stream(self.device)
        self.comm_stream.wait_stream(cur)
        N.check(N.lib().caramel_epoch_advance(self.ctx._ctx,
                                              ctypes.c_void_p(self.comm_stream.cuda_stream)))
        self._ce_epoch += 1

    #: CUDA priority of the comm stream (lower = higher; torch clamps to the
    #: device's range): a high-priority stream's CTAs are scheduled ahead of
    #: queued backward CTAs as SMs free up (measured: lower exposed time for
    #: the gated and copy-engine engines, profiles/r02_engines_priority.txt)
    comm_priority = -1
    #: overlapped mode: while the comm stream is busy, ready buckets are held
    #: back and coalesced into one list launch (per-bucket flags, so ranks may
    #: group differently) until this many are pending or this many bytes
    coalesce_buckets = 16
    coalesce_bytes = 8 << 20
    coalesce_ctas = 32  # grid of a coalesced launch: leave SMs to the backward pass
    #: engine="ce": buckets below this size still run on the SM kernels (their
    #: latency is lower and they hold SMs only for microseconds)
    ce_min_bytes = 0
    ce_tail_us = 150.0
    ce_tail_frac = 0.02
    _ce_tail = None

    def _comm_busy(self) -> bool:
        return self._last_done is not None and not self._last_done.query()

    def _drain(self, force: bool = False) -> None:
        """Launch ready buckets from the head of the launch order: one at a
        time when the comm stream is idle, coalesced while it is busy."""
        j = self._next
        while j < len(self._live) and self._live[j].remaining == 0:
            j += 1
        if j == self._next:
            return
        pending_bytes = 4 * (self._prefix[j] - self._prefix[self._next])
        if self.engine in STREAM_ENGINES:
            self._drain_ce(j)
            return
        if not force and self._comm_busy() and j - self._next < self.coalesce_buckets \
                and pending_bytes < self.coalesce_bytes:
            return
        cur = torch.cuda.current_stream(self.device)
        self.comm_stream.wait_stream(cur)  # the gradients are produced on `cur`
        s = self.comm_stream.cuda_stream
        if j - self._next == 1:
            self._launch(self._live[self._next], s)
        else:
            ctas = min(self.coalesce_ctas, max(lv.spec.ctas for lv in self._live[self._next:j]) * 4)
            self._launch_range(self._next, j, s, N.MANY_FLAGS, ctas)
        ev = torch.cuda.Event()
        ev.record(self.comm_stream)
        for lv in self._live[self._next:j]:
            lv.done = ev
        self._last_done = ev
        self._next = j

    def engine_assignment(self) -> list[str]:
        """Engine of every bucket in launch order (overlapped mode)."""
        if self.engine == "gated":
            return ["gated"] * len(self._live)
        if self.engine != "ce":
            return ["sm"] * len(self._live)
        return [self._ce_engine_of(k) for k in range(len(self._live))]

    def _check_engines(self) -> None:
        """All-gather the per-bucket engine assignment (and the knobs that
        decide it) once, before the first overlapped iteration: a bucket run by
        the copy-engine protocol on one rank and by the SM flag protocol on
        another would hang, so a mismatch raises instead."""
        doc = json.dumps({"plan": self.plan.digest(), "engine": self.engine,
                          "assignment": self.engine_assignment(),
                          "knobs": [self.ce_min_bytes, self.ce_tail_us, self.ce_tail_frac,
                                    self.coalesce_buckets, self.coalesce_bytes, self.coalesce_ctas]})
        agree("engine of some bucket (engine, ce_min_bytes, ce_tail_* or coalescing knobs)", doc, self.world,
              self._group)
        self._engines_checked = True

    def _ce_engine_of(self, k: int) -> str:
        """Engine of bucket k under engine="ce" (a function of the plan only, so
        identical on every rank): the copy engines, except buckets below
        ce_min_bytes and the tail -- buckets the plan makes ready in the last
        ce_tail_frac of the ready-time span (at least ce_tail_us), launched when
        backward is (nearly) over and the SM kernels' lower latency wins."""
        if self._ce_tail is None:
            ready = [lv.spec.ready_time_us for lv in self._live]
            lo, hi = min(ready), max(ready)
            cut = hi - max(self.ce_tail_us, self.ce_tail_frac * (hi - lo))
            self._ce_tail = {i for i, r in enumerate(ready) if r >= cut}
        if k in self._ce_tail or 4 * self._live[k].spec.numel < self.ce_min_bytes:
            return "sm"
        return "ce"

    def _drain_ce(self, j: int) -> None:
        """engine="ce": one call per bucket (every rank groups the launch order
        identically: a stream-memory-op wait stalls its hardware queue).  Both
        engines' calls go to the library's worker thread (caramel_ce_submit),
        which issues them on the comm stream in launch order, so autograd's
        thread only records an event per bucket and never waits."""
        cur = torch.cuda.current_stream(self.device).cuda_stream
        s = self.comm_stream.cuda_stream
        bsz = ctypes.sizeof(N.Bucket)
        for k in range(self._next, j):
            lv = self._live[k]
            if self.engine == "gated":
                eng = N.ENGINE_GATED
            else:
                eng = N.ENGINE_CE if self._ce_engine_of(k) == "ce" else N.ENGINE_SM
            host = ctypes.cast(ctypes.byref(self._host_list, k * bsz), ctypes.POINTER(N.Bucket))
            N.check(N.lib().caramel_ce_submit(self.ctx._ctx, host, 1, k, self._ce_epoch, eng, ctypes.c_void_p(cur),
                                              ctypes.c_void_p(s), ctypes.c_void_p(lv.ce_done.cuda_event)))
            self.launches += 1
            lv.done = lv.ce_done
        self._next = j

    def _ce_flush(self) -> None:
        if self.engine in STREAM_ENGINES:
            N.check(N.lib().caramel_ce_flush(self.ctx._ctx))

    def finish_iteration(self, postpone: bool = False) -> None:
        """Launch whatever is still held back, then make the current stream
        wait for the buckets.  postpone=True executes the plan's postponed
        update (transfer.py:156-160): buckets placed into the next forward pass
        (FP_OVERLAP) are not waited for here but by the forward gate of the
        first module that reads one of their parameters (gate_forward)."""
        self._drain(force=True)
        self._ce_flush()
        self.ctx.poll()  # host-mapped watchdog word: raises if a wait ever timed out (no sync)
        if self._next != len(self._live):
            missing = [lv.spec.group_id for lv in self._live[self._next:]]
            raise RuntimeError(f"buckets never became ready: {missing[:5]}")
        cur = torch.cuda.current_stream(self.device)
        fp = [i for i, lv in enumerate(self._live) if lv.spec.placement == PlacementKind.FP_OVERLAP.value]
        if not postpone or not fp or not self._gated:
            cur.wait_stream(self.comm_stream)
            return
        bp = [i for i in range(len(self._live)) if i not in set(fp)]
        if bp:  # the comm stream is FIFO: the last BP bucket covers every earlier one
            cur.wait_event(self._live[bp[-1]].done)
        self._fp_pending = {i for i in fp if not bp or i > bp[-1]}

    # -- postponed update: forward gates -----------------------------------------
    _gated = False
    _fp_pending: set = set()

    def gate_forward(self, modules: dict) -> int:
        """Register forward pre-hooks: `modules` maps param id -> the module that
        reads it.  A module whose parameters sit in a postponed (FP_OVERLAP)
        bucket makes the current stream wait for that bucket's kernel before it
        runs, and zeroes the bucket's gradients then (the kernel may read them
        until it completes).  Returns the number of gated modules."""
        by_mod: dict = {}
        for i, lv in enumerate(self._live):
            if lv.spec.placement != PlacementKind.FP_OVERLAP.value:
                continue
            for pid in lv.members:
                m = modules[pid]
                by_mod.setdefault(id(m), (m, set()))[1].add(i)
        for m, idxs in by_mod.values():
            self._hooks.append(m.register_forward_pre_hook(self._make_gate(sorted(idxs))))
        self._gated = bool(by_mod)
        return len(by_mod)

    def _make_gate(self, idxs):
        def gate(_m, _inp):
            if not self._fp_pending:
                return
            cur = torch.cuda.current_stream(self.device)
            for i in idxs:
                if i in self._fp_pending:
                    lv = self._live[i]
                    if lv.done is not None:
                        cur.wait_event(lv.done)
                    torch._foreach_zero_([self.params[pid].grad for pid in lv.members])
                    self._fp_pending.discard(i)
        return gate

    def zero_grad(self) -> None:
        """Zero every gradient in place, except those of postponed buckets
        still in flight (their forward gate zeroes them after the wait)."""
        grads = [self.params[pid].grad for i, lv in enumerate(self._live) if i not in self._fp_pending
                 for pid in lv.members]
        if grads:
            torch._foreach_zero_(grads)

    def sync(self) -> None:
        """Wait for everything, including postponed buckets (e.g. before evaluation)."""
        self._ce_flush()
        cur = torch.cuda.current_stream(self.device)
        cur.wait_stream(self.comm_stream)
        for i in sorted(self._fp_pending):
            torch._foreach_zero_([self.params[pid].grad for pid in self._live[i].members])
        self._fp_pending = set()

    def detach_hooks(self) -> None:
        for h in self._hooks:
            h.remove()
        self._hooks = []

    def status(self) -> None:
        self.ctx.status()

    def release_storage(self) -> None:
        """Give every parameter and gradient torch-owned storage again (values
        kept): the arenas they point into are freed by close()."""
        torch.cuda.current_stream(self.device).wait_stream(self.comm_stream)
        for p in self.params.values():
            if self.param_arena:
                p.data = p.data.clone()
            if p.grad is not None and self.grads in ("bucket", "flat"):
                p.grad = p.grad.clone()
        self.grad_flat = None

    def close(self) -> None:
        """Detach hooks, hand parameters/gradients back to torch-owned storage
        and free the arenas.  The model stays usable (e.g. state_dict())."""
        if self.ctx._ctx is None:
            return
        self.detach_hooks()
        self._ce_flush()
        self.release_storage()
        torch.cuda.synchronize(self.device)
        self.ctx.close()


def calibrate_network_model(world: int, rank: int, sizes: tuple[int, ...] = (64, 4 << 20), reps: int = 8,
                            iters: int = 20, group=None):
    """Fit f(d) = latency + per_byte * d on THIS fabric.

    Times the sm_100a two-shot (caramel_allreduce, adaptive-sized buckets at
    depth 1) on `sizes` -- the paper's 64 B and 4 MB microbenchmarks
     -- `reps` times each, `iters` back-to-back launches per
    sample, takes the max over ranks of every sample (so every rank fits the
    identical model and plans identical buckets) and applies the reference's
    least-squares line (costmodel.py:84-108) through the per-size MEDIANS
    (fit_network_model_robust): one late peer or preempted launch among the
    samples cannot move the bucket cap.  Returns (NetworkModel, measurements)."""
    import torch.distributed as dist

    from .costmodel import Measurement, fit_network_model_robust

    dev = torch.device("cuda", torch.cuda.current_device())
    nmax = max(sizes) // 4 + 1
    _, bbytes, fbytes = N.bucket_layout(nmax, 1, N.SHUFFLE, world)
    flag_off = _align(bbytes)
    ctx = comm.Context(rank, world, arena_bytes=flag_off + 4 * _align(fbytes, 1 << 20) * len(sizes))
    if world > 1:
        ctx.bootstrap(group)
    stream = torch.cuda.current_stream(dev)
    meas = []
    epoch = {}
    for k, size in enumerate(sizes):
        n = max(1, size // 4)
        ctas, _, fb = N.bucket_layout(n, 1, N.SHUFFLE, world)
        b = comm.make_bucket(n, 0, flag_off + k * _align(fbytes, 1 << 20), depth=1, pattern=N.SHUFFLE,
                             epilogue=N.EPI_SUM, flags=0, ctas=ctas)
        epoch[k] = 0
        for r in range(reps + 1):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier(group=group)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            for _ in range(iters):
                epoch[k] += 1
                ctx.allreduce(b, epoch[k], stream.cuda_stream)
            e.record(stream)
            e.synchronize()
            us = s.elapsed_time(e) * 1e3 / iters
            if world > 1:
                t = torch.tensor([us], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
                us = t.item()
            if r > 0:  # first round warms up
                meas.append(Measurement(size_bytes=4 * n, observed_time_us=us))
    ctx.status()
    ctx.close()
    return fit_network_model_robust(meas, "median"), meas
