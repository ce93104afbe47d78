"""Symmetric arenas, bootstrap and per-bucket launches over the C ABI.

`Context` owns one rank's (or, under rank emulation, every rank's) bucket and
parameter arenas.  Peers' arenas are mapped through CUDA IPC handles that are
exchanged with `torch.distributed` -- bootstrap only; after that no NCCL (or
any library) call runs on the aggregation path, every byte moves through the
kernels in csrc/caramel.cu.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _native as N


@dataclass(frozen=True)
class SegmentSpec:
    """One member tensor of a bucket, in bucket order."""

    grad: int      # device address of the gradient (0 if none)
    param: int     # device address of the parameter (0 if none)
    offset: int    # element offset inside the bucket
    numel: int


def segment_table(per_rank: list[list[SegmentSpec]], device) -> torch.Tensor:
    """Device copy of caramel_segment[nlocal][nseg] (uint64 words)."""
    rows = []
    for segs in per_rank:
        for s in segs:
            rows.extend((s.grad, s.param, s.offset, s.numel))
    host = torch.tensor(rows, dtype=torch.uint64) if rows else torch.zeros(4, dtype=torch.uint64)
    return host.to(device)


def coalesce(segs: list[SegmentSpec]) -> list[SegmentSpec]:
    """Merge runs of members that are contiguous in memory (gradient AND
    parameter addresses continue where the previous member ends): the packed
    bucket is unchanged, the kernels just see fewer, longer pieces."""
    out: list[SegmentSpec] = []
    for s in segs:
        if out:
            t = out[-1]
            if (t.offset + t.numel == s.offset and t.grad and s.grad == t.grad + 4 * t.numel
                    and ((not t.param and not s.param) or (t.param and s.param == t.param + 4 * t.numel))):
                out[-1] = SegmentSpec(t.grad, t.param, t.offset, t.numel + s.numel)
                continue
        out.append(s)
    return out


def segments_for(tensors: list[torch.Tensor], params: list[torch.Tensor] | None = None) -> list[SegmentSpec]:
    """Segment list for tensors laid out back to back in bucket order."""
    out = []
    off = 0
    for i, g in enumerate(tensors):
        if g.dtype != torch.float32 or not g.is_contiguous():
            raise ValueError("bucket members must be contiguous fp32 tensors")
        p = params[i] if params is not None else None
        if p is not None and (p.numel() != g.numel() or p.dtype != torch.float32 or not p.is_contiguous()):
            raise ValueError("parameter must match its gradient (contiguous fp32)")
        out.append(SegmentSpec(g.data_ptr(), p.data_ptr() if p is not None else 0, off, g.numel()))
        off += g.numel()
    return out


class Context:
    """One process's view of the symmetric arenas.

    nlocal == 1: this process is rank `rank`; call :meth:`bootstrap` (or
    export/import by hand) before launching.  nlocal == world: every rank is
    emulated in this process on one GPU (cooperative launches), no bootstrap.
    """

    def __init__(self, rank: int, world: int, arena_bytes: int, param_bytes: int = 0,
                 nlocal: int = 1):
        self._lib = N.lib()
        self.rank, self.world, self.nlocal = rank, world, nlocal
        ptr = ctypes.c_void_p()
        N.check(self._lib.caramel_init(rank, world, nlocal, arena_bytes, param_bytes, ctypes.byref(ptr)))
        self._ctx = ptr
        self.arena_bytes = arena_bytes
        self.param_bytes = param_bytes
        self.mapped = nlocal == world

    # -- bootstrap -----------------------------------------------------------
    def export(self) -> bytes:
        size = self._lib.caramel_handle_size()
        buf = ctypes.create_string_buffer(size)
        N.check(self._lib.caramel_export(self._ctx, buf))
        return buf.raw

    def import_(self, blobs: list[bytes]) -> None:
        joined = b"".join(blobs)
        buf = ctypes.create_string_buffer(joined, len(joined))
        N.check(self._lib.caramel_import(self._ctx, buf))
        self.mapped = True

    def bootstrap(self, group=None) -> None:
        """Exchange IPC handles with torch.distributed (NCCL/gloo), map peers."""
        import torch.distributed as dist

        mine = self.export()
        blobs: list = [None] * self.world
        dist.all_gather_object(blobs, mine, group=group)
        self.import_(blobs)
        dist.barrier(group=group)  # every rank has zeroed and mapped its arenas

    # -- arenas --------------------------------------------------------------
    def arena_ptrs(self, lr: int = 0) -> tuple[int, int]:
        a = ctypes.c_uint64()
        p = ctypes.c_uint64()
        N.check(self._lib.caramel_arena(self._ctx, lr, ctypes.byref(a), ctypes.byref(p)))
        return a.value, p.value

    def arena_view(self, lr: int, byte_off: int, numel: int, param: bool = False) -> torch.Tensor:
        """fp32 tensor view of arena memory (for tests and host staging)."""
        a, p = self.arena_ptrs(lr)
        base = p if param else a
        limit = self.param_bytes if param else self.arena_bytes
        if byte_off % 4 or byte_off + 4 * numel > limit:
            raise ValueError("view outside the arena")
        return _view_fp32(base + byte_off, numel)

    def status(self) -> None:
        """Raise CaramelError if a flag wait ever timed out (synchronizes)."""
        N.check(self._lib.caramel_status(self._ctx))

    def poll(self) -> None:
        """Same check without synchronizing (host-mapped status word)."""
        N.check(self._lib.caramel_poll(self._ctx))

    def set_timeout_ms(self, ms: int) -> None:
        N.check(self._lib.caramel_set_timeout_ms(self._ctx, ms))

    # -- launches ------------------------------------------------------------
    def allreduce(self, bucket: N.Bucket, epoch: int, stream: int) -> None:
        fn = self._lib.caramel_allreduce_update if bucket.epilogue == N.EPI_SGD else self._lib.caramel_allreduce
        N.check(fn(self._ctx, ctypes.byref(bucket), epoch, ctypes.c_void_p(stream)))

    # -- NVLS multicast arena (the non-fixed-order mode) ----------------------
    def nvls_available(self) -> bool:
        return bool(self._lib.caramel_mc_available(self._ctx))

    def nvls_setup(self, nbytes: int, group=None) -> int:
        """Create, exchange and bind a multicast arena of `nbytes` on every rank
        (collective: every rank calls).  Returns this rank's unicast base
        address; `nvls_view` wraps it."""
        import uuid

        import torch.distributed as dist

        tok: list = [uuid.uuid4().hex[:16] if self.rank == 0 else None]
        dist.broadcast_object_list(tok, src=0, group=group)
        N.check(self._lib.caramel_mc_create(self._ctx, nbytes, tok[0].encode()))
        dist.barrier(group=group)          # rank 0 listens
        N.check(self._lib.caramel_mc_exchange(self._ctx))
        dist.barrier(group=group)          # every GPU added to the multicast object
        base = ctypes.c_uint64()
        N.check(self._lib.caramel_mc_bind(self._ctx, ctypes.byref(base)))
        dist.barrier(group=group)          # every GPU bound
        self.nvls_base, self.nvls_bytes = base.value, nbytes
        return base.value

    def nvls_view(self, byte_off: int, numel: int) -> torch.Tensor:
        if byte_off % 4 or byte_off + 4 * numel > self.nvls_bytes:
            raise ValueError("view outside the multicast arena")
        return _view_fp32(self.nvls_base + byte_off, numel)

    def allreduce_nvls(self, bucket: N.Bucket, epoch: int, stream: int) -> None:
        N.check(self._lib.caramel_allreduce_nvls(self._ctx, ctypes.byref(bucket), epoch, ctypes.c_void_p(stream)))

    def close(self) -> None:
        if self._ctx:
            self._lib.caramel_finalize(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pack(table: torch.Tensor, nseg: int, numel: int, bucket_ptr: int, stream: int) -> None:
    """K1: gather members into a bucket (caramel_pack)."""
    N.check(N.lib().caramel_pack(ctypes.c_void_p(table.data_ptr()), nseg, numel,
                                 ctypes.c_void_p(bucket_ptr), ctypes.c_void_p(stream)))


def unpack(table: torch.Tensor, nseg: int, numel: int, bucket_ptr: int, to_param: bool, stream: int) -> None:
    """K4 scatter: bucket back into the members (caramel_unpack)."""
    N.check(N.lib().caramel_unpack(ctypes.c_void_p(table.data_ptr()), nseg, numel,
                                   ctypes.c_void_p(bucket_ptr), 1 if to_param else 0,
                                   ctypes.c_void_p(stream)))


def _view_fp32(addr: int, numel: int) -> torch.Tensor:
    """Wrap raw device memory (owned by the C library) as a CUDA fp32 tensor."""
    class _CAI:
        __cuda_array_interface__ = {
            "shape": (numel,),
            "typestr": "<f4",
            "data": (addr, False),
            "version": 3,
            "strides": None,
            "stream": None,
        }

    return torch.as_tensor(_CAI(), device="cuda")


def make_bucket(numel: int, bucket_off: int, flag_off: int, *, depth: int = 1, pattern: int = N.SHUFFLE,
                epilogue: int = N.EPI_SUM, flags: int = 0, ctas: int = 1, segs: torch.Tensor | None = None,
                nseg: int = 0, param_off: int = 0, lr: float = 0.0, scale: float = 1.0) -> N.Bucket:
    b = N.Bucket()
    b.numel = numel
    b.bucket_off = bucket_off
    b.param_off = param_off
    b.flag_off = flag_off
    b.segs = segs.data_ptr() if segs is not None else 0
    b.nseg = nseg
    b.depth = depth
    b.pattern = pattern
    b.epilogue = epilogue
    b.flags = flags
    b.ctas = ctas
    b.lr = lr
    b.scale = scale
    return b
