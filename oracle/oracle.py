"""CPU oracle for the aggregation hot path -- TEST INFRASTRUCTURE ONLY.

Two independent restatements of the same semantics (see caramel_oracle.c's
header for the reference file:line each step follows):

* `np_*`      numpy, written directly from the pattern definitions in
              overlapsim/collective.py:1-21 (ring / hd / shuffle);
* `c_*`       ctypes over liboracle.so (caramel_oracle.c), a plain-C port that
              also counts per-stage bytes so it can be checked against
              stage_plan (collective.py:86-103) and is fast enough to be the
              CPU baseline timed by bench.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl
reference` leg may import this module.  The product package never does.

Parity status: plan-side quantities (membership, order, depths, chunk and
stage byte counts) are pinned against the reference; the numeric values have
no reference golden vector (the reference moves no data), so value parity is
"parity unpinned" beyond the stage semantics restated here.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

RING, HD, SHUFFLE = 0, 1, 2
EPI_SUM, EPI_SCALE, EPI_SGD = 0, 1, 2


# ---------------------------------------------------------------------------
# integer chunk / share rule
# ---------------------------------------------------------------------------
def chunk_bounds(n: int, k: int, p: int) -> list[list[int]]:
    """Row c: share starts of chunk c (p values) followed by the chunk end.

    The reference has only float byte counts per chunk, stage.transfer_bytes/k
    (collective.py:124) with transfer_bytes = d/p (collective.py:90); this is
    the integer rule [floor(c n/k), floor((c+1) n/k)) per chunk and
    [floor(s m/p), floor((s+1) m/p)) per share."""
    rows = []
    for c in range(k):
        c0, c1 = (n * c) // k, (n * (c + 1)) // k
        m = c1 - c0
        rows.append([c0 + (m * s) // p for s in range(p)] + [c1])
    return rows


def _shares(n: int, k: int, p: int):
    for c, row in enumerate(chunk_bounds(n, k, p)):
        for s in range(p):
            yield c, s, row[s], row[s + 1]


# ---------------------------------------------------------------------------
# numpy restatement
# ---------------------------------------------------------------------------
def np_pack(members: list[np.ndarray]) -> np.ndarray:
    """batching.py:76,122: members concatenated in BatchGroup.param_ids order."""
    if not members:
        return np.zeros(0, np.float32)
    return np.concatenate([np.ascontiguousarray(m, np.float32).ravel() for m in members])


def np_unpack(bucket: np.ndarray, shapes: list[tuple]) -> list[np.ndarray]:
    out, off = [], 0
    for shp in shapes:
        n = int(np.prod(shp)) if len(shp) else 1
        out.append(bucket[off:off + n].reshape(shp).copy())
        off += n
    return out


def np_epilogue(epi: int, s: np.ndarray, theta: np.ndarray | None, scale: float, lr: float) -> np.ndarray:
    """SUM: s; SCALE: s*scale; SGD: theta - lr*(s*scale) -- separate fp32 roundings."""
    s = s.astype(np.float32, copy=False)
    if epi == EPI_SUM:
        return s.copy()
    g = (s * np.float32(scale)).astype(np.float32)
    if epi == EPI_SCALE:
        return g
    step = (np.float32(lr) * g).astype(np.float32)
    return (theta.astype(np.float32) - step).astype(np.float32)


def np_allreduce(pattern: int, bufs: list[np.ndarray], k: int, epi: int = EPI_SUM,
                 scale: float = 1.0, lr: float = 0.0, theta: np.ndarray | None = None) -> np.ndarray:
    """Result every worker ends with, summed in the pattern's fixed order."""
    p = len(bufs)
    n = bufs[0].size
    B = [np.array(b, dtype=np.float32, copy=True) for b in bufs]
    out = np.empty(n, np.float32)
    if p == 1:
        return np_epilogue(epi, B[0], theta, scale, lr)
    for c, s, lo, hi in _shares(n, k, p):
        if hi <= lo:
            continue
        sl = slice(lo, hi)
        if pattern == SHUFFLE:
            acc = B[0][sl].copy()
            for q in range(1, p):
                acc = (acc + B[q][sl]).astype(np.float32)
        elif pattern == RING:
            # chain of share s: worker s+1, s+2, ..., s  (collective.py:7-8)
            acc = B[(s + 1) % p][sl].copy()
            for t in range(2, p + 1):
                acc = (acc + B[(s + t) % p][sl]).astype(np.float32)
        elif pattern == HD:
            # recursive halving: at round i (distance d = p >> (i+1)) the
            # block is summed pairwise, lower rank first (collective.py:9-11)
            if p & (p - 1):
                raise ValueError("halving-doubling requires a power-of-two worker count")
            vals = {r: B[r][sl].copy() for r in range(p)}
            d = p >> 1
            while d >= 1:
                nxt = {}
                for r in range(p):
                    q = r ^ d
                    lo_r, hi_r = min(r, q), max(r, q)
                    nxt[r] = (vals[lo_r] + vals[hi_r]).astype(np.float32)
                vals = nxt
                d >>= 1
            acc = vals[s]
        else:
            raise ValueError(f"unknown pattern {pattern}")
        out[sl] = np_epilogue(epi, acc, theta[sl] if theta is not None else None, scale, lr)
    return out


def np_shuffle_lean(bufs: list[np.ndarray], epi: int = EPI_SUM, scale: float = 1.0, lr: float = 0.0,
                    theta: np.ndarray | None = None) -> np.ndarray:
    """np_allreduce(SHUFFLE, ...) without its per-worker copies, for buckets of
    hundreds of MB at p = 8.  In the two-shot pattern every element is reduced
    once, by its shard owner, in ascending rank order (collective.py:12-13,
    98-100), so the values do not depend on the chunk/shard bounds and the
    bucket can be summed whole: acc = g0; acc += g1; ... (each += is one fp32
    rounding, the same as (acc + g).astype(float32))."""
    acc = np.array(bufs[0], dtype=np.float32, copy=True)
    for b in bufs[1:]:
        np.add(acc, b, out=acc)
    return np_epilogue(epi, acc, theta, scale, lr)


# ---------------------------------------------------------------------------
# C restatement (ctypes)
# ---------------------------------------------------------------------------
_C = None


def build(force: bool = False) -> Path:
    if force or not LIB.exists() or LIB.stat().st_mtime < (HERE / "caramel_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def c_lib() -> ctypes.CDLL:
    global _C
    if _C is None:
        build()
        h = ctypes.CDLL(str(LIB))
        P = ctypes.POINTER
        h.oracle_chunk_bounds.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, P(ctypes.c_uint64)]
        h.oracle_allreduce.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                                       P(ctypes.c_void_p), ctypes.c_int, ctypes.c_float, ctypes.c_float,
                                       ctypes.c_void_p, P(ctypes.c_void_p), P(ctypes.c_uint64),
                                       P(ctypes.c_uint64), P(ctypes.c_int)]
        h.oracle_bucket_step.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P(ctypes.c_void_p),
                                         P(ctypes.c_void_p), P(ctypes.c_uint64), ctypes.c_int, ctypes.c_int,
                                         ctypes.c_float, ctypes.c_float, ctypes.c_void_p, ctypes.c_int]
        _C = h
    return _C


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def c_allreduce(pattern: int, bufs: list[np.ndarray], k: int, epi: int = EPI_SUM, scale: float = 1.0,
                lr: float = 0.0, theta: np.ndarray | None = None):
    """(per-worker results, per-stage pulled elements, per-stage reduced elements) of worker 0."""
    h = c_lib()
    p = len(bufs)
    n = bufs[0].size
    B = [np.array(b, dtype=np.float32, copy=True) for b in bufs]
    outs = [np.zeros(n, np.float32) for _ in range(p)]
    bp = (ctypes.c_void_p * p)(*[_ptr(b) for b in B])
    op = (ctypes.c_void_p * p)(*[_ptr(o) for o in outs])
    th = np.ascontiguousarray(theta, np.float32) if theta is not None else None
    xfer = (ctypes.c_uint64 * 64)()
    red = (ctypes.c_uint64 * 64)()
    ns = ctypes.c_int()
    rc = h.oracle_allreduce(pattern, p, n, k, bp, epi, scale, lr, _ptr(th) if th is not None else None,
                            op, xfer, red, ctypes.byref(ns))
    if rc:
        raise ValueError("oracle rejected (pattern, workers, depth)")
    return outs, list(xfer[:ns.value]), list(red[:ns.value])


def c_bucket_step(pattern: int, k: int, grads: list[list[np.ndarray]], params: list[np.ndarray],
                  epi: int, scale: float, lr: float, nthreads: int | None = None,
                  scratch: np.ndarray | None = None) -> None:
    """The full CPU path for one bucket on p = len(grads) simulated workers:
    pack -> collective -> update -> unpack into `params` (in place)."""
    h = c_lib()
    p = len(grads)
    nmem = len(params)
    numels = (ctypes.c_uint64 * nmem)(*[a.size for a in params])
    n = sum(a.size for a in params)
    gp = (ctypes.c_void_p * (p * nmem))(*[_ptr(g) for row in grads for g in row])
    pp = (ctypes.c_void_p * nmem)(*[_ptr(a) for a in params])
    if scratch is None or scratch.size < (p + 1) * n:
        scratch = np.empty((p + 1) * n, np.float32)
    nthreads = nthreads or os.cpu_count() or 1
    rc = h.oracle_bucket_step(pattern, p, k, gp, pp, numels, nmem, epi, scale, lr, _ptr(scratch), nthreads)
    if rc:
        raise ValueError("oracle rejected the bucket step")
