"""ctypes binding of the C ABI in include/caramel.h (libcaramel_b200.so).

This is the only way the package reaches its kernels.  There is no CPU
fallback: if the shared library is missing, :func:`lib` raises
:class:`NativeUnavailable` naming the build command.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "csrc" / "libcaramel_b200.so"
HEADER = HERE.parent / "include" / "caramel.h"

RING, HD, SHUFFLE = 0, 1, 2
EPI_SUM, EPI_SCALE, EPI_SGD = 0, 1, 2
F_PACK, F_UNPACK, F_PARAM_ARENA, F_FLAT, F_AUTO_EPOCH = 1, 2, 4, 8, 16
MANY_FUSED, MANY_FLAGS = 0, 1
ENGINE_CE, ENGINE_SM, ENGINE_GATED = 0, 1, 2
MAX_RANKS = 8
MAX_DEPTH = 8

E_INVAL, E_WORKERS, E_CUDA, E_TIMEOUT, E_STATE = -1, -2, -3, -4, -5


class NativeUnavailable(RuntimeError):
    """The sm_100a library has not been built (run __graft_entry__.build())."""


class CaramelError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"caramel error {code}: {message}")
        self.code = code


class Segment(ctypes.Structure):
    _fields_ = [
        ("grad", ctypes.c_uint64),
        ("param", ctypes.c_uint64),
        ("offset", ctypes.c_uint64),
        ("numel", ctypes.c_uint64),
    ]


class Bucket(ctypes.Structure):
    _fields_ = [
        ("numel", ctypes.c_uint64),
        ("bucket_off", ctypes.c_uint64),
        ("param_off", ctypes.c_uint64),
        ("flag_off", ctypes.c_uint64),
        ("segs", ctypes.c_uint64),
        ("nseg", ctypes.c_int32),
        ("depth", ctypes.c_int32),
        ("pattern", ctypes.c_int32),
        ("epilogue", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
        ("ctas", ctypes.c_int32),
        ("lr", ctypes.c_float),
        ("scale", ctypes.c_float),
    ]


SEGMENT_BYTES = ctypes.sizeof(Segment)

_LIB = None

# name -> (restype, argtypes); exactly the functions include/caramel.h declares
SIGNATURES = {
    "caramel_abi_version": (ctypes.c_int, []),
    "caramel_last_error": (ctypes.c_char_p, []),
    "caramel_chunk_bounds": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                            ctypes.POINTER(ctypes.c_uint64)]),
    "caramel_bucket_layout": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.POINTER(ctypes.c_int32),
                                             ctypes.POINTER(ctypes.c_uint64),
                                             ctypes.POINTER(ctypes.c_uint64)]),
    "caramel_init": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                    ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]),
    "caramel_handle_size": (ctypes.c_int, []),
    "caramel_export": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "caramel_import": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "caramel_arena": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64),
                                     ctypes.POINTER(ctypes.c_uint64)]),
    "caramel_status": (ctypes.c_int, [ctypes.c_void_p]),
    "caramel_poll": (ctypes.c_int, [ctypes.c_void_p]),
    "caramel_set_timeout_ms": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64]),
    "caramel_finalize": (ctypes.c_int, [ctypes.c_void_p]),
    "caramel_pack": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p,
                                    ctypes.c_void_p]),
    "caramel_unpack": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p,
                                      ctypes.c_int32, ctypes.c_void_p]),
    "caramel_epoch_advance": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "caramel_allreduce": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Bucket), ctypes.c_uint32,
                                         ctypes.c_void_p]),
    "caramel_allreduce_update": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Bucket), ctypes.c_uint32,
                                                ctypes.c_void_p]),
    "caramel_allreduce_many": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Bucket), ctypes.c_int32,
                                              ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int32,
                                              ctypes.c_int32, ctypes.c_uint32, ctypes.c_void_p]),
    "caramel_allreduce_ce": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Bucket), ctypes.c_int32,
                                            ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p]),
    "caramel_allreduce_gated": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Bucket), ctypes.c_int32,
                                               ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p]),
    "caramel_ce_available": (ctypes.c_int, [ctypes.c_void_p]),
    "caramel_ce_submit": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Bucket), ctypes.c_int32, ctypes.c_uint32,
                                         ctypes.c_uint32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p]),
    "caramel_ce_flush": (ctypes.c_int, [ctypes.c_void_p]),
    "caramel_mc_available": (ctypes.c_int, [ctypes.c_void_p]),
    "caramel_mc_create": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_char_p]),
    "caramel_mc_exchange": (ctypes.c_int, [ctypes.c_void_p]),
    "caramel_mc_bind": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)]),
    "caramel_allreduce_nvls": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Bucket), ctypes.c_uint32,
                                              ctypes.c_void_p]),
}


def lib() -> ctypes.CDLL:
    """Load libcaramel_b200.so (once).  Raises NativeUnavailable if absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = Path(os.environ.get("CARAMEL_LIB", LIB_PATH))
    if not path.exists():
        raise NativeUnavailable(
            f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc -gencode arch=compute_100a,code=sm_100a).  There is no CPU fallback."
        )
    handle = ctypes.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = handle
    return handle


def last_error() -> str:
    msg = lib().caramel_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    if rc != 0:
        raise CaramelError(rc, last_error())


def chunk_bounds(numel: int, depth: int, workers: int) -> list[list[int]]:
    """Absolute element bounds per chunk: row c = share starts + chunk end."""
    out = (ctypes.c_uint64 * (depth * (workers + 1)))()
    check(lib().caramel_chunk_bounds(numel, depth, workers, out))
    return [list(out[c * (workers + 1):(c + 1) * (workers + 1)]) for c in range(depth)]


def bucket_layout(numel: int, depth: int, pattern: int, world: int) -> tuple[int, int, int]:
    """(ctas, bucket_bytes, flag_bytes) for one bucket; identical on every rank."""
    ctas = ctypes.c_int32()
    bbytes = ctypes.c_uint64()
    fbytes = ctypes.c_uint64()
    check(lib().caramel_bucket_layout(numel, depth, pattern, world, ctypes.byref(ctas),
                                      ctypes.byref(bbytes), ctypes.byref(fbytes)))
    return ctas.value, bbytes.value, fbytes.value


def flag_bytes_for(depth: int, ctas: int, pattern: int, world: int) -> int:
    """Flag-block bytes for an explicit CTA count (mirrors caramel.cu nslots)."""
    if world == 1:
        return 0
    if pattern == SHUFFLE:
        ns = 2
    elif pattern == RING:
        ns = 2 * world
    else:
        ns = 2 * (world - 1).bit_length() + 2
    return (depth * ctas * ns * world * 4 + 255) & ~255
