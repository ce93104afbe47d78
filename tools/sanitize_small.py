"""Small invocations of every kernel family for compute-sanitizer (racecheck /
synccheck / memcheck): the world=1 TMA update (k_local_flat_tma), the TMA
pack/unpack (k_pack_tma), an emulated 2-rank two-shot (k_collective pull + LL,
cooperative), an emulated bucket list (k_shuffle_fused, k_collective_many) and,
with CARAMEL_PUSH=1 in the environment, the TMA push engine (k_push)."""
import ctypes, os, sys
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle")); sys.path.insert(0, str(ROOT / "tests"))
import oracle as O
from paper_2004_14020_b200 import _native as N, comm

dev = torch.device("cuda:0")
st = torch.cuda.current_stream().cuda_stream

# 1. world = 1: Aggregator step (k_local_flat_tma with grads="flat")
from test_gpu_robustness import test_close_returns_torch_owned_storage
test_close_returns_torch_owned_storage()
print("world=1 step ok", flush=True)

# 2. pack / unpack through the TMA tiles, aligned and misaligned members
from test_gpu_kernels import test_pack_unpack_standalone
test_pack_unpack_standalone()
print("pack/unpack ok", flush=True)

# 3. emulated two-shot: a bucket over the LL cutoff and one under it
from test_gpu_kernels import run_emulated, assert_bitexact, SHAPES_SMALL, SHAPES_LARGE
assert_bitexact(run_emulated(N.SHUFFLE, 2, 2, SHAPES_LARGE, N.EPI_SGD, ctas=8))
assert_bitexact(run_emulated(N.SHUFFLE, 2, 1, SHAPES_SMALL, N.EPI_SUM, ctas=2))
print("emulated two-shot ok", flush=True)

# 4. emulated lists (fused and flags)
from test_gpu_kernels import run_emulated_many, MANY_BUCKETS, MANY_DEPTHS
run_emulated_many(N.SHUFFLE, 2, MANY_BUCKETS, MANY_DEPTHS, N.EPI_SGD, param_arena=True, epochs=1)
run_emulated_many(N.SHUFFLE, 2, MANY_BUCKETS, MANY_DEPTHS, N.EPI_SGD, param_arena=True, epochs=1, mode=N.MANY_FLAGS)
print("emulated lists ok", flush=True)
