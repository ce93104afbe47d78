"""Parity at the BASELINE.json sizes, on one GPU, bit-exact against the oracle.

Every rank of a p-rank job is emulated on cuda:0 (all ranks' arenas on one
device, cooperative launch), so these run on the driver's single-GPU test box.
Covered here, all through the C ABI:

* the full launch-ordered bucket plans of the four BASELINE gradient sets
  (ResNet-50, Inception-v3, AlexNet, VGG-16) at p = 2, 4, 8, as
  ONE caramel_allreduce_many launch in both list modes -- CARAMEL_MANY_FUSED
  (k_shuffle_fused: flat phases + grid barriers) and CARAMEL_MANY_FLAGS
  (k_collective_many: per-(bucket, chunk, tile) flags) -- with the
  production layout (gradients in the bucket arena, SGD fused, results
  stored into every replica's parameter arena) and with the packed layout;
* single buckets of 4 MiB and 64 MiB and VGG-16's fc6 (102,760,448
  elements, the largest tensor of any config) at depth 8, through
  k_collective (per-chunk flags, chunk-parallel CTA groups), in the three
  patterns.

The oracle is oracle.np_shuffle_lean / np_allreduce (the CPU restatement of
collective.py's pattern semantics); plans come from this package's planner,
whose bucket membership, order and depths are pinned to the reference by
tests/test_plan_parity.py.
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

NVLINK_MODEL = (10.0, 1.0 / 460e3)  # SURVEY §8a "NVLink-ish" network model (threshold 6.9 MB)
LR = 0.1


def _plan(model: str, p: int):
    from paper_2004_14020_b200 import gradsets
    from paper_2004_14020_b200.collective import Pattern, ReduceModel
    from paper_2004_14020_b200.costmodel import NetworkModel
    from paper_2004_14020_b200.executor import lower
    from paper_2004_14020_b200.pipeline import run_pipeline
    from paper_2004_14020_b200.sim import SimConfig

    tensors = gradsets.gradient_set(model)
    art = run_pipeline(gradsets.layered_chain_dag(model),
                       SimConfig(workers=max(2, p), network=NetworkModel(*NVLINK_MODEL),
                                 reduce=ReduceModel(400.0, 10.0)))
    numels = {gradsets.param_id(i, len(tensors)): t.numel for i, t in enumerate(tensors)}
    # all p emulated ranks' CTAs must be co-resident under the cooperative
    # launch (the list kernels run one 512-thread CTA per SM): at most 148/p
    # CTAs per rank.  Tile counts are a launch parameter; the element
    # ownership (chunk/shard rule) does not depend on them.
    return lower(art, numels, p, Pattern.SHUFFLE, max_ctas=148 // p)


def _device_list(descs, dev):
    from paper_2004_14020_b200 import _native as N

    host = (N.Bucket * len(descs))(*descs)
    dlist = torch.frombuffer(bytearray(bytes(host)), dtype=torch.uint8).to(dev)
    pre = torch.tensor(np.concatenate([[0], np.cumsum([d.numel for d in descs])]), dtype=torch.int64, device=dev)
    spre = torch.tensor(np.concatenate([[0], np.cumsum([d.nseg for d in descs])]), dtype=torch.int64, device=dev)
    return host, dlist, pre, spre


def run_plan(model: str, p: int, mode: int, packed: bool = False, epochs: int = 2, seed: int = 0) -> None:
    """One emulated p-rank job over the whole plan of `model`; every bucket of
    every rank checked bit for bit after every epoch."""
    from paper_2004_14020_b200 import _native as N
    from paper_2004_14020_b200 import comm

    dev = torch.device("cuda:0")
    plan = _plan(model, p)
    ctx = comm.Context(0, p, arena_bytes=plan.arena_bytes, param_bytes=plan.param_bytes, nlocal=p)
    gens = [torch.Generator(device=dev).manual_seed(1000 * seed + r) for r in range(p)]
    tgen = torch.Generator(device=dev).manual_seed(7)
    # identical parameters on every replica: N(0, 0.01)
    theta0 = torch.empty(plan.param_bytes // 4, device=dev).normal_(0.0, 0.01, generator=tgen)
    for r in range(p):
        ctx.arena_view(r, 0, plan.param_bytes // 4, param=True).copy_(theta0)
    flat = None
    if packed:  # the "flat" gradient layout: one buffer per rank, PACK gathers it (nseg == 1 per bucket)
        flat = [torch.empty(plan.param_bytes // 4, device=dev) for _ in range(p)]
    stream = torch.cuda.current_stream().cuda_stream
    theta = {b.index: theta0[b.param_off // 4:b.param_off // 4 + b.numel].cpu().numpy() for b in plan.buckets}
    for e in range(epochs):
        descs, tables = [], []
        for b in plan.buckets:
            for r in range(p):
                if packed:
                    flat[r][b.param_off // 4:b.param_off // 4 + b.numel].normal_(generator=gens[r])
                else:
                    ctx.arena_view(r, b.bucket_off, b.numel).normal_(generator=gens[r])
            flags = N.F_PARAM_ARENA
            tab, nseg = None, 0
            if packed:
                segs = [[comm.SegmentSpec(flat[r].data_ptr() + b.param_off, 0, 0, b.numel)] for r in range(p)]
                tab, nseg = comm.segment_table(segs, dev), 1
                tables.append(tab)
                flags |= N.F_PACK | N.F_FLAT
            descs.append(comm.make_bucket(b.numel, b.bucket_off, b.flag_off, depth=b.depth, pattern=N.SHUFFLE,
                                          epilogue=N.EPI_SGD, flags=flags, ctas=b.ctas, segs=tab, nseg=nseg,
                                          param_off=b.param_off, lr=LR, scale=1.0 / p))
        host, dlist, pre, spre = _device_list(descs, dev)
        N.check(N.lib().caramel_epoch_advance(ctx._ctx, ctypes.c_void_p(stream)))
        N.check(N.lib().caramel_allreduce_many(ctx._ctx, host, len(descs), dlist.data_ptr(), pre.data_ptr(),
                                               spre.data_ptr(), 0, mode, 0, ctypes.c_void_p(stream)))
        ctx.status()
        torch.cuda.synchronize()
        for b in plan.buckets:
            if packed:
                bufs = [flat[r][b.param_off // 4:b.param_off // 4 + b.numel].cpu().numpy() for r in range(p)]
            else:  # SGD into the parameter arena leaves the gradients in place
                bufs = [ctx.arena_view(r, b.bucket_off, b.numel).cpu().numpy() for r in range(p)]
            want = O.np_shuffle_lean(bufs, O.EPI_SGD, 1.0 / p, LR, theta[b.index])
            del bufs
            for r in range(p):
                got = ctx.arena_view(r, b.param_off, b.numel, param=True).cpu().numpy()
                bad = np.nonzero(got.view(np.uint32) != want.view(np.uint32))[0]
                assert bad.size == 0, (f"{model} p={p} mode={mode} epoch={e} bucket {b.index} ({b.group_id}, "
                                       f"{b.numel} elems, depth {b.depth}) rank {r}: {bad.size} mismatches, "
                                       f"first {bad[:5]}")
            theta[b.index] = want
    ctx.close()


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("model", ["resnet50", "inception_v3", "alexnet", "vgg16"])
def test_full_plan_fused_list(model, p):
    from paper_2004_14020_b200 import _native as N

    run_plan(model, p, N.MANY_FUSED, epochs=1 if (model == "vgg16" and p == 8) else 2)


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("model", ["resnet50", "inception_v3", "alexnet", "vgg16"])
def test_full_plan_flags_list(model, p):
    from paper_2004_14020_b200 import _native as N

    run_plan(model, p, N.MANY_FLAGS, epochs=1 if (model == "vgg16" and p == 8) else 2)


@pytest.mark.parametrize("model,p,mode", [("resnet50", 4, 0), ("inception_v3", 8, 1), ("alexnet", 2, 0)])
def test_full_plan_packed_layout(model, p, mode):
    run_plan(model, p, mode, packed=True)


FC6 = 102_760_448  # VGG-16 classifier.0.weight, 4096 x 25088


def run_single(numel: int, p: int, depth: int, pattern: int, epochs: int = 2, epi: int = O.EPI_SGD) -> None:
    """One bucket through k_collective (caramel_allreduce[_update]), zero-copy
    input, result in the parameter arena (SGD) or in place (SUM)."""
    from paper_2004_14020_b200 import _native as N
    from paper_2004_14020_b200 import comm

    dev = torch.device("cuda:0")
    ctas, bbytes, _ = N.bucket_layout(numel, depth, pattern, p)
    ctas = min(ctas, 148 // p)  # co-resident under the cooperative (emulated) launch: one CTA per SM
    fbytes = N.flag_bytes_for(depth, ctas, pattern, p)
    flag_off = (bbytes + 255) // 256 * 256
    sgd = epi == O.EPI_SGD
    ctx = comm.Context(0, p, arena_bytes=flag_off + fbytes, param_bytes=4 * numel if sgd else 0, nlocal=p)
    gens = [torch.Generator(device=dev).manual_seed(77 + r) for r in range(p)]
    theta = None
    if sgd:
        t0 = torch.empty(numel, device=dev).normal_(0.0, 0.01, generator=torch.Generator(device=dev).manual_seed(7))
        for r in range(p):
            ctx.arena_view(r, 0, numel, param=True).copy_(t0)
        theta = t0.cpu().numpy()
    # ring / hd keep the result in a second half of the bucket region
    out_off = 0 if (pattern == N.SHUFFLE or sgd) else 4 * ((numel + 3) // 4 * 4)
    stream = torch.cuda.current_stream().cuda_stream
    b = comm.make_bucket(numel, 0, flag_off, depth=depth, pattern=pattern, epilogue=epi,
                         flags=N.F_PARAM_ARENA if sgd else 0, ctas=ctas, lr=LR, scale=1.0 / p)
    for e in range(1, epochs + 1):
        for r in range(p):
            ctx.arena_view(r, 0, numel).normal_(generator=gens[r])
        bufs = [ctx.arena_view(r, 0, numel).cpu().numpy() for r in range(p)]
        ctx.allreduce(b, e, stream)
        ctx.status()
        torch.cuda.synchronize()
        if pattern == N.SHUFFLE:
            want = O.np_shuffle_lean(bufs, epi, 1.0 / p, LR, theta)
        else:
            want = O.np_allreduce(pattern, bufs, depth, epi, 1.0 / p, LR, theta)
        del bufs
        for r in range(p):
            got = (ctx.arena_view(r, 0, numel, param=True) if sgd else ctx.arena_view(r, out_off, numel)).cpu().numpy()
            bad = np.nonzero(got.view(np.uint32) != want.view(np.uint32))[0]
            assert bad.size == 0, f"n={numel} p={p} depth={depth} pattern={pattern} epoch={e} rank {r}: {bad[:5]}"
        theta = want if sgd else theta
    ctx.close()


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("mib", [4, 64])
def test_single_bucket_shuffle(mib, p):
    from paper_2004_14020_b200.collective import adaptive_depth

    n = mib * (1 << 20) // 4
    run_single(n, p, adaptive_depth(4 * n, 6_900_001), O.SHUFFLE)
    run_single(n, p, 8, O.SHUFFLE, epochs=1)


@pytest.mark.parametrize("p", [2, 4, 8])
def test_vgg_fc6_depth8(p):
    """The largest tensor of any BASELINE config, split at the maximum depth
    (adaptive_depth(411,041,792 B, 6.9 MB) = 8)."""
    from paper_2004_14020_b200.collective import adaptive_depth

    assert adaptive_depth(4 * FC6, 6_900_001) == 8
    run_single(FC6, p, 8, O.SHUFFLE, epochs=2 if p < 8 else 1)


@pytest.mark.parametrize("pattern,p", [("ring", 4), ("hd", 8), ("ring", 3)])
def test_single_bucket_ring_hd_64mib(pattern, p):
    n = 64 * (1 << 20) // 4 + 3  # ragged: shard bounds off the 4-element grid
    run_single(n, p, 4, {"ring": O.RING, "hd": O.HD}[pattern], epochs=2, epi=O.EPI_SUM)
