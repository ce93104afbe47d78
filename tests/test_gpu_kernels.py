"""Kernel parity on one GPU: the sm_100a collectives over emulated ranks
(cooperative launch, every rank's arena on one device) against the CPU
oracle, bit-exact, through the C ABI."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

SHAPES_SMALL = [(3, 5), (129,), (64, 7), (1,), (1000,)]
SHAPES_RAGGED = [(1,), (2,), (3,), (5, 5), (7,), (4097,), (1,), (33, 3)]
SHAPES_LARGE = [(512, 1024), (3,), (256, 257), (1000,)]


def _native():
    from paper_2004_14020_b200 import _native as N
    from paper_2004_14020_b200 import comm

    return N, comm


def _members(dev, shapes, arrays, misalign: bool):
    """Device tensors holding `arrays`; with misalign=True they are carved out
    of one buffer at odd element offsets (not 16-byte aligned)."""
    if not misalign:
        return [torch.from_numpy(a.copy()).to(dev) for a in arrays]
    total = sum(a.size for a in arrays) + 2 * len(arrays) + 4
    big = torch.zeros(total, device=dev)
    out, off = [], 1
    for a in arrays:
        t = big[off:off + a.size].view(a.shape)
        t.copy_(torch.from_numpy(a))
        out.append(t)
        off += a.size + 1 + (off % 2)
    return out


def _flat(ts):
    return torch.cat([t.reshape(-1) for t in ts]).cpu().numpy()


def run_emulated(pattern, p, depth, shapes, epi, *, unpack=True, param_arena=False, epochs=1,
                 ctas=None, misalign=False, seed=0, int_valued=False, auto_epoch=False):
    N, comm = _native()
    dev = torch.device("cuda:0")
    numel = sum(int(np.prod(s)) for s in shapes)
    c0, bbytes, _ = N.bucket_layout(numel, depth, pattern, p)
    ctas = min(ctas or c0, max(1, 96 // p))
    fbytes = N.flag_bytes_for(depth, ctas, pattern, p)
    flag_off = (bbytes + 255) // 256 * 256
    ctx = comm.Context(0, p, arena_bytes=flag_off + fbytes, param_bytes=(4 * numel if param_arena else 0),
                       nlocal=p)
    rng = np.random.default_rng(seed)
    lr, scale = 0.125, 1.0 / p
    theta = [rng.standard_normal(s).astype(np.float32) for s in shapes]
    th_dev = [_members(dev, shapes, theta, misalign) for _ in range(p)]
    if param_arena:
        for r in range(p):
            ctx.arena_view(r, 0, numel, param=True).copy_(torch.from_numpy(O.np_pack(theta)).to(dev))
    stream = torch.cuda.current_stream().cuda_stream
    flags = N.F_PACK | (N.F_UNPACK if unpack else 0) | (N.F_PARAM_ARENA if param_arena else 0)
    flags |= N.F_AUTO_EPOCH if auto_epoch else 0
    results = []
    for e in range(1, epochs + 1):
        if int_valued:
            grads = [[rng.integers(-1024, 1025, size=s).astype(np.float32) for s in shapes] for _ in range(p)]
        else:
            grads = [[rng.standard_normal(s).astype(np.float32) for s in shapes] for _ in range(p)]
        g_dev = [_members(dev, shapes, grads[r], misalign) for r in range(p)]
        table = comm.segment_table(
            [comm.segments_for(g_dev[r], None if param_arena else th_dev[r]) for r in range(p)], dev)
        b = comm.make_bucket(numel, 0, flag_off, depth=depth, pattern=pattern, epilogue=epi, flags=flags,
                             ctas=ctas, segs=table, nseg=len(shapes), lr=lr, scale=scale)
        ctx.allreduce(b, 0 if auto_epoch else e, stream)
        ctx.status()
        torch.cuda.synchronize()
        theta_flat = O.np_pack(theta)
        want = O.np_allreduce(pattern, [O.np_pack(row) for row in grads], depth, epi, scale, lr, theta_flat)
        got = []
        for r in range(p):
            if epi == N.EPI_SGD and param_arena:
                got.append(ctx.arena_view(r, 0, numel, param=True).cpu().numpy().copy())
            elif unpack:
                got.append(_flat(th_dev[r] if epi == N.EPI_SGD else g_dev[r]))
            else:
                out_off = 0 if (pattern == N.SHUFFLE or p == 1) else 4 * ((numel + 3) // 4 * 4)
                got.append(ctx.arena_view(r, out_off, numel).cpu().numpy().copy())
        results.append((want, got))
        if epi == N.EPI_SGD:
            theta = O.np_unpack(want, shapes)
    ctx.close()
    return results


def assert_bitexact(results):
    for want, got in results:
        for r, g in enumerate(got):
            bad = np.nonzero(g.view(np.uint32) != want.view(np.uint32))[0]
            assert bad.size == 0, f"rank {r}: {bad.size} mismatches, first at {bad[:8]}: {g[bad[:4]]} vs {want[bad[:4]]}"


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("depth", [1, 3, 8])
def test_shuffle_sum_bitexact(p, depth):
    N, _ = _native()
    assert_bitexact(run_emulated(N.SHUFFLE, p, depth, SHAPES_RAGGED, N.EPI_SUM))


# 16K-64K elements: the upper range of the LL (flag-in-word) protocol
SHAPES_MID = [(128, 300), (3,), (7, 1111), (1,)]         # 46,181 elements
SHAPES_LL_EDGE = [(65536,)]                                # exactly the LL cutoff


@pytest.mark.parametrize("shapes", ["mid", "edge"])
@pytest.mark.parametrize("p", [2, 4, 8])
def test_shuffle_mid_size_buckets_bitexact(shapes, p):
    N, _ = _native()
    sh = SHAPES_MID if shapes == "mid" else SHAPES_LL_EDGE
    assert_bitexact(run_emulated(N.SHUFFLE, p, 1, sh, N.EPI_SGD, epochs=3))


@pytest.mark.parametrize("pattern", ["ring", "hd", "shuffle"])
@pytest.mark.parametrize("p", [2, 4, 8])
def test_patterns_sgd_fused_update_bitexact(pattern, p):
    N, _ = _native()
    pat = {"ring": N.RING, "hd": N.HD, "shuffle": N.SHUFFLE}[pattern]
    assert_bitexact(run_emulated(pat, p, 2, SHAPES_SMALL, N.EPI_SGD))


@pytest.mark.parametrize("p", [3, 5, 6])
def test_ring_non_power_of_two(p):
    N, _ = _native()
    assert_bitexact(run_emulated(N.RING, p, 3, SHAPES_RAGGED, N.EPI_SCALE))


@pytest.mark.parametrize("pattern", ["ring", "hd", "shuffle"])
def test_result_in_bucket_without_unpack(pattern):
    N, _ = _native()
    pat = {"ring": N.RING, "hd": N.HD, "shuffle": N.SHUFFLE}[pattern]
    assert_bitexact(run_emulated(pat, 4, 4, SHAPES_SMALL, N.EPI_SUM, unpack=False))


@pytest.mark.parametrize("pattern", ["ring", "hd", "shuffle"])
def test_param_arena_update(pattern):
    N, _ = _native()
    pat = {"ring": N.RING, "hd": N.HD, "shuffle": N.SHUFFLE}[pattern]
    assert_bitexact(run_emulated(pat, 4, 2, SHAPES_LARGE, N.EPI_SGD, param_arena=True, epochs=2))


@pytest.mark.parametrize("pattern", ["ring", "hd", "shuffle"])
def test_epochs_reuse_flags(pattern):
    N, _ = _native()
    pat = {"ring": N.RING, "hd": N.HD, "shuffle": N.SHUFFLE}[pattern]
    assert_bitexact(run_emulated(pat, 8, 3, SHAPES_SMALL, N.EPI_SGD, epochs=4, ctas=3))


@pytest.mark.parametrize("pattern", ["ring", "hd", "shuffle"])
@pytest.mark.parametrize("shapes", [SHAPES_SMALL, [(300, 1000)], SHAPES_LARGE], ids=["ll", "ll128", "plain"])
def test_auto_epoch_one_kernel_per_call(pattern, shapes):
    """CARAMEL_F_AUTO_EPOCH: epoch 0, the device counter + 1, advanced by the
    launch's last CTA -- consecutive calls with no caramel_epoch_advance
    between them stay bit-exact (each call's flags carry a fresh epoch)."""
    N, _ = _native()
    pat = {"ring": N.RING, "hd": N.HD, "shuffle": N.SHUFFLE}[pattern]
    assert_bitexact(run_emulated(pat, 4, 2, shapes, N.EPI_SGD, epochs=4, auto_epoch=True))


def test_auto_epoch_is_rejected_where_it_cannot_apply():
    N, comm = _native()
    import ctypes

    ctx = comm.Context(0, 2, arena_bytes=1 << 20, nlocal=2)
    b = comm.make_bucket(1000, 0, 1 << 19, pattern=N.SHUFFLE, epilogue=N.EPI_SUM, flags=N.F_AUTO_EPOCH, ctas=2)
    stream = torch.cuda.current_stream().cuda_stream
    with pytest.raises(RuntimeError, match="AUTO_EPOCH"):
        ctx.allreduce(b, 3, stream)  # an explicit epoch with the flag
    host = (N.Bucket * 1)(b)
    dl = torch.frombuffer(bytearray(bytes(host)), dtype=torch.uint8).to("cuda:0")
    pre = torch.tensor([0, 1000], dtype=torch.int64, device="cuda:0")
    spre = torch.tensor([0, 0], dtype=torch.int64, device="cuda:0")
    rc = N.lib().caramel_allreduce_many(ctx._ctx, host, 1, dl.data_ptr(), pre.data_ptr(), spre.data_ptr(), 0,
                                        N.MANY_FLAGS, 0, ctypes.c_void_p(stream))
    assert rc != 0 and b"AUTO_EPOCH" in N.lib().caramel_last_error()
    ctx.close()


def test_misaligned_members():
    N, _ = _native()
    assert_bitexact(run_emulated(N.SHUFFLE, 4, 3, SHAPES_RAGGED, N.EPI_SGD, misalign=True))
    assert_bitexact(run_emulated(N.RING, 4, 3, SHAPES_RAGGED, N.EPI_SUM, misalign=True))


def test_large_bucket_many_ctas():
    N, _ = _native()
    assert_bitexact(run_emulated(N.SHUFFLE, 2, 8, SHAPES_LARGE, N.EPI_SGD, ctas=40))


def test_integer_valued_order_independent_across_patterns():
    """Mode A inputs (integers in [-2^10, 2^10]): every summation order is
    exact, so all three patterns must agree with each other bit for bit."""
    N, _ = _native()
    outs = [run_emulated(pat, 4, 2, SHAPES_SMALL, N.EPI_SUM, int_valued=True, seed=5)[0][1][0]
            for pat in (N.RING, N.HD, N.SHUFFLE)]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])


@pytest.mark.parametrize("epi", [0, 1, 2])
def test_single_rank_fused_path(epi):
    assert_bitexact(run_emulated(2, 1, 1, SHAPES_RAGGED, epi, misalign=True))


def test_pack_unpack_standalone():
    N, comm = _native()
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(3)
    for misalign in (False, True):
        arrays = [rng.standard_normal(s).astype(np.float32) for s in SHAPES_RAGGED + SHAPES_LARGE]
        shapes = [a.shape for a in arrays]
        ts = _members(dev, shapes, arrays, misalign)
        numel = sum(a.size for a in arrays)
        table = comm.segment_table([comm.segments_for(ts)], dev)
        bucket = torch.empty(numel + 4, device=dev)
        stream = torch.cuda.current_stream().cuda_stream
        comm.pack(table, len(ts), numel, bucket.data_ptr(), stream)
        torch.cuda.synchronize()
        assert np.array_equal(bucket[:numel].cpu().numpy(), O.np_pack(arrays))
        bucket.mul_(-2.0)
        comm.unpack(table, len(ts), numel, bucket.data_ptr(), False, stream)
        torch.cuda.synchronize()
        for t, a in zip(ts, arrays):
            assert np.array_equal(t.cpu().numpy(), -2.0 * a)


def test_errors_are_reported_not_raised_in_c():
    N, comm = _native()
    ctx = comm.Context(0, 4, arena_bytes=1 << 20, nlocal=4)
    b = comm.make_bucket(1024, 0, 1 << 19, depth=9, ctas=1)
    with pytest.raises(N.CaramelError, match="depth"):
        ctx.allreduce(b, 1, torch.cuda.current_stream().cuda_stream)
    ctx.close()
    ctx3 = comm.Context(0, 3, arena_bytes=1 << 20, nlocal=3)
    b = comm.make_bucket(1024, 0, 1 << 19, pattern=N.HD, ctas=1)
    with pytest.raises(N.CaramelError, match="power-of-two"):
        ctx3.allreduce(b, 1, torch.cuda.current_stream().cuda_stream)
    ctx3.close()


def run_emulated_many(pattern, p, bucket_shapes, depths, epi, *, param_arena=False, epochs=2, seed=11, mode=0):
    """Several buckets in ONE launch (caramel_allreduce_many), device epoch
    counter; every bucket checked against the oracle on every rank."""
    import ctypes

    N, comm = _native()
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(seed)
    lr = 0.25
    # layout
    off, poff, specs = 0, 0, []
    for shapes, depth in zip(bucket_shapes, depths):
        numel = sum(int(np.prod(s)) for s in shapes)
        c0, bbytes, _ = N.bucket_layout(numel, depth, pattern, p)
        ctas = min(c0, max(1, 64 // p))
        fbytes = N.flag_bytes_for(depth, ctas, pattern, p)
        boff = off
        foff = (boff + bbytes + 255) // 256 * 256
        off = (foff + fbytes + 255) // 256 * 256
        specs.append((shapes, depth, numel, ctas, boff, foff, poff))
        poff = (poff + 4 * numel + 255) // 256 * 256
    ctx = comm.Context(0, p, arena_bytes=off, param_bytes=poff if param_arena else 0, nlocal=p)
    thetas = [[rng.standard_normal(s).astype(np.float32) for s in sp[0]] for sp in specs]
    th_dev = [[_members(dev, sp[0], thetas[i], False) for _ in range(p)] for i, sp in enumerate(specs)]
    if param_arena:
        for i, sp in enumerate(specs):
            for r in range(p):
                ctx.arena_view(r, sp[6], sp[2], param=True).copy_(torch.from_numpy(O.np_pack(thetas[i])).to(dev))
    stream = torch.cuda.current_stream().cuda_stream
    flags = N.F_PACK | (N.F_PARAM_ARENA if param_arena else N.F_UNPACK)
    for e in range(epochs):
        grads, g_devs, descs, tables = [], [], [], []
        for i, (shapes, depth, numel, ctas, boff, foff, pof) in enumerate(specs):
            gr = [[rng.standard_normal(s).astype(np.float32) for s in shapes] for _ in range(p)]
            gd = [_members(dev, shapes, gr[r], False) for r in range(p)]
            tab = comm.segment_table([comm.segments_for(gd[r], None if param_arena else th_dev[i][r])
                                      for r in range(p)], dev)
            grads.append(gr)
            g_devs.append(gd)
            tables.append(tab)
            descs.append(comm.make_bucket(numel, boff, foff, depth=depth, pattern=pattern, epilogue=epi,
                                          flags=flags, ctas=ctas, segs=tab, nseg=len(shapes), param_off=pof,
                                          lr=lr, scale=1.0 / p))
        host = (N.Bucket * len(descs))(*descs)
        dev_list = torch.frombuffer(bytearray(bytes(host)), dtype=torch.uint8).to(dev)
        prefix = torch.tensor(np.concatenate([[0], np.cumsum([sp[2] for sp in specs])]), dtype=torch.int64,
                              device=dev)
        segprefix = torch.tensor(np.concatenate([[0], np.cumsum([len(sp[0]) for sp in specs])]),
                                 dtype=torch.int64, device=dev)
        N.check(N.lib().caramel_epoch_advance(ctx._ctx, ctypes.c_void_p(stream)))
        N.check(N.lib().caramel_allreduce_many(ctx._ctx, host, len(descs), dev_list.data_ptr(), prefix.data_ptr(),
                                               segprefix.data_ptr(), 0, mode, 0, ctypes.c_void_p(stream)))
        ctx.status()
        torch.cuda.synchronize()
        for i, (shapes, depth, numel, ctas, boff, foff, pof) in enumerate(specs):
            want = O.np_allreduce(pattern, [O.np_pack(row) for row in grads[i]], depth, epi, 1.0 / p, lr,
                                  O.np_pack(thetas[i]))
            for r in range(p):
                if epi == N.EPI_SGD and param_arena:
                    got = ctx.arena_view(r, pof, numel, param=True).cpu().numpy()
                elif epi == N.EPI_SGD:
                    got = _flat(th_dev[i][r])
                else:
                    got = _flat(g_devs[i][r])
                assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (i, r, e)
            if epi == N.EPI_SGD:
                thetas[i] = O.np_unpack(want, shapes)
    ctx.close()


MANY_BUCKETS = [SHAPES_RAGGED, [(129,)], SHAPES_SMALL, [(1,)], SHAPES_LARGE, [(7, 7), (3,)]]
MANY_DEPTHS = [3, 1, 2, 1, 8, 2]


@pytest.mark.parametrize("p", [1, 2, 4, 8])
@pytest.mark.parametrize("pattern", ["shuffle", "ring", "hd"])
def test_many_buckets_one_launch(p, pattern):
    N, _ = _native()
    pat = {"ring": N.RING, "hd": N.HD, "shuffle": N.SHUFFLE}[pattern]
    run_emulated_many(pat, p, MANY_BUCKETS, MANY_DEPTHS, N.EPI_SGD, param_arena=True)


@pytest.mark.parametrize("p", [2, 3, 8])
def test_many_buckets_flags_mode(p):
    N, _ = _native()
    run_emulated_many(N.SHUFFLE, p, MANY_BUCKETS, MANY_DEPTHS, N.EPI_SGD, param_arena=True, mode=N.MANY_FLAGS)
    run_emulated_many(N.SHUFFLE, p, MANY_BUCKETS, MANY_DEPTHS, N.EPI_SUM, mode=N.MANY_FLAGS)


@pytest.mark.parametrize("epi", [0, 1, 2])
def test_many_buckets_unpack_modes(epi):
    N, _ = _native()
    run_emulated_many(N.SHUFFLE, 4, MANY_BUCKETS, MANY_DEPTHS, epi, param_arena=False)
    run_emulated_many(N.SHUFFLE, 1, MANY_BUCKETS, MANY_DEPTHS, epi, param_arena=False)


# 64K < n <= 512K elements: the LL128 protocol (128-byte lines: 30 floats + an epoch flag)
SHAPES_LL128 = [(3, 33331), (7,), (1,), (250, 401)]      # 200,107 elements: a ragged last line
SHAPES_LL128_EDGE = [(1 << 19,)]                          # exactly the LL128 cutoff


@pytest.mark.parametrize("p", [2, 3, 5, 8])
def test_ll128_bitexact(p):
    N, _ = _native()
    assert_bitexact(run_emulated(N.SHUFFLE, p, 2, SHAPES_LL128, N.EPI_SGD, epochs=3))
    assert_bitexact(run_emulated(N.SHUFFLE, p, 1, SHAPES_LL128, N.EPI_SUM, misalign=True, epochs=2))


@pytest.mark.parametrize("p", [2, 4])
def test_ll128_cutoff_and_param_arena(p):
    N, _ = _native()
    assert_bitexact(run_emulated(N.SHUFFLE, p, 1, SHAPES_LL128_EDGE, N.EPI_SGD, param_arena=True, epochs=2))
    assert_bitexact(run_emulated(N.SHUFFLE, p, 3, SHAPES_LL128_EDGE, N.EPI_SCALE, unpack=False))
