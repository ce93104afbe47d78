"""Emulated-rank check of the opt-in push engine (CARAMEL_PUSH=1, read at library
load, hence a separate process: tests/test_gpu_robustness.py runs it).  Single
buckets and bucket lists of every protocol (LL, one-shot, two-shot), p ranks on
cuda:0, bit-exact against the oracle; after a watchdog timeout the flag words
of every rank are printed.  Prints "MISMATCH" / "TIMEOUT" on failure."""
import ctypes, sys, time
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
import oracle as O
from paper_2004_14020_b200 import _native as N, comm

def run(n, p, depth, epi=N.EPI_SUM, epochs=2, ctas_cap=None):
    dev = torch.device("cuda:0")
    ctas, bbytes, _ = N.bucket_layout(n, depth, N.SHUFFLE, p)
    ctas = min(ctas, ctas_cap or 148 // p)
    fb = N.flag_bytes_for(depth, ctas, N.SHUFFLE, p)
    foff = (bbytes + 255) // 256 * 256
    sgd = epi == N.EPI_SGD
    ctx = comm.Context(0, p, arena_bytes=foff + fb, param_bytes=4 * n if sgd else 0, nlocal=p)
    ctx.set_timeout_ms(1000)
    b = comm.make_bucket(n, 0, foff, depth=depth, pattern=N.SHUFFLE, epilogue=epi,
                         flags=N.F_PARAM_ARENA if sgd else 0, ctas=ctas, lr=0.1, scale=1.0 / p)
    st = torch.cuda.current_stream().cuda_stream
    for e in range(1, epochs + 1):
        for r in range(p):
            ctx.arena_view(r, 0, n).copy_(torch.randn(n, device=dev))
        bufs = [ctx.arena_view(r, 0, n).cpu().numpy() for r in range(p)]
        t0 = time.time()
        ctx.allreduce(b, e, st)
        torch.cuda.synchronize()
        dt = time.time() - t0
        try:
            ctx.status()
        except N.CaramelError as exc:
            print(f"n={n} p={p} depth={depth} ctas={ctas} epoch {e}: TIMEOUT {dt:.2f}s")
            for r in range(p):
                f = ctx.arena_view(r, foff, fb // 4).cpu().numpy().view(np.uint32)
                f = f[:depth * ctas * 2 * p].reshape(depth, ctas, 2, p)
                print(f"  rank {r} READY[c,j,src]=\n{f[:, :, 0, :]}\n  DONE=\n{f[:, :, 1, :]}")
            ctx.close()
            return False
        want = O.np_shuffle_lean(bufs, O.EPI_SUM)
        ok = all(np.array_equal(ctx.arena_view(r, 0, n).cpu().numpy().view(np.uint32), want.view(np.uint32))
                 for r in range(p))
        print(f"n={n} p={p} depth={depth} ctas={ctas} epoch {e}: {'ok' if ok else 'MISMATCH'} {dt*1e3:.2f} ms")
    ctx.close()
    return True

def run_list(model, p, mode, epochs=3):
    """Whole plan of `model` as one caramel_allreduce_many list, emulated; on a
    timeout print every bucket whose flags never reached the epoch."""
    sys.path.insert(0, str(ROOT / "tests"))
    from test_gpu_baseline_sizes import _plan, _device_list
    dev = torch.device("cuda:0")
    plan = _plan(model, p)
    ctx = comm.Context(0, p, arena_bytes=plan.arena_bytes, param_bytes=plan.param_bytes, nlocal=p)
    ctx.set_timeout_ms(1000)
    st = torch.cuda.current_stream().cuda_stream
    descs = [comm.make_bucket(b.numel, b.bucket_off, b.flag_off, depth=b.depth, pattern=N.SHUFFLE,
                              epilogue=N.EPI_SUM, flags=0, ctas=b.ctas, lr=0.1, scale=1.0 / p) for b in plan.buckets]
    host, dl, pre, spre = _device_list(descs, dev)
    for e in range(1, epochs + 1):
        for b in plan.buckets:
            for r in range(p):
                ctx.arena_view(r, b.bucket_off, b.numel).normal_()
        N.check(N.lib().caramel_epoch_advance(ctx._ctx, ctypes.c_void_p(st)))
        t0 = time.time()
        N.check(N.lib().caramel_allreduce_many(ctx._ctx, host, len(descs), dl.data_ptr(), pre.data_ptr(),
                                               spre.data_ptr(), 0, mode, 0, ctypes.c_void_p(st)))
        torch.cuda.synchronize()
        try:
            ctx.status()
            print(f"{model} p={p} mode={mode} epoch {e}: ok {(time.time()-t0)*1e3:.1f} ms")
        except N.CaramelError:
            print(f"{model} p={p} mode={mode} epoch {e}: TIMEOUT")
            for b in plan.buckets:
                fb = N.flag_bytes_for(b.depth, b.ctas, N.SHUFFLE, p)
                for r in range(p):
                    f = ctx.arena_view(r, b.flag_off, fb // 4).cpu().numpy().view(np.uint32)[:b.depth * b.ctas * 2 * p]
                    low = int((f < e).sum())
                    if low:
                        print(f"  bucket {b.index} n={b.numel} depth={b.depth} ctas={b.ctas} rank {r}: "
                              f"{low}/{f.size} flag words below epoch {e}")
            break
    ctx.close()


def run_custom(sizes, p, mode=N.MANY_FLAGS, depth=1, epochs=3):
    """A synthetic list of buckets of the given element counts, emulated."""
    dev = torch.device("cuda:0")
    specs, off = [], 0
    for n in sizes:
        ctas, bb, _ = N.bucket_layout(n, depth, N.SHUFFLE, p)
        ctas = min(ctas, 148 // p)
        fb = N.flag_bytes_for(depth, ctas, N.SHUFFLE, p)
        boff = off
        foff = (boff + bb + 255) // 256 * 256
        off = (foff + fb + 255) // 256 * 256
        specs.append((n, ctas, boff, foff, fb))
    ctx = comm.Context(0, p, arena_bytes=off, nlocal=p)
    ctx.set_timeout_ms(1000)
    st = torch.cuda.current_stream().cuda_stream
    descs = [comm.make_bucket(n, bo, fo, depth=depth, pattern=N.SHUFFLE, epilogue=N.EPI_SUM, flags=0, ctas=c)
             for n, c, bo, fo, _ in specs]
    host = (N.Bucket * len(descs))(*descs)
    dl = torch.frombuffer(bytearray(bytes(host)), dtype=torch.uint8).to(dev)
    pre = torch.tensor(np.concatenate([[0], np.cumsum(sizes)]), dtype=torch.int64, device=dev)
    spre = torch.zeros(len(sizes) + 1, dtype=torch.int64, device=dev)
    for e in range(1, epochs + 1):
        bufs = []
        for n, c, bo, fo, fb in specs:
            for r in range(p):
                ctx.arena_view(r, bo, n).normal_()
            bufs.append([ctx.arena_view(r, bo, n).cpu().numpy() for r in range(p)])
        N.check(N.lib().caramel_epoch_advance(ctx._ctx, ctypes.c_void_p(st)))
        N.check(N.lib().caramel_allreduce_many(ctx._ctx, host, len(descs), dl.data_ptr(), pre.data_ptr(),
                                               spre.data_ptr(), 0, mode, 0, ctypes.c_void_p(st)))
        torch.cuda.synchronize()
        try:
            ctx.status()
        except N.CaramelError:
            print(f"sizes={sizes} p={p} mode={mode} epoch {e}: TIMEOUT")
            for i, (n, c, bo, fo, fb) in enumerate(specs):
                f = ctx.arena_view(0, fo, fb // 4).cpu().numpy().view(np.uint32)[:depth * c * 2 * p]
                print(f"  bucket {i} n={n} ctas={c}: flags rank0 = {f.reshape(depth, c, 2, p)[:, :, :, :].tolist()}")
            ctx.close()
            return
        bad = []
        for i, (n, c, bo, fo, fb) in enumerate(specs):
            want = O.np_shuffle_lean(bufs[i], O.EPI_SUM)
            for r in range(p):
                if not np.array_equal(ctx.arena_view(r, bo, n).cpu().numpy().view(np.uint32), want.view(np.uint32)):
                    bad.append((i, r))
        print(f"sizes={sizes} p={p} mode={mode} epoch {e}: {'ok' if not bad else 'MISMATCH ' + str(bad[:6])}")
    ctx.close()


if __name__ == "__main__":
    for (n, p, d) in [(1 << 20, 2, 1), (70000, 4, 1), (300000, 4, 1), (1 << 20, 4, 1), (1 << 20, 4, 3), (1 << 20, 3, 1),
                      (1 << 22, 8, 2), (3 << 20, 2, 2)]:
        run(n, p, d)
    for p in (4, 2, 8):
        run_custom([300000, 400000], p)           # one-shot
        run_custom([2000000, 3000000], p)         # two-shot
        run_custom([1000, 300000, 5000, 2000000, 200, 100000], p)  # LL interleaved
        run_custom([1000, 300000, 5000, 2000000, 200, 100000], p, mode=N.MANY_FUSED)
    for m in ("resnet50", "inception_v3"):
        run_list(m, 4, N.MANY_FLAGS)
        run_list(m, 8, N.MANY_FUSED)
