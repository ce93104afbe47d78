"""One rank of the multi-GPU parity check (launched by tests/test_multigpu.py
under torch.distributed.run).  Every rank packs its own gradients, runs the
collective through the C ABI with peer arenas mapped over CUDA IPC, and the
result is compared with the CPU oracle run on all ranks' inputs (gathered to
every rank over NCCL -- test plumbing only)."""

from __future__ import annotations

import os

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before any CUDA context: one hardware queue per stream
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import oracle as O  # noqa: E402
from paper_2004_14020_b200 import _native as N  # noqa: E402
from paper_2004_14020_b200 import comm  # noqa: E402


def main() -> int:
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    shapes = [(3, 5), (129,), (64, 7), (1,), (100_003,), (256, 1024), (7,)]
    numel = sum(int(np.prod(s)) for s in shapes)
    cases = [(N.SHUFFLE, 1), (N.SHUFFLE, 3), (N.SHUFFLE, 8), (N.RING, 2), (N.RING, 8)]
    if world & (world - 1) == 0:
        cases += [(N.HD, 1), (N.HD, 4)]
    # one arena holds every case's bucket + flag block at distinct offsets
    layout, off = [], 0
    for pat, depth in cases:
        ctas, bbytes, fbytes = N.bucket_layout(numel, depth, pat, world)
        boff = off
        foff = (boff + bbytes + 255) // 256 * 256
        off = (foff + fbytes + 255) // 256 * 256
        layout.append((pat, depth, ctas, boff, foff))
    ctx = comm.Context(rank, world, arena_bytes=off, param_bytes=4 * numel)
    ctx.bootstrap()
    stream = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(100 + rank)
    theta_rng = np.random.default_rng(7)
    theta = [theta_rng.standard_normal(s).astype(np.float32) for s in shapes]
    failures = 0
    for pat, depth, ctas, boff, foff in layout:
        for epi, arena in ((N.EPI_SUM, False), (N.EPI_SGD, False), (N.EPI_SGD, True)):
            for epoch in (1, 2):
                key_epoch = epoch + (0 if epi == N.EPI_SUM else 2 if not arena else 4)
                grads = [rng.standard_normal(s).astype(np.float32) for s in shapes]
                g_dev = [torch.from_numpy(g).to(dev) for g in grads]
                th_dev = [torch.from_numpy(t).to(dev) for t in theta]
                if arena:
                    ctx.arena_view(0, 0, numel, param=True).copy_(torch.from_numpy(O.np_pack(theta)).to(dev))
                table = comm.segment_table([comm.segments_for(g_dev, None if arena else th_dev)], dev)
                flags = N.F_PACK | N.F_UNPACK | (N.F_PARAM_ARENA if arena else 0)
                b = comm.make_bucket(numel, boff, foff, depth=depth, pattern=pat, epilogue=epi, flags=flags,
                                     ctas=ctas, segs=table, nseg=len(shapes), lr=0.05, scale=1.0 / world)
                torch.cuda.synchronize()
                dist.barrier()
                ctx.allreduce(b, key_epoch, stream)
                ctx.status()
                # oracle on everyone's inputs
                flat = torch.from_numpy(O.np_pack(grads)).to(dev)
                allg = [torch.empty_like(flat) for _ in range(world)]
                dist.all_gather(allg, flat)
                bufs = [a.cpu().numpy() for a in allg]
                want = O.np_allreduce(pat, bufs, depth, epi, 1.0 / world, 0.05, O.np_pack(theta))
                if epi == N.EPI_SUM:
                    got = torch.cat([t.flatten() for t in g_dev]).cpu().numpy()
                elif arena:
                    got = ctx.arena_view(0, 0, numel, param=True).cpu().numpy()
                else:
                    got = torch.cat([t.flatten() for t in th_dev]).cpu().numpy()
                ok = np.array_equal(got.view(np.uint32), want.view(np.uint32))
                if not ok:
                    failures += 1
                    bad = np.nonzero(got.view(np.uint32) != want.view(np.uint32))[0]
                    print(f"rank {rank}: MISMATCH pattern={pat} depth={depth} epi={epi} arena={arena} "
                          f"epoch={epoch}: {bad.size} elems, first {bad[:5]}", flush=True)
    ctx.close()
    failures += mixed_grouping_check(rank, world, dev)
    failures += overlapped_hooks_check(rank, world, dev)
    failures += overlapped_hooks_check(rank, world, dev, grads="bucket")
    failures += ce_check(rank, world, dev)
    failures += ce_check(rank, world, dev, gated="pull")
    failures += nvls_check(rank, world, dev)
    failures += overlapped_hooks_check(rank, world, dev, grads="bucket", engine="ce")
    failures += overlapped_hooks_check(rank, world, dev, grads="bucket", engine="gated")
    t = torch.tensor([failures], device=dev)
    dist.all_reduce(t)
    if rank == 0:
        print(f"multigpu parity: world={world} cases={len(layout) * 6 + 5} failures={int(t.item())}", flush=True)
    dist.destroy_process_group()
    return 0 if int(t.item()) == 0 else 1


def mixed_grouping_check(rank: int, world: int, dev) -> int:
    """Same launch order, different grouping per rank: rank 0 issues the five
    buckets as ONE per-bucket-flag list (CARAMEL_MANY_FLAGS), odd ranks one
    launch per bucket, the rest as two lists.  Every rank must match the oracle."""
    import ctypes

    rng = np.random.default_rng(300 + rank)
    bucket_shapes = [[(5,), (300,)], [(7, 7)], [(1,)], [(4096,), (3,)], [(64, 65)]]
    depths = [1, 2, 1, 3, 2]
    specs, off = [], 0
    for shapes, depth in zip(bucket_shapes, depths):
        numel = sum(int(np.prod(s)) for s in shapes)
        ctas, bbytes, fbytes = N.bucket_layout(numel, depth, N.SHUFFLE, world)
        boff = off
        foff = (boff + bbytes + 255) // 256 * 256
        off = (foff + fbytes + 255) // 256 * 256
        specs.append((shapes, depth, numel, ctas, boff, foff))
    ctx = comm.Context(rank, world, arena_bytes=off)
    ctx.bootstrap()
    stream = torch.cuda.current_stream().cuda_stream
    fails = 0
    for epoch in (1, 2, 3):
        grads, gdev, descs, tables = [], [], [], []
        for shapes, depth, numel, ctas, boff, foff in specs:
            g = [rng.standard_normal(s).astype(np.float32) for s in shapes]
            gd = [torch.from_numpy(a).to(dev) for a in g]
            t = comm.segment_table([comm.segments_for(gd)], dev)
            grads.append(g)
            gdev.append(gd)
            tables.append(t)
            descs.append(comm.make_bucket(numel, boff, foff, depth=depth, pattern=N.SHUFFLE, epilogue=N.EPI_SUM,
                                          flags=N.F_PACK | N.F_UNPACK, ctas=ctas, segs=t, nseg=len(shapes)))
        host = (N.Bucket * len(descs))(*descs)
        dlist = torch.frombuffer(bytearray(bytes(host)), dtype=torch.uint8).to(dev)
        pre = torch.tensor(np.concatenate([[0], np.cumsum([sp[2] for sp in specs])]), dtype=torch.int64, device=dev)
        spre = torch.tensor(np.concatenate([[0], np.cumsum([len(sp[0]) for sp in specs])]), dtype=torch.int64,
                            device=dev)
        bsz = ctypes.sizeof(N.Bucket)

        def launch_list(i, j):
            h = ctypes.cast(ctypes.byref(host, i * bsz), ctypes.POINTER(N.Bucket))
            N.check(N.lib().caramel_allreduce_many(ctx._ctx, h, j - i, dlist.data_ptr() + i * bsz,
                                                   pre.data_ptr() + 8 * i, spre.data_ptr() + 8 * i, 0,
                                                   N.MANY_FLAGS, epoch, ctypes.c_void_p(stream)))

        torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            launch_list(0, len(descs))
        elif rank % 2 == 1:
            for d in descs:
                ctx.allreduce(d, epoch, stream)
        else:
            launch_list(0, 2)
            launch_list(2, len(descs))
        ctx.status()
        for i, (shapes, depth, numel, ctas, boff, foff) in enumerate(specs):
            flat = torch.from_numpy(O.np_pack(grads[i])).to(dev)
            allg = [torch.empty_like(flat) for _ in range(world)]
            dist.all_gather(allg, flat)
            want = O.np_allreduce(N.SHUFFLE, [a.cpu().numpy() for a in allg], depth)
            got = torch.cat([t.flatten() for t in gdev[i]]).cpu().numpy()
            if not np.array_equal(got.view(np.uint32), want.view(np.uint32)):
                fails += 1
                print(f"rank {rank}: mixed grouping mismatch bucket {i} epoch {epoch}", flush=True)
    ctx.close()
    return fails


def ce_check(rank: int, world: int, dev, gated: str = "") -> int:
    """Copy-engine two-shot (caramel_allreduce_ce) -- or the
    gated SM engine (gated="pull": caramel_allreduce_gated) -- through the C ABI: six
    buckets, gradients in the bucket arena, SUM and fused SGD, the launch
    order in one call, one call per bucket, and two calls.  Bit-exact with the
    oracle's SHUFFLE order."""
    import ctypes

    fn = {"": N.lib().caramel_allreduce_ce, "pull": N.lib().caramel_allreduce_gated}[gated]
    what = f"gated SM engine ({gated})" if gated else "copy-engine"

    rng = np.random.default_rng(500 + rank)
    theta_rng = np.random.default_rng(9)
    sizes = [1, 5, 300, 4099, 70_001, 1 << 20]
    specs, off, poff = [], 0, 0
    for n in sizes:
        ctas, bbytes, fbytes = N.bucket_layout(n, 1, N.SHUFFLE, world)
        boff = off
        foff = (boff + bbytes + 255) // 256 * 256
        off = (foff + fbytes + 255) // 256 * 256
        specs.append((n, ctas, boff, foff, poff))
        poff = (poff + 4 * n + 255) // 256 * 256
    ctx = comm.Context(rank, world, arena_bytes=off, param_bytes=poff)
    ctx.bootstrap()
    if not N.lib().caramel_ce_available(ctx._ctx):
        print(f"rank {rank}: copy-engine path unavailable on this device", flush=True)
        ctx.close()
        return 1
    stream = torch.cuda.current_stream().cuda_stream  # gradients' stream: READY goes out here
    side = torch.cuda.Stream()                         # the collective's stream
    fails = 0
    epoch = 0
    for epi in (N.EPI_SUM, N.EPI_SGD):
        for grouping in range(3):
            epoch += 1
            grads = [rng.standard_normal(n).astype(np.float32) for n in sizes]
            theta = [theta_rng.standard_normal(n).astype(np.float32) for n in sizes]
            descs = []
            for (n, ctas, boff, foff, po), g, th in zip(specs, grads, theta):
                ctx.arena_view(0, boff, n).copy_(torch.from_numpy(g).to(dev))
                ctx.arena_view(0, po, n, param=True).copy_(torch.from_numpy(th).to(dev))
                descs.append(comm.make_bucket(n, boff, foff, pattern=N.SHUFFLE, epilogue=epi, ctas=ctas,
                                              flags=N.F_PARAM_ARENA if epi == N.EPI_SGD else 0, param_off=po,
                                              lr=0.05, scale=1.0 / world))
            host = (N.Bucket * len(descs))(*descs)
            bsz = ctypes.sizeof(N.Bucket)

            def call(i, j):
                h = ctypes.cast(ctypes.byref(host, i * bsz), ctypes.POINTER(N.Bucket))
                N.check(fn(ctx._ctx, h, j - i, i, epoch, ctypes.c_void_p(stream), ctypes.c_void_p(side.cuda_stream)))

            torch.cuda.synchronize()
            dist.barrier()
            side.wait_stream(torch.cuda.current_stream())
            if grouping == 0:
                call(0, len(descs))
            elif grouping == 1:
                for i in range(len(descs)):
                    call(i, i + 1)
            else:
                call(0, 3)
                call(3, len(descs))
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            for i, (n, ctas, boff, foff, po) in enumerate(specs):
                flat = torch.from_numpy(grads[i]).to(dev)
                allg = [torch.empty_like(flat) for _ in range(world)]
                dist.all_gather(allg, flat)
                want = O.np_allreduce(N.SHUFFLE, [a.cpu().numpy() for a in allg], 1, epi, 1.0 / world, 0.05,
                                      theta[i])
                got = ctx.arena_view(0, po if epi == N.EPI_SGD else boff, n, param=epi == N.EPI_SGD).cpu().numpy()
                if not np.array_equal(got.view(np.uint32), want.view(np.uint32)):
                    fails += 1
                    bad = np.nonzero(got.view(np.uint32) != want.view(np.uint32))[0]
                    print(f"rank {rank}: {what} mismatch bucket {i} (n={n}) epi={epi} epoch {epoch}: "
                          f"{bad.size} elems, first {bad[:5]}", flush=True)
    ctx.close()
    return fails


def nvls_check(rank: int, world: int, dev) -> int:
    """NVLS two-shot (caramel_allreduce_nvls: multimem.ld_reduce / multimem.st
    through the NVSwitch) -- the non-fixed-order mode.  Every element within
    1e-6 x sum_r |g_r| of the float64 sum (SURVEY §8c's bound; SGD adds the
    update's own fp32 rounding), and every replica bit-identical."""
    rng = np.random.default_rng(900 + rank)
    th_rng = np.random.default_rng(11)
    sizes = [5, 1000, 70_001, 1 << 20, (3 << 20) + 7]
    probe = comm.Context(rank, world, arena_bytes=1 << 20)
    ok = torch.tensor([probe.nvls_available()], device=dev, dtype=torch.int32)
    probe.close()
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if not int(ok.item()):
        if rank == 0:
            print("nvls: multicast objects not available on this box (skipped)", flush=True)
        return 0
    specs, moff, foff, poff = [], 0, 0, 0
    for n in sizes:
        for depth in (1, 3):
            ctas = min(N.bucket_layout(n, depth, N.SHUFFLE, world)[0], 16)
            fb = N.flag_bytes_for(depth, ctas, N.SHUFFLE, world)
            specs.append((n, depth, ctas, moff, foff, poff))
            moff = (moff + 4 * n + 255) // 256 * 256
            foff = (foff + fb + 255) // 256 * 256
            poff = (poff + 4 * n + 255) // 256 * 256
    ctx = comm.Context(rank, world, arena_bytes=foff, param_bytes=poff)
    ctx.bootstrap()
    ctx.nvls_setup(moff)
    stream = torch.cuda.current_stream().cuda_stream
    fails, epoch, lr = 0, 0, 0.05
    for epi in (N.EPI_SUM, N.EPI_SCALE, N.EPI_SGD):
        epoch += 1
        grads, thetas = [], []
        for n, depth, ctas, mo, fo, po in specs:
            g = rng.standard_normal(n).astype(np.float32)
            th = th_rng.standard_normal(n).astype(np.float32)
            ctx.nvls_view(mo, n).copy_(torch.from_numpy(g).to(dev))
            ctx.arena_view(0, po, n, param=True).copy_(torch.from_numpy(th).to(dev))
            grads.append(g)
            thetas.append(th)
        torch.cuda.synchronize()
        dist.barrier()
        for (n, depth, ctas, mo, fo, po) in specs:
            b = comm.make_bucket(n, mo, fo, depth=depth, pattern=N.SHUFFLE, epilogue=epi, ctas=ctas,
                                 flags=N.F_PARAM_ARENA if epi == N.EPI_SGD else 0, param_off=po, lr=lr,
                                 scale=1.0 / world)
            ctx.allreduce_nvls(b, epoch, stream)
        ctx.status()
        torch.cuda.synchronize()
        for i, (n, depth, ctas, mo, fo, po) in enumerate(specs):
            flat = torch.from_numpy(grads[i]).to(dev)
            allg = [torch.empty_like(flat) for _ in range(world)]
            dist.all_gather(allg, flat)
            G = np.stack([a.cpu().numpy().astype(np.float64) for a in allg])
            s64, a64 = G.sum(axis=0), np.abs(G).sum(axis=0)
            if epi == N.EPI_SGD:
                got = ctx.arena_view(0, po, n, param=True).clone()
                step = lr * s64 / world
                ref = thetas[i].astype(np.float64) - step
                tol = 1e-6 * lr * a64 / world + 2.0 ** -23 * (np.abs(thetas[i]) + np.abs(step))
            else:
                got = ctx.nvls_view(mo, n).clone()
                scale = 1.0 if epi == N.EPI_SUM else 1.0 / world
                ref, tol = s64 * scale, 1e-6 * a64 * scale
            err = np.abs(got.cpu().numpy().astype(np.float64) - ref)
            if not (err <= tol).all():
                fails += 1
                k = int(np.argmax(err - tol))
                print(f"rank {rank}: nvls epi={epi} n={n} depth={depth}: err {err[k]:.3e} > tol {tol[k]:.3e}",
                      flush=True)
            reps = [torch.empty_like(got) for _ in range(world)]
            dist.all_gather(reps, got)
            if any(not torch.equal(reps[0], r) for r in reps[1:]):
                fails += 1
                print(f"rank {rank}: nvls epi={epi} n={n}: replicas differ", flush=True)
    if rank == 0:
        print(f"nvls: {len(specs) * 3} bucket checks (1e-6 x sum|g| vs float64, replicas identical)", flush=True)
    ctx.close()
    return fails


def overlapped_hooks_check(rank: int, world: int, dev, grads: str = "flat", engine: str = "sm") -> int:
    """Real backward on every rank, buckets launched from gradient hooks in the
    enforced order, SGD fused into the all-gather; every replica must equal
    theta - lr * ((sum of all ranks' grads in rank order) * (1/p))."""
    from paper_2004_14020_b200 import gradsets
    from paper_2004_14020_b200.collective import Pattern, ReduceModel
    from paper_2004_14020_b200.costmodel import NetworkModel
    from paper_2004_14020_b200.executor import Aggregator, lower
    from paper_2004_14020_b200.pipeline import run_pipeline
    from paper_2004_14020_b200.sim import SimConfig

    def tiny():
        torch.manual_seed(0)
        return torch.nn.Sequential(torch.nn.Linear(37, 64), torch.nn.ReLU(), torch.nn.Linear(64, 129),
                                   torch.nn.ReLU(), torch.nn.Linear(129, 10)).to(dev)

    lr = 0.05
    model, ref = tiny(), tiny()
    tensors = tuple(gradsets.Tensor(n, tuple(p.shape)) for n, p in model.named_parameters())
    art = run_pipeline(gradsets.layered_chain_dag(tensors),
                       SimConfig(workers=world, network=NetworkModel(10.0, 1e-4), reduce=ReduceModel(400.0, 10.0)))
    ids = [gradsets.param_id(i, len(tensors)) for i in range(len(tensors))]
    plan = lower(art, {pid: t.numel for pid, t in zip(ids, tensors)}, world, Pattern.SHUFFLE)
    agg = Aggregator(plan, dict(zip(ids, model.parameters())), rank=rank, lr=lr, epilogue="sgd", grads=grads,
                     engine=engine)
    if engine == "ce":
        agg.ce_min_bytes = 4 * 1024 if world % 2 == 0 else 0  # mixed SM / copy-engine buckets, or all copy-engine
    agg.attach_hooks()
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    fails = 0
    for it in range(3):
        x = torch.randn(16, 37, device=dev, generator=gen)
        ref.zero_grad(set_to_none=False)
        ref(x).square().mean().backward()
        flat = torch.cat([p.grad.reshape(-1) for p in ref.parameters()])
        allg = [torch.empty_like(flat) for _ in range(world)]
        dist.all_gather(allg, flat)
        s = allg[0].clone()
        for q in range(1, world):
            s = s + allg[q]
        step = lr * (s * (1.0 / world))
        off = 0
        with torch.no_grad():
            for p in ref.parameters():
                n = p.numel()
                p.copy_(p - step[off:off + n].view_as(p))
                off += n
        model.zero_grad(set_to_none=False)
        agg.begin_iteration()
        model(x).square().mean().backward()
        agg.finish_iteration()
        torch.cuda.synchronize()
        agg.status()
        for a, b in zip(model.parameters(), ref.parameters()):
            if not torch.equal(a, b):
                fails += 1
                print(f"rank {rank}: overlapped hooks ({grads}, {engine}) mismatch at iteration {it}", flush=True)
                break
    agg.close()
    return fails


if __name__ == "__main__":
    sys.exit(main())
