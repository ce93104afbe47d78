"""Randomised stress of the single-GPU TMA kernels (compute-sanitizer is closed
on this pool, so races in the mbarrier / bulk-copy pipelines are hunted by
volume instead): thousands of random member sets -- sizes 1..300K elements,
random 4-byte misalignment, 1..400 members -- through caramel_pack /
caramel_unpack (k_pack_tma), and random bucket lists through the world = 1
fused update (k_local_flat_tma / k_local_many), each checked bit for bit
against plain PyTorch (torch.cat; theta - lr * (g * scale) with separate fp32
roundings).  One JSON summary line."""
import ctypes, json, sys, time
from pathlib import Path
import numpy as np
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2004_14020_b200 import _native as N, comm


def main(iters=3000, seed=0):
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(seed)
    stream = torch.cuda.current_stream().cuda_stream
    big = torch.empty(64 << 20, device=dev)
    fails = {"pack": 0, "unpack": 0, "update": 0}
    t0 = time.time()
    nbytes = 0
    for it in range(iters):
        k = int(rng.integers(1, 400))
        sizes = np.minimum(rng.geometric(1.0 / rng.choice([8, 300, 20000]), size=k), 300_000)
        # carve members out of `big` at random element offsets (misaligned by 0..3 elements)
        offs, pos = [], int(rng.integers(0, 4))
        for n in sizes:
            offs.append(pos)
            pos += int(n) + int(rng.integers(0, 9))
        if pos > big.numel():
            continue
        members = [big[o:o + int(n)] for o, n in zip(offs, sizes)]
        for m in members:
            m.normal_()
        numel = int(sizes.sum())
        bucket = torch.empty(numel + 8, device=dev)
        tab = comm.segment_table([comm.segments_for(members)], dev)
        comm.pack(tab, len(members), numel, bucket.data_ptr(), stream)
        want = torch.cat(members)
        if not torch.equal(bucket[:numel], want):
            fails["pack"] += 1
        bucket[:numel].mul_(-0.5)
        comm.unpack(tab, len(members), numel, bucket.data_ptr(), False, stream)
        if not torch.equal(torch.cat(members), want * -0.5):
            fails["unpack"] += 1
        nbytes += 16 * numel
    # world = 1 fused update over random bucket lists
    for it in range(iters // 10):
        nb = int(rng.integers(1, 200))
        numels = [int(x) for x in np.minimum(rng.geometric(1.0 / rng.choice([16, 4000, 200000]), size=nb), 2_000_000)]
        offs, boff = [], 0
        for n in numels:
            offs.append(boff)
            boff = (boff + 4 * n + 255) // 256 * 256
        ctx = comm.Context(0, 1, arena_bytes=boff + 4096, param_bytes=boff + 4096)
        descs = []
        for n, o in zip(numels, offs):
            ctx.arena_view(0, o, n).normal_()
            ctx.arena_view(0, o, n, param=True).normal_()
            descs.append(comm.make_bucket(n, o, 0, epilogue=N.EPI_SGD, flags=N.F_PARAM_ARENA, ctas=1,
                                          param_off=o, lr=0.37, scale=0.25))
        ref = [ctx.arena_view(0, o, n, param=True) - 0.37 * (ctx.arena_view(0, o, n) * 0.25)
               for n, o in zip(numels, offs)]
        host = (N.Bucket * nb)(*descs)
        dl = torch.frombuffer(bytearray(bytes(host)), dtype=torch.uint8).to(dev)
        pre = torch.tensor(np.concatenate([[0], np.cumsum(numels)]), dtype=torch.int64, device=dev)
        spre = torch.zeros(nb + 1, dtype=torch.int64, device=dev)
        N.check(N.lib().caramel_allreduce_many(ctx._ctx, host, nb, dl.data_ptr(), pre.data_ptr(), spre.data_ptr(),
                                               0, N.MANY_FUSED, 1, ctypes.c_void_p(stream)))
        torch.cuda.synchronize()
        for r, n, o in zip(ref, numels, offs):
            if not torch.equal(ctx.arena_view(0, o, n, param=True), r):
                fails["update"] += 1
                break
        ctx.close()
    torch.cuda.synchronize()
    print(json.dumps({"summary": "stress_local", "pack_unpack_cases": iters, "update_lists": iters // 10,
                      "failures": fails, "pack_unpack_bytes": nbytes, "elapsed_s": round(time.time() - t0, 1)}),
          flush=True)
    return 0 if not any(fails.values()) else 1


if __name__ == "__main__":
    sys.exit(main())
