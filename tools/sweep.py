"""Bucket-size sweep (config 5): caramel two-shot / ring / hd bus GB/s vs
NCCL all_reduce, one process per GPU.  Launch with torch.distributed.run."""
import ctypes, json, os, sys
from pathlib import Path
import torch, torch.distributed as dist
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2004_14020_b200 import _native as N, comm

def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local); dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    max_bytes = int(os.environ.get("SWEEP_MAX", 1 << 30))
    sizes = [4096 * 4 ** i for i in range(12) if 4096 * 4 ** i <= max_bytes]
    pats = [int(x) for x in os.environ.get("SWEEP_PATTERNS", "2").split(",")]
    engines = os.environ.get("SWEEP_ENGINES", "single").split(",")
    depths = [int(x) for x in os.environ.get("SWEEP_DEPTHS", "1").split(",")]
    iters = int(os.environ.get("SWEEP_ITERS", 20))
    maxel = max_bytes // 4
    region = max(N.bucket_layout(maxel, d, pt, world)[1] for pt in (0, 1, 2) if not (pt == 1 and world & (world - 1))
                 for d in (1, 8))
    region = (region + (1 << 20)) // (1 << 20) * (1 << 20)
    ctx = comm.Context(rank, world, arena_bytes=region + (256 << 20))
    ctx.bootstrap()
    if "nvls" in engines:
        if not ctx.nvls_available():
            engines = [e for e in engines if e != "nvls"]
        else:
            ctx.nvls_setup(max_bytes + (1 << 21))
            comm._view_fp32(ctx.nvls_base, maxel).normal_()
    base, _ = ctx.arena_ptrs(0)
    buf = comm._view_fp32(base, maxel)
    buf.normal_()
    stream = torch.cuda.current_stream()
    rows = []
    epoch = {}
    for size in sizes:
        n = size // 4
        for engine in engines:
          for pat in pats:
            if pat == N.HD and world & (world - 1):
                continue
            if engine in ("fused", "nvls") and pat != N.SHUFFLE:
                continue
            for depth in depths:
                ctas, bbytes, fbytes = N.bucket_layout(n, depth, pat, world)
                if os.environ.get("SWEEP_CTAS"):
                    ctas = min(ctas, int(os.environ["SWEEP_CTAS"]))
                if engine == "nvls":  # switch round trips only: the whole GPU
                    ctas = int(max(1, min(int(os.environ.get("SWEEP_NVLS_CTAS", 148)), n // world // 2048)))
                foff = region
                b = comm.make_bucket(n, 0, foff, depth=depth, pattern=pat, epilogue=N.EPI_SUM, flags=0, ctas=ctas)
                key = (engine, pat, depth, ctas)
                idx = list(epoch).index(key) if key in epoch else len(epoch)
                epoch.setdefault(key, 0)
                b.flag_off = foff + idx * (1 << 20)
                if engine == "fused":
                    host = (N.Bucket * 1)(b)
                    dlist = torch.frombuffer(bytearray(bytes(host)), dtype=torch.uint8).to(dev)
                    pre = torch.tensor([0, n], dtype=torch.int64, device=dev)
                    spre = torch.tensor([0, 0], dtype=torch.int64, device=dev)

                def launch(ep):
                    if engine == "fused":
                        N.check(N.lib().caramel_allreduce_many(ctx._ctx, host, 1, dlist.data_ptr(), pre.data_ptr(),
                                                               spre.data_ptr(), 0, N.MANY_FUSED, ep,
                                                               ctypes.c_void_p(stream.cuda_stream)))
                    elif engine == "nvls":
                        ctx.allreduce_nvls(b, ep, stream.cuda_stream)
                    else:
                        ctx.allreduce(b, ep, stream.cuda_stream)

                for it in range(5):
                    epoch[key] += 1
                    launch(epoch[key])
                torch.cuda.synchronize(); dist.barrier()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                for it in range(iters):
                    epoch[key] += 1
                    launch(epoch[key])
                e.record(stream); e.synchronize()
                ctx.status()
                t = torch.tensor(s.elapsed_time(e) / iters, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                us = t.item() * 1e3
                bus = 2 * (world - 1) / world * size / (us * 1e-6) / 1e9
                rows.append(dict(impl="caramel-" + engine, pattern=pat, depth=depth, ctas=ctas, bytes=size,
                                 us=round(us, 2), busbw=round(bus, 1)))
        # NCCL
        x = buf[:n]
        for it in range(5):
            dist.all_reduce(x)
        torch.cuda.synchronize(); dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for it in range(iters):
            dist.all_reduce(x)
        e.record(stream); e.synchronize()
        t = torch.tensor(s.elapsed_time(e) / iters, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        us = t.item() * 1e3
        rows.append(dict(impl="nccl", bytes=size, us=round(us, 2), busbw=round(2 * (world - 1) / world * size / (us * 1e-6) / 1e9, 1)))
    if rank == 0:
        for r in rows: print(json.dumps(r), flush=True)
    ctx.close(); dist.destroy_process_group()

if __name__ == "__main__":
    main()
