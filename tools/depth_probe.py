"""Per-depth cost of one k_collective launch under rank emulation (1 GPU, p
ranks in one cooperative grid): 16 MiB SHUFFLE bucket, no pack, depth 1/2/3/4/8,
20 graph-captured calls per depth (CARAMEL_F_AUTO_EPOCH)."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2004_14020_b200 import _native as N  # noqa: E402
from paper_2004_14020_b200 import comm  # noqa: E402

p = int(os.environ.get("P", "2"))
nbytes = int(os.environ.get("BYTES", str(16 << 20)))
depths = [int(x) for x in os.environ.get("DEPTHS", "1,2,3,4,8").split(",")]
iters = int(os.environ.get("ITERS", "20"))
n = nbytes // 4
region = max(N.bucket_layout(n, d, N.SHUFFLE, p)[1] for d in depths)
region = (region + 4095) // 4096 * 4096
ctx = comm.Context(0, p, arena_bytes=region + (1 << 20), nlocal=p)
for r in range(p):
    ctx.arena_view(r, 0, n).normal_()
stream = torch.cuda.current_stream()
for d in depths:
    ctas, _, _ = N.bucket_layout(n, d, N.SHUFFLE, p)
    ctas = min(ctas, 148 // p)  # emulation: the whole grid must be co-resident
    b = comm.make_bucket(n, 0, region, depth=d, pattern=N.SHUFFLE, epilogue=N.EPI_SUM, flags=N.F_AUTO_EPOCH,
                         ctas=ctas)
    for _ in range(3):
        ctx.allreduce(b, 0, stream.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(stream)
    with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
        for _ in range(iters):
            ctx.allreduce(b, 0, side.cuda_stream)
    stream.wait_stream(side)
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g.replay()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / iters * 1e3)
    print(f"p={p} bytes={nbytes} depth={d} ctas={ctas}: {best:.2f} us", flush=True)
ctx.status()
ctx.close()
