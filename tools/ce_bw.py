"""Copy-engine NVLink bandwidth on this box: pull (destination-side stream,
remote source) vs push (source-side stream, remote destination), one peer at a
time or all peers at once, every GPU transferring simultaneously.

    python tools/ce_bw.py [MB]        (one process, all visible GPUs)
"""
import sys

import torch
from cuda.bindings import runtime as rt

MB = int(sys.argv[1]) if len(sys.argv) > 1 else 64
n = torch.cuda.device_count()
size = MB << 20
bufs = {}
for d in range(n):
    torch.cuda.set_device(d)
    for q in range(n):
        if q != d:
            rt.cudaDeviceEnablePeerAccess(q, 0)
    bufs[d] = (torch.empty(size * n, dtype=torch.uint8, device=d), torch.empty(size * n, dtype=torch.uint8, device=d))
streams = {(d, k): torch.cuda.Stream(device=d) for d in range(n) for k in range(n)}


def run(mode: str, fan: int, reps: int = 10) -> float:
    """All GPUs at once; each moves `fan` peer copies of `size` bytes per rep.
    Returns per-GPU GB/s (bytes it receives (pull) or sends (push))."""
    evs = []
    for d in range(n):
        torch.cuda.set_device(d)
        s = torch.cuda.Event(enable_timing=True)
        s.record(streams[(d, 0)])
        evs.append([s, None])
    for d in range(n):
        for k in range(1, n):
            streams[(d, k)].wait_event(evs[d][0])
    for _ in range(reps):
        for d in range(n):
            for k in range(1, fan + 1):
                q = (d + k) % n
                st = streams[(d, k if fan > 1 else 0)]
                src, dst = bufs[d][0], bufs[d][1]
                if mode == "pull":   # stream on d: remote q -> local d
                    a, b = bufs[q][0].data_ptr() + d * size, dst.data_ptr() + q * size
                else:                # stream on d: local d -> remote q
                    a, b = src.data_ptr() + q * size, bufs[q][1].data_ptr() + d * size
                rt.cudaMemcpyAsync(b, a, size, rt.cudaMemcpyKind.cudaMemcpyDefault, st.cuda_stream)
    for d in range(n):
        torch.cuda.set_device(d)
        for k in range(1, n):
            streams[(d, 0)].wait_stream(streams[(d, k)])
        e = torch.cuda.Event(enable_timing=True)
        e.record(streams[(d, 0)])
        evs[d][1] = e
    for d in range(n):
        torch.cuda.synchronize(d)
    ms = max(s.elapsed_time(e) for s, e in evs)
    return fan * reps * size / ms / 1e6


for mode in ("pull", "push"):
    for fan in sorted({1, n - 1}):
        run(mode, fan, 2)
        print(f"{mode} fan {fan}: {run(mode, fan):.1f} GB/s per GPU ({MB} MB copies, {n} GPUs at once)", flush=True)
