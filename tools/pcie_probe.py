import torch, time
n = 102228128 // 4
h = torch.randn(n).pin_memory(); h2 = torch.empty(n).pin_memory()
d = torch.empty(n, device="cuda"); d2 = torch.randn(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, k=10):
    fn(); torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / k * 1e3
def h2d():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
print(f"H2D {t(h2d):.3f} ms, D2H {t(d2h):.3f} ms, both concurrent {t(both):.3f} ms for 102.2 MB each")
