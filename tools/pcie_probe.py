import torch, time
n = 34020000 // 8
h = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
d = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / reps * 1e3
h2d = t(lambda: d[0].copy_(h[0], non_blocking=True))
d2h = t(lambda: h[1].copy_(d[1], non_blocking=True))
def both():
    with torch.cuda.stream(s1): d[0].copy_(h[0], non_blocking=True)
    with torch.cuda.stream(s2): h[1].copy_(d[1], non_blocking=True)
bo = t(both)
print(f"34 MB: H2D {h2d:.3f} ms ({34.02/h2d:.1f} GB/s)  D2H {d2h:.3f} ms ({34.02/d2h:.1f} GB/s)  both concurrently {bo:.3f} ms")
