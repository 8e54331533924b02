import torch, time
N = 400_000_000 // 4
h1 = torch.empty(N, dtype=torch.float32).pin_memory(); h2 = torch.empty(N, dtype=torch.float32).pin_memory()
d1 = torch.empty(N, device='cuda'); d2 = torch.empty(N, device='cuda')
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
def t(f, reps=5):
    f(); torch.cuda.synchronize(); t0=time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter()-t0)/reps
h2d = t(lambda: d1.copy_(h1, non_blocking=True)); d2h = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bb = t(both)
print(f"H2D {0.4/h2d:.1f} GB/s  D2H {0.4/d2h:.1f} GB/s  both-concurrent {0.8/bb:.1f} GB/s total ({bb*1e3:.2f} ms for 400+400 MB)")
