import torch, time
n = 268435456
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device='cuda')
d2 = torch.empty(n, dtype=torch.uint8, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def t(fn, k=5):
    torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - a) / k
h2d = t(lambda: d.copy_(h, non_blocking=True))
d2h = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bb = t(both)
print(f"H2D {n/h2d/1e9:.1f} GB/s ({h2d*1e3:.2f} ms)  D2H {n/d2h/1e9:.1f} GB/s ({d2h*1e3:.2f} ms)  both {bb*1e3:.2f} ms")
# chunked H2D (4 MB chunks) to check
# chunked H2D + D2H on two streams each (8 chunks of 32 MB per direction)
sa, sb = [torch.cuda.Stream() for _ in range(2)], [torch.cuda.Stream() for _ in range(2)]
def chunked():
    c = n // 8
    for j in range(8):
        with torch.cuda.stream(sa[j & 1]): d[j * c:(j + 1) * c].copy_(h[j * c:(j + 1) * c], non_blocking=True)
        with torch.cuda.stream(sb[j & 1]): h2[j * c:(j + 1) * c].copy_(d2[j * c:(j + 1) * c], non_blocking=True)
ch = t(chunked)
print(f"both chunked {ch*1e3:.2f} ms")
