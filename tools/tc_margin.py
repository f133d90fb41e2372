"""How many (range, domain) elements of the c4 identity full search pass the continuous level-1
bound |x| >= scl - e_row, with x = N / (n sqrt D) and scl from the final exact best, for a few
error margins e_row = c * max|r - mean r| (sizing the normalised-operand filter)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1501_02894_b200.synth import config_image

img = torch.from_numpy(config_image("c4")).cuda().double()
H, W = img.shape
B, n = 8, 64
s2 = img[:-1, :-1] + img[:-1, 1:] + img[1:, :-1] + img[1:, 1:]          # 2x2 sums at every offset
nd = H - 2 * B + 1
q = torch.stack([s2[2 * i:2 * i + nd, 2 * j:2 * j + nd] for i in range(B) for j in range(B)], -1).reshape(-1, n)
r = img.reshape(H // B, B, W // B, B).permute(0, 2, 1, 3).reshape(-1, n)
Sq, Sr = q.sum(1), r.sum(1)
D = n * (q * q).sum(1) - Sq * Sr.new_tensor(1.0) * Sq
rc = r - Sr[:, None] / n
emax = rc.abs().amax(1)
qh = ((q - Sq[:, None] / n) / D.clamp(min=1).sqrt()[:, None]) * (D > 0)[:, None]
k2 = torch.arange(-7, 8, 2, device="cuda", dtype=torch.float64)
best = torch.full((r.shape[0],), float("inf"), device="cuda", dtype=torch.float64)
CH = 8192
for d0 in range(0, q.shape[0], CH):
    C = r @ q[d0:d0 + CH].T
    N = n * C - Sr[:, None] * Sq[None, d0:d0 + CH]
    Dd = D[None, d0:d0 + CH]
    v = torch.stack([kk * kk * Dd - 64 * kk * N for kk in k2]).amin(0)
    best = torch.minimum(best, v.amin(1))
scl = torch.sqrt((-best).clamp(min=0) / 1024) / n
cs = [0.0, 2 ** -11, 2 ** -9, 2 ** -7]
cnt = {c: 0 for c in cs}
for d0 in range(0, q.shape[0], CH):
    x = (rc @ qh[d0:d0 + CH].T).abs()
    for c in cs:
        cnt[c] += int((x >= (scl - c * emax)[:, None]).sum())
tot = r.shape[0] * q.shape[0]
for c in cs:
    print(f"margin c={c:.2e}: {cnt[c]} of {tot} elements ({cnt[c] / tot * 1e6:.1f} ppm)")
print("median scl", float(scl.median()), "median emax", float(emax.median()), "flat ranges", int((best >= 0).sum()))
