"""Comparator only (never the product path): cuFFT via torch.fft for the same
spectral Poisson solve, to calibrate what NVIDIA's library reaches on B200."""
import sys
import time

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
dt = torch.float64 if (len(sys.argv) < 3 or sys.argv[2] == "64") else torch.float32
f = torch.randn(n, n, n, dtype=dt, device="cuda")
k = torch.fft.fftfreq(n, 1.0 / n, dtype=dt, device="cuda")
kk = torch.arange(n // 2 + 1, dtype=dt, device="cuda")
k2 = k[:, None, None] ** 2 + k[None, :, None] ** 2 + kk[None, None, :] ** 2
sym = torch.where(k2 == 0, torch.zeros_like(k2), 1.0 / (4 * torch.pi ** 2 * k2))
del k2


def solve():
    F = torch.fft.rfftn(f)
    F *= sym
    return torch.fft.irfftn(F, s=f.shape)


for _ in range(3):
    solve()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    u = solve()
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 5
# separate transforms
s.record()
for _ in range(5):
    F = torch.fft.rfftn(f)
e.record()
torch.cuda.synchronize()
ms_f = s.elapsed_time(e) / 5
print(f"cuFFT (torch.fft) n={n} {dt}: solve {ms:.3f} ms ({n**3/ms/1e6:.1f} G unknowns/s), rfftn alone {ms_f:.3f} ms")
