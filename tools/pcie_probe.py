"""Host<->device copy rates on the GPU box (pinned memory): H2D alone, D2H alone,
both at once, and H2D split over 2 / 4 streams.  Bounds the e2e (host-buffer) metric."""
import time

import torch

GB = 1 << 30
nbytes = 8 * GB
h_in = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
h_out = torch.empty_like(h_in, pin_memory=True)
d_a = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
d_b = torch.empty_like(d_a)
h_in.fill_(1.0)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def h2d():
    d_a.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_b, non_blocking=True)


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def h2d_split(k):
    streams = [torch.cuda.Stream() for _ in range(k)]
    m = d_a.numel() // k

    def run():
        for i, st in enumerate(streams):
            with torch.cuda.stream(st):
                d_a[i * m:(i + 1) * m].copy_(h_in[i * m:(i + 1) * m], non_blocking=True)
    return run


for name, fn, b in [("H2D", h2d, nbytes), ("D2H", d2h, nbytes), ("H2D+D2H", both, 2 * nbytes),
                    ("H2D x2 streams", h2d_split(2), nbytes), ("H2D x4 streams", h2d_split(4), nbytes)]:
    t = timed(fn)
    print(f"{name:16s} {t * 1e3:8.1f} ms  {b / t / 1e9:6.1f} GB/s")
