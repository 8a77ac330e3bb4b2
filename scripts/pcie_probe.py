"""Measure pinned H2D, D2H and concurrent H2D+D2H bandwidth on this box."""
import time
import torch

dev = torch.device("cuda", 0)
n = 128 << 20
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device=dev)
d_b = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


a, b, c = t(h2d), t(d2h), t(both)
print(f"H2D {n / a / 1e9:.1f} GB/s  D2H {n / b / 1e9:.1f} GB/s  both {2 * n / c / 1e9:.1f} GB/s total")

# the e2e step's transfer pattern alone (no kernels, no dependencies):
# 102.5 MB H2D in 6 pieces on one stream, 131.3 MB D2H in 6 x 5 pieces on another
H, D = 102_522_448, 131_291_299
hs = torch.empty(H, dtype=torch.uint8, pin_memory=True)
hd = torch.empty(D, dtype=torch.uint8, pin_memory=True)
dh = torch.empty(H, dtype=torch.uint8, device=dev)
dd = torch.empty(D, dtype=torch.uint8, device=dev)


def pattern(nh=6, nd=30):
    with torch.cuda.stream(s1):
        step = H // nh
        for i in range(nh):
            dh[i * step:(i + 1) * step].copy_(hs[i * step:(i + 1) * step], non_blocking=True)
    with torch.cuda.stream(s2):
        step = D // nd
        for i in range(nd):
            hd[i * step:(i + 1) * step].copy_(dd[i * step:(i + 1) * step], non_blocking=True)


for nh, nd in ((1, 1), (6, 6), (6, 30)):
    tt = t(lambda: pattern(nh, nd))
    print(f"e2e transfer pattern H2D {nh} + D2H {nd} pieces: {tt * 1e3:.3f} ms "
          f"({(H + D) / tt / 1e9:.1f} GB/s) -> bound {1e6 / tt / 1e6:.0f} M rec/s")
