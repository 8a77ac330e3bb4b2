"""Is a pinned H2D slower right after the host wrote the buffer (pread / fill)?"""
import os
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_07768_b200 import runtime  # noqa: E402

n = 48 << 20
f = Path(tempfile.mkdtemp()) / "x.bin"
np.random.randint(0, 255, size=n, dtype=np.uint8).tofile(f)
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()


def h2d():
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        d.copy_(h, non_blocking=True)
        b.record(s)
    s.synchronize()
    return n / a.elapsed_time(b) / 1e6


for rep in range(3):
    runtime.read_spans(f, h.data_ptr(), [0], [n], [0], 8)
    g1 = h2d()
    g2 = h2d()
    h.fill_(rep)
    g3 = h2d()
    time.sleep(0.01)
    g4 = h2d()
    print(f"after pread {g1:.1f} GB/s, again {g2:.1f}, after fill {g3:.1f}, after sleep {g4:.1f}")

# write-combined pinned staging (fbx_host_alloc)
wc = runtime.HostBuffer(n, write_combined=True)
hw = wc.tensor()
for rep in range(3):
    runtime.read_spans(f, wc.ptr, [0], [n], [0], 8)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    runtime.read_spans(f, wc.ptr, [0], [n], [0], 8)
    tr = time.perf_counter() - t0
    with torch.cuda.stream(s):
        a.record(s)
        d.copy_(hw, non_blocking=True)
        b.record(s)
    s.synchronize()
    print(f"WC: pread {n / tr / 1e9:.1f} GB/s, then H2D {n / a.elapsed_time(b) / 1e6:.1f} GB/s")
for rep in range(2):
    t0 = time.perf_counter()
    runtime.read_spans(f, h.data_ptr(), [0], [n], [0], 8)
    tr = time.perf_counter() - t0
    print(f"cached pinned: pread {n / tr / 1e9:.1f} GB/s, H2D {h2d():.1f} GB/s")

# pread, then touch one byte per 4 KiB page from user space, then H2D
for rep in range(3):
    runtime.read_spans(f, h.data_ptr(), [0], [n], [0], 8)
    t0 = time.perf_counter()
    hv = h.numpy()
    hv[::4096] = hv[::4096]
    tt = time.perf_counter() - t0
    print(f"pread + page touch ({tt * 1e3:.2f} ms): H2D {h2d():.1f} GB/s")
for th in (1, 2, 4):
    runtime.read_spans(f, h.data_ptr(), [0], [n], [0], th)
    print(f"pread with {th} threads: H2D {h2d():.1f} GB/s")
