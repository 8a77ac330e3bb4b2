"""After a multi-threaded pread into a pinned buffer, does evicting (clflushopt) or
writing back (clwb) the lines from the reader cores' caches restore the pinned
H2D rate?  (under gpurun; compiles a tiny helper with gcc)."""
import ctypes
import os
import subprocess
import tempfile
import threading
import time
from pathlib import Path

import numpy as np
import torch

src = r'''
#include <stddef.h>
#include <stdint.h>
#include <unistd.h>
#include <immintrin.h>
void flush_range(char* p, size_t n, int mode) {
  char* e = p + n;
  for (char* q = (char*)((uintptr_t)p & ~63ull); q < e; q += 64) {
    if (mode == 1) _mm_clflushopt(q); else _mm_clwb(q);
  }
  _mm_sfence();
}
long pread_flush(int fd, char* dst, size_t n, long off, int mode) {
  size_t done = 0;
  while (done < n) {
    size_t piece = n - done < (1u << 20) ? n - done : (1u << 20);
    ssize_t r = pread(fd, dst + done, piece, off + done);
    if (r <= 0) return -1;
    if (mode) flush_range(dst + done, (size_t)r, mode);
    done += (size_t)r;
  }
  return (long)done;
}
'''
d = Path(tempfile.mkdtemp())
(d / "f.c").write_text(src)
subprocess.run(["gcc", "-O2", "-shared", "-fPIC", "-mclflushopt", "-mclwb", "-o", str(d / "f.so"), str(d / "f.c")], check=True)
L = ctypes.CDLL(str(d / "f.so"))
L.pread_flush.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_long, ctypes.c_int]
L.pread_flush.restype = ctypes.c_long

n = 48 << 20
f = d / "x.bin"
np.random.randint(0, 255, size=n, dtype=np.uint8).tofile(f)
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
dv = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()


def h2d():
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        dv.copy_(h, non_blocking=True)
        b.record(s)
    s.synchronize()
    return n / a.elapsed_time(b) / 1e6


def read(threads, mode):
    fd = os.open(f, os.O_RDONLY)
    per = n // threads
    base = h.data_ptr()
    ts = [threading.Thread(target=L.pread_flush, args=(fd, base + i * per, per, i * per, mode))
          for i in range(threads)]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    dt = time.perf_counter() - t0
    os.close(fd)
    return n / dt / 1e9


for rep in range(3):
    for threads in (1, 8):
        for mode, name in ((0, "plain"), (1, "clflushopt"), (2, "clwb")):
            r = read(threads, mode)
            g = h2d()
            print(f"{threads} thr {name:10s} read {r:5.1f} GB/s  then H2D {g:5.1f} GB/s  "
                  f"(read+H2D {n / 1e6 / (n / r / 1e9 * 1e3 + n / g / 1e6):5.1f} GB/s serial)")
