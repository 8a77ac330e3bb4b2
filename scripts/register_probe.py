"""Can the driver file's page-cache pages be DMA'd directly (cudaHostRegister of a
read-only file mapping), and what does registering cost per call?  (under gpurun)"""
import ctypes
import mmap
import os
import tempfile
import time
from pathlib import Path

import numpy as np
import torch

cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
if cudart is None:
    import glob
    cudart = ctypes.CDLL(glob.glob("/usr/local/cuda/lib64/libcudart.so*")[0])
torch.cuda.init()
n = 96 << 20
f = Path(tempfile.mkdtemp()) / "x.bin"
np.random.randint(0, 255, size=n, dtype=np.uint8).tofile(f)
fd = os.open(f, os.O_RDONLY)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
READONLY, PORTABLE = 0x08, 0x01
v = ctypes.c_int(-1)
cudart.cudaDeviceGetAttribute(ctypes.byref(v), ctypes.c_int(113), ctypes.c_int(0))
print("HostRegisterReadOnlySupported", v.value)
cudart.cudaDeviceGetAttribute(ctypes.byref(v), ctypes.c_int(99), ctypes.c_int(0))
print("HostRegisterSupported", v.value)
cudart.cudaGetErrorString.restype = ctypes.c_char_p
for flags in (READONLY, READONLY | PORTABLE, 0):
    mm = mmap.mmap(fd, n, prot=mmap.PROT_READ, flags=mmap.MAP_SHARED)
    arr = np.frombuffer(mm, dtype=np.uint8)
    rc = cudart.cudaHostRegister(ctypes.c_void_p(arr.ctypes.data), ctypes.c_size_t(n), ctypes.c_uint(flags))
    print("flags", flags, "rc", rc, cudart.cudaGetErrorString(rc))
    cudart.cudaGetLastError()
    if rc == 0:
        cudart.cudaHostUnregister(ctypes.c_void_p(arr.ctypes.data))
    del arr
    mm.close()
for rep in range(4):
    t0 = time.perf_counter()
    mm = mmap.mmap(fd, n, prot=mmap.PROT_READ, flags=mmap.MAP_SHARED | getattr(mmap, "MAP_POPULATE", 0))
    buf = ctypes.c_char.from_buffer_copy(b"\0")  # placeholder
    addr = ctypes.c_void_p.from_buffer(ctypes.c_char_p(0))
    ptr = ctypes.cast(ctypes.c_char_p.from_buffer(mm), ctypes.c_void_p) if False else None
    # address of the mapping via numpy
    arr = np.frombuffer(mm, dtype=np.uint8)
    p = arr.ctypes.data
    t1 = time.perf_counter()
    rc = cudart.cudaHostRegister(ctypes.c_void_p(p), ctypes.c_size_t(n), ctypes.c_uint(READONLY))
    t2 = time.perf_counter()
    if rc != 0:
        print("register failed rc", rc)
        break
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        cudart.cudaMemcpyAsync(ctypes.c_void_p(d.data_ptr()), ctypes.c_void_p(p), ctypes.c_size_t(n),
                               ctypes.c_int(1), ctypes.c_void_p(s.cuda_stream))
        b.record(s)
    s.synchronize()
    t3 = time.perf_counter()
    rc2 = cudart.cudaHostUnregister(ctypes.c_void_p(p))
    t4 = time.perf_counter()
    ok = bool((d[:4096].cpu().numpy() == arr[:4096]).all())
    del arr
    mm.close()
    print(f"mmap+populate {1e3*(t1-t0):.2f} ms, register {1e3*(t2-t1):.2f} ms, H2D {n/a.elapsed_time(b)/1e6:.1f} GB/s "
          f"({1e3*(t3-t2):.2f} ms), unregister {1e3*(t4-t3):.2f} ms rc {rc2}, data ok {ok}")
