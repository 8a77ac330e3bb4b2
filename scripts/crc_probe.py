"""Device CRC-32 throughput (fbx_crc32) vs host zlib on a 1 GiB buffer (under gpurun)."""
import sys
import time
import zlib
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_07768_b200.engine import crc32_device  # noqa: E402

n = 1 << 30
host = np.random.default_rng(0).integers(0, 256, size=n, dtype=np.uint8)
dev = torch.from_numpy(host).cuda()
crc32_device(dev)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    got = crc32_device(dev)
b.record()
torch.cuda.synchronize()
dt = a.elapsed_time(b) / 5 / 1e3
t0 = time.perf_counter()
want = zlib.crc32(host) & 0xFFFFFFFF
ht = time.perf_counter() - t0
assert got == want
print(f"device crc32 {n / dt / 1e9:.0f} GB/s (incl. the 4-byte readback), host zlib {n / ht / 1e9:.1f} GB/s")
