"""Is the slow pinned H2D after a multi-threaded pread a NUMA effect?  (under gpurun)
Reads a 48 MB file into a pinned buffer with 8 threads pinned to (a) all CPUs,
(b) the GPU-local NUMA node, (c) the other node(s), then times the H2D."""
import os
import sys
import tempfile
import threading
from pathlib import Path

import numpy as np
import torch

n = 48 << 20
f = Path(tempfile.mkdtemp()) / "x.bin"
np.random.randint(0, 255, size=n, dtype=np.uint8).tofile(f)
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
props = torch.cuda.get_device_properties(0)
bus = f"{props.pci_domain_id:04x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
local = Path(f"/sys/bus/pci/devices/{bus}/local_cpulist")
print("gpu", bus, "local cpus", local.read_text().strip() if local.exists() else "?")
print("numa node", Path(f"/sys/bus/pci/devices/{bus}/numa_node").read_text().strip()
      if Path(f"/sys/bus/pci/devices/{bus}/numa_node").exists() else "?")
nodes = sorted(Path("/sys/devices/system/node").glob("node[0-9]*"))
for nd in nodes:
    print(nd.name, (nd / "cpulist").read_text().strip())
allowed = sorted(os.sched_getaffinity(0))
print("allowed", len(allowed), allowed[:4], "...", allowed[-4:])


def parse(lst):
    out = []
    for part in lst.split(","):
        if "-" in part:
            a, b = part.split("-")
            out += list(range(int(a), int(b) + 1))
        elif part:
            out.append(int(part))
    return out


def h2d():
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        d.copy_(h, non_blocking=True)
        b.record(s)
    s.synchronize()
    return n / a.elapsed_time(b) / 1e6


mv = memoryview(h.numpy())


def read(cpus, threads=8):
    fd = os.open(f, os.O_RDONLY)
    per = n // threads

    def work(i):
        if cpus:
            os.sched_setaffinity(0, {cpus[i % len(cpus)]})
        os.preadv(fd, [mv[i * per:(i + 1) * per]], i * per)
    ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    os.close(fd)


sets = {"all": [c for c in allowed]}
if local.exists():
    lc = [c for c in parse(local.read_text().strip()) if c in allowed]
    sets["gpu-local"] = lc
    sets["remote"] = [c for c in allowed if c not in lc]
for nd in nodes:
    sets[nd.name] = [c for c in parse((nd / "cpulist").read_text().strip()) if c in allowed]
sets["one-thread"] = None
for rep in range(2):
    for name, cpus in sets.items():
        if cpus is not None and not cpus:
            continue
        if name == "one-thread":
            read(None, 1)
        else:
            read(cpus)
        g1 = h2d()
        g2 = h2d()
        print(f"{name:10s} after pread {g1:5.1f} GB/s, again {g2:5.1f}")
