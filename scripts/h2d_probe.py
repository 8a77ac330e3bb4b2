import time, torch, os, sys
sys.path.insert(0, "/root/repo")
dev = torch.device("cuda", 0)
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
for n in (25 << 20, 100 << 20):
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    def f():
        with torch.cuda.stream(s): d.copy_(h, non_blocking=True)
    print(n >> 20, "MB H2D", round(n / t(f) / 1e9, 1), "GB/s")
    def g():
        with torch.cuda.stream(s): d[:n-7].copy_(h[7:], non_blocking=True)
    print(n >> 20, "MB H2D unaligned", round(n / t(g) / 1e9, 1), "GB/s")
print(open("/proc/cpuinfo").read().count("processor"), "cpus")
os.system("nvidia-smi topo -m 2>/dev/null | head -5; numactl -H 2>/dev/null | head -3; lscpu | grep -i numa")
