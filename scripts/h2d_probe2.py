import sys, time, torch
sys.path.insert(0, "/root/repo")
from paper_2210_07768_b200 import runtime
n = 28_500_000
for rep in range(3):
    host = torch.empty(n + 16, dtype=torch.uint8, pin_memory=True)
    host.fill_(3)
    body = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    body[:n].copy_(host[:n], non_blocking=True)
    b.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"copy: enqueue {1e3*(t1-t0):.2f} ms, sync {1e3*(t2-t1):.2f} ms, event {a.elapsed_time(b):.2f} ms, pinned={host.is_pinned()}")
    s = torch.cuda.Stream()
    a.record(s)
    with torch.cuda.stream(s):
        body[:n].copy_(host[:n], non_blocking=True)
    b.record(s)
    s.synchronize()
    print(f"  side stream event {a.elapsed_time(b):.2f} ms")
