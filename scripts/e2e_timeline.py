"""Per-slice event timeline of the streamed e2e run (under gpurun).

    python scripts/e2e_timeline.py [slice_rows] [dag]
"""
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2210_07768_b200 import engine as E  # noqa: E402
from paper_2210_07768_b200.config import config_from_dict  # noqa: E402
from paper_2210_07768_b200.corpus import make_corpus, write_corpus  # noqa: E402
from paper_2210_07768_b200.workloads import workload_config  # noqa: E402

slice_rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 17
dag = sys.argv[2] if len(sys.argv) > 2 else "sign_heavy"
dev = torch.device("cuda", 0)
c = make_corpus(1_000_000, 5000, 11)
tmp = Path(tempfile.mkdtemp())
write_corpus(c, tmp)
cfg = config_from_dict(workload_config(dag), tmp)
views = {"user_events": c.driver, "user_profile": c.profile}
eng = E.Engine(E.prepare(cfg, views, c.basic), views, c.basic, device=str(dev))
sr = E.StreamedRun(eng, c.driver, slice_rows=slice_rows)
for it in range(4):
    torch.cuda.synchronize()
    eng.begin_run(c.driver.row_count)
    torch.cuda.synchronize()
    sr.trace = [] if it == 3 else None
    t0 = time.perf_counter()
    sr.run()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(f"step {dt * 1e3:.3f} ms  -> {1e6 / dt / 1e6:.1f} M rec/s  slices {len(sr.bounds)}")
ev = {}
for nm, k, te, th in sr.trace:
    ev[(nm, k)] = te
for k in range(len(sr.bounds)):
    g = lambda a: ev.get((a, k), float("nan"))  # noqa: E731
    print(f"slice {k:2d} rows {sr.bounds[k][1] - sr.bounds[k][0]:7d}  h2d {g('h2d0'):6.3f}-{g('h2d1'):6.3f}"
          f"  kern {g('k0'):6.3f}-{g('k1'):6.3f}  d2h {g('d2h0'):6.3f}-{g('d2h1'):6.3f}")
