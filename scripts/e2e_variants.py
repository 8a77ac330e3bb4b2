"""e2e throughput of StreamedRun variants (DMA drain vs zero-copy CSR), under gpurun."""
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

dag = sys.argv[1] if len(sys.argv) > 1 else "sign_heavy"
dev = torch.device("cuda", 0)
c = make_corpus(1_000_000, 5000, 11)
tmp = Path(tempfile.mkdtemp())
write_corpus(c, tmp)
cfg = config_from_dict(workload_config(dag), tmp)
views = {"user_events": c.driver, "user_profile": c.profile}
eng = E.Engine(E.prepare(cfg, views, c.basic), views, c.basic, device=str(dev))
for zc in (False, True):
    for rows in (65536, 131072, 262144, 1 << 20):
        sr = E.StreamedRun(eng, c.driver, slice_rows=rows, zero_copy=zc)
        ts = []
        for it in range(6):
            torch.cuda.synchronize()
            eng.begin_run(c.driver.row_count)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tot = sr.run()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        t = sorted(ts[1:])[len(ts[1:]) // 2]
        print(f"zero_copy={zc!s:5s} slice {rows:8d} x{len(sr.bounds):2d}: {t * 1e3:6.3f} ms "
              f"{1e6 / t / 1e6:6.1f} M rec/s  digest 0x{tot.digest:016x}", flush=True)
