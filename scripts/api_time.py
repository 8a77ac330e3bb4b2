"""Wall time of the drop-in run_pipelined(load_config(...)) over a 1M-record corpus
on disk (under gpurun), with the per-stage breakdown of the RunReport.

    python scripts/api_time.py [dag] [slice_rows]
"""
import json
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2210_07768_b200 import load_config  # noqa: E402
from paper_2210_07768_b200.config import config_from_dict  # noqa: E402
from paper_2210_07768_b200.corpus import gen_corpus  # noqa: E402
from paper_2210_07768_b200.engine import run_pipelined  # noqa: E402
from paper_2210_07768_b200.workloads import workload_config  # noqa: E402

dag = sys.argv[1] if len(sys.argv) > 1 else "sign_heavy"
slice_rows = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 18
d = Path(tempfile.mkdtemp())
t = time.time()
paths = gen_corpus(d, rows=1_000_000, users=5_000, seed=11)
print("gen", round(time.time() - t, 2))
cfg = (load_config(paths["config"]) if dag == "published" else
       config_from_dict(workload_config(dag), d))
for i in range(6):
    t = time.perf_counter()
    rep = run_pipelined(cfg, slice_rows=slice_rows)
    dt = time.perf_counter() - t
    print(f"run_pipelined {dt * 1e3:.2f} ms -> {1 / dt:.1f} M rec/s/M", hex(rep.digest),
          rep.instances, json.dumps({k: round(v * 1e3, 2) for k, v in rep.stage_seconds.items()}),
          "launches", rep.launches, "overhead_us", round(rep.overhead_us, 1), "h2d", rep.bytes_h2d)
