"""Host + device timeline of one drop-in run_pipelined call on a 1M-record log
(under gpurun): wall-clock marks of every phase (wrapped, no product change) and
the file stream's per-slice H2D / kernel events on the same clock."""
import sys
import tempfile
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2210_07768_b200 import engine as E, runtime, stream as S  # noqa: E402
from paper_2210_07768_b200.config import config_from_dict  # noqa: E402
from paper_2210_07768_b200.corpus import gen_corpus  # noqa: E402
from paper_2210_07768_b200.workloads import workload_config  # noqa: E402

marks = []
T0 = [0.0]


def mark(name):
    marks.append((time.perf_counter() - T0[0], threading.current_thread().name, name))


def wrap(owner, attr, label):
    f = getattr(owner, attr)

    def g(*a, **k):
        mark(label + " >")
        try:
            return f(*a, **k)
        finally:
            mark(label + " <")
    setattr(owner, attr, g)


wrap(E, "_prepared", "plan")
wrap(S.FileRun, "__init__", "FileRun.init")
wrap(E.DeviceView, "from_file", "from_file")
wrap(E.Engine, "__init__", "Engine.init")
wrap(E.Engine, "reserve", "reserve")
wrap(E.Engine, "begin_run", "begin_run")
wrap(E.Engine, "launch", "launch")
wrap(S.FileRun, "run", "stream.run")
wrap(E.Engine, "_read_state", "read_state")
wrap(runtime, "read_spans", "pread")

d = Path(tempfile.mkdtemp())
gen_corpus(d, rows=1_000_000, users=5_000, seed=11)
cfg = config_from_dict(workload_config("sign_heavy"), d)
for _ in range(3):
    E.run_pipelined(cfg)
orig_run = S.FileRun.run
cap = {}


def run_capture(self, eng):
    cap["fr"] = self
    return orig_run(self, eng)


S.FileRun.run = run_capture
torch.cuda.synchronize()
ref = torch.cuda.Event(enable_timing=True)
marks.clear()
T0[0] = time.perf_counter()
ref.record()
rep = E.run_pipelined(cfg)
total = time.perf_counter() - T0[0]
for t, th, name in marks:
    print(f"{t * 1e3:8.3f} ms  {th:10s} {name}")
fr = cap["fr"]
for k in range(len(fr.bounds)):
    print(f"slice {k}: H2D {ref.elapsed_time(fr.h2d_start[k]):.3f}-{ref.elapsed_time(fr.h2d_done[k]):.3f} "
          f"kernel {ref.elapsed_time(fr.comp_start[k]):.3f}-{ref.elapsed_time(fr.comp_done[k]):.3f} ms")
print(f"total {total * 1e3:.3f} ms", hex(rep.digest))
