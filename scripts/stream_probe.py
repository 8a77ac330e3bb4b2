"""FileRun timeline on a 1M-record log: per-slice read / H2D / kernel times and a
bare H2D of the same pinned buffer (under gpurun)."""
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2210_07768_b200.config import config_from_dict  # noqa: E402
from paper_2210_07768_b200.corpus import gen_corpus  # noqa: E402
from paper_2210_07768_b200.engine import DeviceView, Engine, _prepared  # noqa: E402
from paper_2210_07768_b200.stream import FileRun  # noqa: E402
from paper_2210_07768_b200.workloads import workload_config  # noqa: E402

slice_rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
d = Path(tempfile.mkdtemp())
gen_corpus(d, rows=1_000_000, users=5_000, seed=11)
cfg = config_from_dict(workload_config("sign_heavy"), d)
prep = _prepared(cfg)
dvs = {"user_profile": DeviceView.from_file(cfg.view("user_profile").path),
       "basic": DeviceView.from_file(cfg.basic_path, cfg.basic_columns)}
eng = Engine(prep, device_views=dvs)
for rep in range(4):
    fr = FileRun(prep, cfg.view("user_events").path, cfg.view("user_events").columns,
                 slice_rows=slice_rows)
    eng.reserve(fr.n, fr.slice_rows, ring=True)
    eng.begin_run(fr.n)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t = fr.run(eng)
    wall = time.perf_counter() - t0
    st = eng._read_state()
    print(f"wall {wall * 1e3:.2f} ms read {t['read_s'] * 1e3:.2f} h2d {t['h2d_s'] * 1e3:.2f} "
          f"kernel {t['kernel_s'] * 1e3:.2f} bytes {t['h2d_bytes']} -> "
          f"{t['h2d_bytes'] / t['h2d_s'] / 1e9:.1f} GB/s  digest {st['digest']:#x}")
n = fr.cap - 64
s = torch.cuda.Stream()
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record(s)
        fr.dev[0][:n].copy_(fr.host[0][:n], non_blocking=True)
        b.record(s)
    s.synchronize()
    print(f"bare H2D of the staging buffer: {n / a.elapsed_time(b) / 1e6:.1f} GB/s ({n} B)")
