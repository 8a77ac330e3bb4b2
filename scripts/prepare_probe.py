"""Where run_pipelined's prepare phase goes (1M-record log, under gpurun)."""
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2210_07768_b200.config import config_from_dict  # noqa: E402
from paper_2210_07768_b200.corpus import gen_corpus  # noqa: E402
from paper_2210_07768_b200.engine import DeviceView, Engine, _prepared  # noqa: E402
from paper_2210_07768_b200.workloads import workload_config  # noqa: E402

d = Path(tempfile.mkdtemp())
gen_corpus(d, rows=1_000_000, users=5_000, seed=11)
cfg = config_from_dict(workload_config("sign_heavy"), d)
for rep in range(4):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    prep = _prepared(cfg)
    t.append(time.perf_counter())
    p = DeviceView.from_file(cfg.view("user_profile").path, cfg.view("user_profile").columns)
    t.append(time.perf_counter())
    b = DeviceView.from_file(cfg.basic_path, cfg.basic_columns)
    t.append(time.perf_counter())
    eng = Engine(prep, device_views={"user_profile": p, "basic": b})
    t.append(time.perf_counter())
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    print("plan {:.2f} profile {:.2f} basic {:.2f} engine {:.2f} sync {:.2f} ms".format(
        *[(t[i + 1] - t[i]) * 1e3 for i in range(len(t) - 1)]))

# the basic ingest step by step
from paper_2210_07768_b200 import runtime  # noqa: E402
from paper_2210_07768_b200.columns import open_view  # noqa: E402
from paper_2210_07768_b200.engine import crc32_device  # noqa: E402
for rep in range(3):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    vf = open_view(cfg.basic_path)
    t.append(time.perf_counter())
    host = torch.empty(vf.body_bytes + 16, dtype=torch.uint8, pin_memory=True)
    t.append(time.perf_counter())
    runtime.read_spans(vf.path, host.data_ptr(), [vf.body_offset], [vf.body_bytes], [0])
    t.append(time.perf_counter())
    body = torch.empty(vf.body_bytes + 64, dtype=torch.uint8, device="cuda")
    body[:vf.body_bytes].copy_(host[:vf.body_bytes], non_blocking=True)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    crc = crc32_device(body[:vf.body_bytes])
    t.append(time.perf_counter())
    print("open {:.2f} pin {:.2f} read {:.2f} h2d {:.2f} crc {:.2f} ms".format(
        *[(t[i + 1] - t[i]) * 1e3 for i in range(len(t) - 1)]), vf.body_bytes, crc == vf.checksum)
