"""ptxas register / spill summary of fbx_pipeline for a DAG (CPU; NVRTC --ptxas-options=-v).

    FBX_SORT_ROWS=1 python scripts/ptxas_info.py cross_heavy
"""
import ctypes
import os
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2210_07768_b200 import codegen, engine, runtime  # noqa: E402
from paper_2210_07768_b200.config import config_from_dict  # noqa: E402
from paper_2210_07768_b200.corpus import make_corpus, write_corpus  # noqa: E402
from paper_2210_07768_b200.workloads import workload_config, write_lookup_tables  # noqa: E402

dag = sys.argv[1] if len(sys.argv) > 1 else "sign_heavy"
c = make_corpus(2000, 300, 7)
d = Path(tempfile.mkdtemp())
write_corpus(c, d)
write_lookup_tables(d, 300, 1000)
p = engine.prepare(config_from_dict(workload_config(dag), d),
                   {"user_events": c.driver, "user_profile": c.profile}, c.basic,
                   compile_program=False)
src = p.program.source
opts = ("-arch=sm_100a", "-std=c++17", "-lineinfo", "-diag-suppress=177,550", "--ptxas-options=-v",
        *os.environ.get("FBX_NVRTC_OPTS", "").split())
arr = (ctypes.c_char_p * len(opts))(*[o.encode() for o in opts])
img, n = ctypes.c_void_p(), ctypes.c_size_t()
log = ctypes.create_string_buffer(1 << 20)
runtime.lib().fbx_compile(src.encode(), b"plan.cu", arr, len(opts), ctypes.byref(img),
                          ctypes.byref(n), log, len(log))
lines = log.value.decode().splitlines()
for i, ln in enumerate(lines):
    if "fbx_pipeline" in ln and "Function properties" in ln:
        print(dag, "|", lines[i + 1].strip(), "|", lines[i + 2].strip())
print("dyn smem", p.program.smem_bytes)
