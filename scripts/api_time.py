"""Wall time of the drop-in run_pipelined(load_config(...)) over a 1M-record corpus on disk (under gpurun)."""
import sys, time, tempfile
from pathlib import Path
sys.path.insert(0, "/root/repo")
from paper_2210_07768_b200 import load_config, run_pipelined
from paper_2210_07768_b200.corpus import gen_corpus
d = Path(tempfile.mkdtemp())
t = time.time(); paths = gen_corpus(d, rows=1_000_000, users=5_000, seed=11); print("gen", round(time.time() - t, 2))
cfg = load_config(paths["config"])
for i in range(3):
    t = time.time(); rep = run_pipelined(cfg); dt = time.time() - t
    print(f"run_pipelined {dt:.3f} s -> {1e6/dt/1e6:.2f} M rec/s", hex(rep.digest), rep.instances)
