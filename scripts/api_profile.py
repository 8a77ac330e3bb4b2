"""cProfile of the drop-in run_pipelined on a 1M-record log (under gpurun): where
the host time of a call goes."""
import cProfile
import pstats
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2210_07768_b200.config import config_from_dict  # noqa: E402
from paper_2210_07768_b200.corpus import gen_corpus  # noqa: E402
from paper_2210_07768_b200.engine import run_pipelined  # noqa: E402
from paper_2210_07768_b200.workloads import workload_config  # noqa: E402

d = Path(tempfile.mkdtemp())
gen_corpus(d, rows=1_000_000, users=5_000, seed=11)
cfg = config_from_dict(workload_config("sign_heavy"), d)
for _ in range(3):
    run_pipelined(cfg)
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    run_pipelined(cfg)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(35)
st.sort_stats("tottime").print_stats(25)
