"""Per-shard reference goldens for C5 and the weak-scaling ranks (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_shard_goldens.py [--procs 6]

Runs the UNMODIFIED reference, one independent pipeline per shard, on CPU
processes:

* C5 (SURVEY.md §8 d): seeds 1000..1099, 1M rows / 5000 users each, the
  reference's own generated ``pipeline.json`` (default DAG, full emit);
* weak-scaling ranks of ``bench.py`` (one 1M-row log per rank, seed 11 + r):
  seeds 12..18 through the default DAG and through sign_heavy (seed 11 is in
  SURVEY Appendix B / goldens.json).

Each shard's corpus comes from the reference's ``gen_corpus`` and its files are
hashed, so the repo's C generator (``corpus.gen_corpus_fast``) can be checked
byte for byte before the GPU box regenerates the shard.  Results are appended
to ``shard_goldens.jsonl`` one line per shard as they finish (the script
resumes where it stopped); ``shard_goldens.json`` is the sorted summary with
the C5 XOR digest.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import multiprocessing as mp
import platform
import shutil
import sys
import tempfile
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, "/root/reference/pkg/src")

JSONL = HERE / "shard_goldens.jsonl"
SUMMARY = HERE / "shard_goldens.json"

ROWS, USERS = 1_000_000, 5000


def jobs():
    out = [("default", s) for s in range(11, 19)]  # seed 11 re-checks SURVEY App. B
    out += [("sign_heavy", s) for s in range(12, 19)]
    out += [("default", s) for s in range(1000, 1100)]
    return out


def run_one(job):
    dag, seed = job
    from featurebox.corpus import gen_corpus
    from featurebox.pipeline import load_config, run_pipelined

    from paper_2210_07768_b200.workloads import workload_config

    tmp = Path(tempfile.mkdtemp(prefix=f"fbx_shard_{dag}_{seed}_"))
    try:
        t0 = time.time()
        files = gen_corpus(tmp, rows=ROWS, users=USERS, seed=seed, views=2)
        sha = {k: hashlib.sha256(Path(v).read_bytes()).hexdigest() for k, v in files.items()}
        t1 = time.time()
        if dag == "default":
            cfg_path = tmp / "pipeline.json"  # the reference's own generated config
        else:
            cfg_path = tmp / "cfg.json"
            cfg_path.write_text(json.dumps(workload_config(dag)))
        rep = run_pipelined(load_config(cfg_path))
        t2 = time.time()
        return {"dag": dag, "seed": seed, "rows": ROWS, "users": USERS,
                "digest": f"0x{rep.digest:016x}", "instances": rep.instances,
                "signs": rep.signs, "batches": rep.batches,
                "rows_dropped": rep.rows_dropped, "rows_filtered": rep.rows_filtered,
                "corpus_sha256": sha, "gen_s": round(t1 - t0, 1), "run_s": round(t2 - t1, 1)}
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def summarise():
    rows = [json.loads(x) for x in JSONL.read_text().splitlines() if x.strip()]
    rows.sort(key=lambda r: (r["dag"], r["seed"]))
    c5 = [r for r in rows if r["dag"] == "default" and 1000 <= r["seed"] < 1100]
    x = 0
    for r in c5:
        x ^= int(r["digest"], 16)
    out = {"python": platform.python_version(),
           "generator": "reference featurebox.corpus.gen_corpus + featurebox.pipeline.run_pipelined",
           "c5": {"shards": len(c5), "xor_digest": f"0x{x:016x}",
                  "instances": sum(r["instances"] for r in c5),
                  "signs": sum(r["signs"] for r in c5),
                  "rows": sum(r["rows"] for r in c5)},
           "shards": rows}
    SUMMARY.write_text(json.dumps(out, indent=1) + "\n")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=6)
    ap.add_argument("--summary-only", action="store_true")
    a = ap.parse_args()
    if not a.summary_only:
        done = set()
        if JSONL.exists():
            for line in JSONL.read_text().splitlines():
                if line.strip():
                    r = json.loads(line)
                    done.add((r["dag"], r["seed"]))
        todo = [j for j in jobs() if j not in done]
        print(f"{len(todo)} shards to run on {a.procs} processes", flush=True)
        with mp.get_context("spawn").Pool(a.procs, maxtasksperchild=1) as pool:
            for r in pool.imap_unordered(run_one, todo):
                with open(JSONL, "a") as fh:
                    fh.write(json.dumps(r) + "\n")
                print(r["dag"], r["seed"], r["digest"], r["instances"], r["run_s"], flush=True)
    s = summarise()
    print(json.dumps(s["c5"]))


if __name__ == "__main__":
    main()
