"""Generate golden fixtures by running the UNMODIFIED reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``goldens.json`` (run digests and counters per corpus x DAG, full and
ops-only) and ``csr_<dag>.npz`` (the emitted mini-batches of the 2k corpus,
flattened to CSR in emission order).  The reference is imported from
/root/reference (read-only) and run from a temporary directory; its corpus
files come from its own ``gen_corpus``.  Python version is recorded.
"""

from __future__ import annotations

import hashlib
import json
import platform
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, "/root/reference/pkg/src")

import featurebox.pipeline as ref_pipeline  # noqa: E402
from featurebox.corpus import gen_corpus  # noqa: E402
from featurebox.pipeline import load_config, run_pipelined  # noqa: E402

from paper_2210_07768_b200.workloads import DAGS, workload_config, write_lookup_tables  # noqa: E402

CORPORA = [  # rows, users, seed, views
    (2000, 300, 7, 2),
    (20000, 2000, 7, 2),
    (1200, 200, 11, 1),
]


def run(dest: Path, cfg: dict, capture: bool):
    path = dest / "cfg.json"
    path.write_text(json.dumps(cfg))
    batches = []
    orig = ref_pipeline.TrainingSink.consume
    if capture:
        def consume(self, batch):
            batches.append(batch)
            return orig(self, batch)
        ref_pipeline.TrainingSink.consume = consume
    try:
        rep = run_pipelined(load_config(path))
    finally:
        ref_pipeline.TrainingSink.consume = orig
    return rep, batches


def to_csr(batches):
    ids, labels, offs, slots, signs = [], [], [0], [], []
    for b in batches:
        for i in range(len(b)):
            ids.append(b.ids[i])
            labels.append(b.labels[i])
            for s, g in b.features[i]:
                slots.append(s)
                signs.append(g)
            offs.append(len(slots))
    return {"ids": np.array(ids, np.uint64), "labels": np.array(labels, np.uint8),
            "offsets": np.array(offs, np.uint64), "slots": np.array(slots, np.uint16),
            "signs": np.array(signs, np.uint64),
            "batch_sizes": np.array([len(b) for b in batches], np.int64)}


def main():
    out = {"python": platform.python_version(), "runs": []}
    with tempfile.TemporaryDirectory() as tmp:
        for rows, users, seed, views in CORPORA:
            dest = Path(tmp) / f"c{rows}_{seed}_{views}"
            files = gen_corpus(dest, rows=rows, users=users, seed=seed, views=views)
            out.setdefault("corpus_sha256", {})[f"{rows}_{users}_{seed}_{views}"] = {
                k: hashlib.sha256(Path(v).read_bytes()).hexdigest() for k, v in files.items()}
            write_lookup_tables(dest, users)
            dags = DAGS if views == 2 else ("default",)
            for dag in dags:
                for ops_only in (False, True):
                    if views == 1:
                        cfg = json.loads((dest / "pipeline.json").read_text())
                        if ops_only:
                            cfg["emit"]["features"] = {c: s for c, s in cfg["emit"]["features"].items()
                                                       if not c.startswith("basic_")}
                    else:
                        cfg = workload_config(dag, ops_only=ops_only)
                    capture = rows == 2000 and not ops_only
                    rep, batches = run(dest, cfg, capture)
                    out["runs"].append({
                        "rows": rows, "users": users, "seed": seed, "views": views, "dag": dag,
                        "ops_only": ops_only, "digest": f"0x{rep.digest:016x}",
                        "instances": rep.instances, "signs": rep.signs, "batches": rep.batches,
                        "rows_dropped": rep.rows_dropped, "rows_filtered": rep.rows_filtered})
                    print(out["runs"][-1], flush=True)
                    if capture:
                        np.savez_compressed(HERE / f"csr_{dag}.npz", **to_csr(batches))
    (HERE / "goldens.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
