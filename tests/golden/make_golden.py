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


def extract_fixtures(dest: Path):
    """Reference `_extract_batch` over the whole cleaned + joined 2k table
    (what staged mode extracts, pipeline.py:839-845), one fixture per DAG."""
    from featurebox.columnstore import read_columns, write_view
    from featurebox.device import ExecContext, LaunchCostModel
    from featurebox.mempool import create_pool
    from featurebox.pipeline import _extract_batch, prepare
    from featurebox.viewpipe import JoinSpec, clean_views, join_views
    joined = None
    for dag in DAGS:
        path = dest / "cfg_x.json"
        path.write_text(json.dumps(workload_config(dag)))
        cfg = load_config(path)
        prep = prepare(cfg)
        if joined is None:
            drv = cfg.views[0]
            side = cfg.views[1]
            a, _ = read_columns(drv.path)
            b, _ = read_columns(side.path)
            joined = join_views(clean_views(a, drv.policy), clean_views(b, side.policy),
                                JoinSpec(cfg.join_keys))
            write_view(joined, HERE / "joined_2k.fbxc")
        ctx = ExecContext(cost_model=LaunchCostModel(3.45), pool=create_pool(64 << 20))
        out = _extract_batch(joined, prep, ctx)
        arrays = {}
        for col, kind, domain in prep.extract_outputs:
            vals = out.columns[col].to_pylist()
            arrays[col + ".null"] = np.array([v is None for v in vals], bool)
            if domain == "u64":
                arrays[col] = np.array([0 if v is None else v for v in vals], np.int64)
            else:
                blob = [b"" if v is None else v.encode("utf-8") for v in vals]
                arrays[col + ".offsets"] = np.cumsum([0] + [len(x) for x in blob]).astype(np.uint64)
                arrays[col] = np.frombuffer(b"".join(blob), np.uint8)
        np.savez_compressed(HERE / f"extract_{dag}.npz", **arrays)


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
            if rows == 2000 and views == 2:
                extract_fixtures(dest)
    (HERE / "goldens.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
