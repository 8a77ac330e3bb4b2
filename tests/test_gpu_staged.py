"""GPU: the staged mode (pipeline.run_staged, pipeline.py:783-895) on the B200
against the UNMODIFIED reference's own staged run (baseline/_ref, CPU): the
same report (digest, counts, intermediate file names and bytes) and every
intermediate FBXC file byte-identical -- cleaned views, the joined, extracted
and merged tables -- and failures raised at the same stage."""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import pytest

from conftest import reference_package_path

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(reference_package_path() is None,
                               reason="reference package not installed (baseline/_ref)")

DAGS = ("default", "fig4", "sign_heavy", "cross_heavy", "lookup_heavy")


def _ref():
    p = str(reference_package_path())
    if p not in sys.path:
        sys.path.insert(0, p)
    import featurebox.corpus as RC
    import featurebox.pipeline as P
    return P, RC


def _both(raw: dict, d: Path):
    """(reference report | exception, B200 report | exception, ref dir, our dir)."""
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.engine import run_pipeline
    P, _ = _ref()
    sr, so = d / "stage_ref", d / "stage_b200"
    rr = dict(raw, mode="staged", staging_dir=str(sr))
    (d / "cfg_ref.json").write_text(json.dumps(rr))
    try:
        ref = P.run_pipeline(P.load_config(d / "cfg_ref.json"))
    except Exception as exc:  # noqa: BLE001
        ref = exc
    try:
        got = run_pipeline(config_from_dict(dict(raw, mode="staged", staging_dir=str(so)), d))
    except Exception as exc:  # noqa: BLE001
        got = exc
    return ref, got, sr, so


def _digest(p: Path) -> str:
    return hashlib.sha256(p.read_bytes()).hexdigest()


@needs_ref
@pytest.mark.parametrize("dag", DAGS)
def test_staged_matches_reference_files(dag):
    from paper_2210_07768_b200.workloads import workload_config, write_lookup_tables
    _, RC = _ref()
    d = Path(tempfile.mkdtemp(prefix="fbxstaged"))
    RC.gen_corpus(d, rows=2000, users=300, seed=7, views=2)
    write_lookup_tables(d, 300)
    ref, got, sr, so = _both(workload_config(dag), d)
    assert not isinstance(ref, Exception), ref
    assert not isinstance(got, Exception), got
    for f in ("digest", "batches", "instances", "signs", "rows_dropped", "rows_filtered",
              "intermediate_files", "intermediate_bytes_written", "batch_size", "mode"):
        assert getattr(got, f) == getattr(ref, f), f
    for name in ref.intermediate_files:
        assert _digest(so / name) == _digest(sr / name), name


@needs_ref
def test_staged_equals_pipelined_digest():
    """The reference's promise: both modes give the same digest."""
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.engine import run_pipeline
    from paper_2210_07768_b200.workloads import workload_config
    _, RC = _ref()
    d = Path(tempfile.mkdtemp(prefix="fbxstaged"))
    RC.gen_corpus(d, rows=5000, users=500, seed=11, views=2)
    raw = workload_config("sign_heavy")
    a = run_pipeline(config_from_dict(dict(raw, mode="staged", staging_dir=str(d / "s")), d))
    b = run_pipeline(config_from_dict(raw, d))
    assert (a.digest, a.instances, a.signs, a.batches) == (b.digest, b.instances, b.signs,
                                                           b.batches)


def _edge_dir(mutate):
    import test_gpu_edge as T
    d = Path(tempfile.mkdtemp(prefix="fbxstagededge"))
    drv, prof, bas = mutate(*T._views(2000, 5))
    T._write_views(d, drv, prof, bas)
    return d


@needs_ref
@pytest.mark.parametrize("case", ["adversarial", "dup_ids", "bad_label", "null_label",
                                  "basic_dup"])
def test_staged_edge_cases_match_reference(case):
    """Adversarial records (JSON corners, fills, filters, Json-kind leaves) and the
    failures of the later stages: a repeated id (merge), a bad / null label
    (emit), a repeated basic id (merge) -- same stage, same cause."""
    import test_gpu_edge as T
    from paper_2210_07768_b200.config import StageError
    muts = {"adversarial": lambda *v: v,
            "dup_ids": T._set_ids([(1500, 1400), (702, 1400)]),
            "bad_label": T._set_labels([505], 3),
            "null_label": T._set_labels([1030], None),
            "basic_dup": T._basic_dup(5, 6)}
    d = _edge_dir(muts[case])
    raw = T._config(512, T.OPS, T.FEATS) if case == "adversarial" else \
        T._config(512, [{"name": "c", "inputs": ["query"], "outputs": ["c"],
                         "body": {"fn": "hash:3"}}], {"c": 3}, filt="age != -12345")
    ref, got, sr, so = _both(raw, d)
    if isinstance(ref, Exception):
        assert isinstance(got, StageError), got
        assert (got.stage, got.batch_index) == (ref.stage, ref.batch_index)
        assert type(got.__cause__).__name__ == type(ref.__cause__).__name__
        assert str(got.__cause__) == str(ref.__cause__)
        return
    assert not isinstance(got, Exception), got
    assert (got.digest, got.instances, got.signs) == (ref.digest, ref.instances, ref.signs)
    for name in ref.intermediate_files:
        assert _digest(so / name) == _digest(sr / name), name
