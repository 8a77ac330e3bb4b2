"""GPU: the C-ABI engine object (include/fbx.h: fbx_create / fbx_extract /
fbx_emit_csr / fbx_last_error) and the reference-side shim that puts it in the
seat of the reference's own ``featurebox.pipeline._extract_batch``.

The shim tests run the UNMODIFIED reference (baseline/_ref, pip-installed from
/root/reference; or /root/reference itself) end to end -- its own clean, join,
merge, emit and digest -- with only ``_extract_batch`` replaced, and compare
with the reference's published / generated goldens."""

from __future__ import annotations

import json
import random
import sys
import tempfile
from pathlib import Path

import numpy as np
import pytest

import featurebox_oracle as O
from conftest import golden_run, reference_package_path

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(reference_package_path() is None,
                               reason="reference package not installed (baseline/_ref)")


def _ref():
    p = str(reference_package_path())
    if p not in sys.path:
        sys.path.insert(0, p)
    import featurebox.corpus as RC
    import featurebox.pipeline as P
    return P, RC


def _ref_run(P, cfg_path):
    return P.run_pipelined(P.load_config(cfg_path))


@needs_ref
@pytest.mark.parametrize("dag", ["default", "fig4", "sign_heavy", "cross_heavy", "lookup_heavy"])
def test_shim_reference_pipeline_equals_golden(dag, goldens):
    """20k rows / 2000 users / seed 7 through the reference's
    own run_pipelined with the B200 engine as its _extract_batch."""
    from paper_2210_07768_b200 import refshim
    from paper_2210_07768_b200.workloads import workload_config, write_lookup_tables
    P, RC = _ref()
    d = Path(tempfile.mkdtemp(prefix="fbxshim"))
    RC.gen_corpus(d, rows=20000, users=2000, seed=7, views=2)
    write_lookup_tables(d, 2000)
    cfg = d / "cfg.json"
    cfg.write_text(json.dumps(workload_config(dag)))
    refshim.install(P)
    try:
        rep = _ref_run(P, cfg)
    finally:
        refshim.uninstall(P)
    g = golden_run(goldens, 20000, 7, dag)
    assert f"0x{rep.digest:016x}" == g["digest"]
    assert (rep.instances, rep.signs, rep.batches) == (g["instances"], g["signs"], g["batches"])


@needs_ref
def test_shim_reference_published_run():
    """The reference's own acceptance run (gen_corpus 100k / 5k users / seed 11,
    its generated pipeline.json): digest 0xb2bcd7004cff26a0, 90,326 instances,
    177 batches, 517,976 signs (pkg/test_output.txt:19, 25)."""
    from paper_2210_07768_b200 import refshim
    P, RC = _ref()
    d = Path(tempfile.mkdtemp(prefix="fbxshim"))
    RC.gen_corpus(d, rows=100000, users=5000, seed=11, views=2)
    refshim.install(P)
    try:
        rep = _ref_run(P, d / "pipeline.json")
    finally:
        refshim.uninstall(P)
    assert (rep.digest, rep.instances, rep.batches, rep.signs) == \
        (0xB2BCD7004CFF26A0, 90326, 177, 517976)


@needs_ref
@pytest.mark.parametrize("pool,lpg", [(128, 256), (1024, 7), (8 << 20, 256)])
def test_shim_failures_equal_unpatched_reference(pool, lpg):
    """Failures surface exactly as the unpatched reference's: StageError stage and
    batch, LayerExecutionError layer / node, PoolExhausted bytes."""
    from paper_2210_07768_b200 import refshim
    P, RC = _ref()
    d = Path(tempfile.mkdtemp(prefix="fbxshim"))
    RC.gen_corpus(d, rows=3000, users=300, seed=5, views=2)
    raw = json.loads((d / "pipeline.json").read_text())
    raw["operators"].append({"name": "tq", "inputs": ["query"], "outputs": ["tq"],
                             "pre": [{"fn": "token: :1"}], "body": {"fn": "hash:21"}})
    raw["operators"].append({"name": "mx", "inputs": ["city_x"], "outputs": ["mx"],
                             "pre": [{"fn": "mix"}], "body": {"fn": "hash:22"}} if pool == 1024 else
                            {"name": "mx", "inputs": ["query"], "outputs": ["mx"],
                             "body": {"fn": "hash:22"}})
    raw["emit"]["features"].update({"tq": 21, "mx": 22})
    raw["device"].update({"pool_bytes": pool, "lanes_per_group": lpg})
    cfg = d / "cfg.json"
    cfg.write_text(json.dumps(raw))

    def run():
        try:
            return _ref_run(P, cfg), None
        except P.StageError as exc:
            return None, exc
    want, werr = run()
    refshim.install(P)
    try:
        got, gerr = run()
    finally:
        refshim.uninstall(P)
    if werr is None:
        assert gerr is None, gerr
        assert (got.digest, got.instances, got.signs) == (want.digest, want.instances, want.signs)
        return
    assert gerr is not None
    assert (gerr.stage, gerr.batch_index) == (werr.stage, werr.batch_index)
    wl, gl = werr.__cause__, gerr.__cause__
    assert type(gl).__name__ == type(wl).__name__ == "LayerExecutionError"
    assert (gl.layer_index, gl.node) == (wl.layer_index, wl.node)
    assert type(gl.__cause__).__name__ == type(wl.__cause__).__name__
    if type(wl.__cause__).__name__ == "PoolExhausted":
        assert (gl.__cause__.requested, gl.__cause__.remaining) == \
            (wl.__cause__.requested, wl.__cause__.remaining)


def _int_col(vals):
    from paper_2210_07768_b200.columns import ColumnImage, Kind
    return ColumnImage.from_values(Kind.INT64, vals)


def _emit_engine():
    from paper_2210_07768_b200.capi import CEngine
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.engine import prepare_extract
    from paper_2210_07768_b200.columns import Kind
    from paper_2210_07768_b200.workloads import workload_config
    raw = workload_config("sign_heavy")
    cfg = config_from_dict(raw, Path(tempfile.mkdtemp()))
    return CEngine(prepare_extract(cfg, {"query": Kind.UTF8, "city_x": Kind.UTF8,
                                         "city": Kind.UTF8, "age": Kind.INT64,
                                         "score": Kind.FLOAT32, "user_id": Kind.INT64}), 0)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_emit_csr_matches_oracle(seed):
    """fbx_emit_csr == emit_minibatch + batch_digest (pipeline.py:375-433): random
    signs, shared slots (a set), nulls, wrapped (negative) Int64 images."""
    rng = random.Random(seed)
    n, k = 700, 9
    slots = [rng.choice([3, 3, 5, 7, 9, 11, 40]) for _ in range(k)]
    feats = [[None if rng.random() < 0.2 else rng.choice([rng.getrandbits(64) - (1 << 63),
                                                          7, -7, 0]) for _ in range(n)]
             for _ in range(k)]
    ids = list({rng.getrandbits(64) - (1 << 63) for _ in range(n)})[:n]
    n = len(ids)
    feats = [f[:n] for f in feats]
    labels = [rng.choice([0, 1]) for _ in range(n)]
    eng = _emit_engine()  # (n rows after de-duplicating the random ids)
    out = eng.emit_csr(_int_col(ids), _int_col(labels),
                       [(_int_col(f), s) for f, s in zip(feats, slots)])
    want_sets = []
    dig = 0
    for i in range(n):
        pairs = sorted({(slots[q], feats[q][i] & ((1 << 64) - 1)) for q in range(k)
                        if feats[q][i] is not None})
        want_sets.append(pairs)
        dig ^= O.instance_digest(ids[i] & ((1 << 64) - 1), labels[i], pairs)
    assert out["digest"] == dig
    np.testing.assert_array_equal(out["ids"], np.array(ids, np.int64).view(np.uint64))
    np.testing.assert_array_equal(out["labels"], np.array(labels, np.uint8))
    offs = np.cumsum([0] + [len(p) for p in want_sets]).astype(np.uint64)
    np.testing.assert_array_equal(out["offsets"], offs)
    np.testing.assert_array_equal(out["slots"], np.array([s for p in want_sets for s, _ in p],
                                                         np.uint16))
    np.testing.assert_array_equal(out["signs"], np.array([g for p in want_sets for _, g in p],
                                                         np.uint64))


def test_emit_csr_failures_like_the_reference():
    from paper_2210_07768_b200.config import BatchInvariantError, EmitError
    eng = _emit_engine()
    f = [(_int_col([1, 2, 3, 4]), 3)]
    with pytest.raises(EmitError, match="null label"):
        eng.emit_csr(_int_col([1, 2, 3, 4]), _int_col([0, None, 1, 0]), f)
    with pytest.raises(EmitError, match="null instance id"):  # row order, id before label
        eng.emit_csr(_int_col([1, None, 3, 4]), _int_col([0, None, None, 0]), f)
    with pytest.raises(BatchInvariantError, match="duplicate"):
        eng.emit_csr(_int_col([1, 2, 1, 4]), _int_col([0, 5, 1, 0]), f)
    with pytest.raises(BatchInvariantError, match="label"):
        eng.emit_csr(_int_col([1, 2, 3, 4]), _int_col([0, 5, 1, 0]), f)


def test_last_error_locates_the_failing_node():
    """fbx_last_error(engine, &layer, &node): a TypeError of mix over a str is
    LayerExecutionError(layer 1, 'm.pre1') like device.py:402-403."""
    from paper_2210_07768_b200.capi import CEngine
    from paper_2210_07768_b200.columns import ColumnImage, Kind, ViewImage
    from paper_2210_07768_b200.config import LayerExecutionError, config_from_dict
    from paper_2210_07768_b200.engine import prepare_extract
    from paper_2210_07768_b200.workloads import workload_config
    raw = workload_config("default")
    raw["operators"] = [{"name": "m", "inputs": ["q"], "outputs": ["m"],
                         "pre": [{"fn": "mix"}], "body": {"fn": "hash:3"}}]
    raw["tables"] = {}
    cfg = config_from_dict(raw, Path(tempfile.mkdtemp()))
    eng = CEngine(prepare_extract(cfg, {"q": Kind.UTF8}), 0)
    table = ViewImage({"q": ColumnImage.from_values(Kind.UTF8, [None, "a", "b"])}, (), ("q",))
    with pytest.raises(LayerExecutionError) as ei:
        eng.extract(table)
    assert (ei.value.layer_index, ei.value.node) == (1, "m.pre1")
    assert isinstance(ei.value.__cause__, TypeError)
    ok = ViewImage({"q": ColumnImage.from_values(Kind.UTF8, [None, None])}, (), ("q",))
    out = eng.extract(ok)
    assert out.columns["m"].to_pylist() == [None, None]
    assert eng.counters.rows == 2 and eng.counters.launches >= 1
