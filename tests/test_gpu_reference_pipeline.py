"""GPU: the reference's end-to-end pipeline scenarios (pkg/tests/test_pipeline.py:380-640)
restated against this package's public API -- a config built as the reference's
PipelineConfig, both modes, the report fields and the failures a user of the
reference relies on.  The tiny corpus's digest is recomputed here from first
principles (FNV-1a over the instance layout), not taken from either side."""

from __future__ import annotations

import dataclasses
from functools import reduce

import pytest

pytestmark = pytest.mark.gpu

MASK64 = (1 << 64) - 1
# (instance_id, label, query, basic_a); instance 3 has no basic row: the inner
# merge drops it
TINY = [(1, 0, "red shoes", 1000), (2, 1, "", 2000), (3, 1, "blue", None),
        (4, 0, "green hat", 4000)]


def _fnv(data: bytes) -> int:
    return reduce(lambda h, b: ((h ^ b) * 0x100000001B3) & MASK64, data, 0xCBF29CE484222325)


def _write(tmp, driver_rows, basic_rows):
    from paper_2210_07768_b200.columns import Kind, ViewImage, write_view
    drv = ViewImage.from_pydict(
        [("instance_id", Kind.INT64), ("label", Kind.INT64), ("query", Kind.UTF8)],
        {"instance_id": [r[0] for r in driver_rows], "label": [r[1] for r in driver_rows],
         "query": [r[2] for r in driver_rows]}, ("instance_id",))
    write_view(drv, tmp / "events.fbxc")
    bas = ViewImage.from_pydict(
        [("instance_id", Kind.INT64), ("basic_a", Kind.INT64)],
        {"instance_id": [r[0] for r in basic_rows], "basic_a": [r[1] for r in basic_rows]},
        ("instance_id",))
    write_view(bas, tmp / "basic.fbxc")


def _config(tmp, rows=TINY, **kw):
    from paper_2210_07768_b200 import FunctionRef, OperatorSpec
    from paper_2210_07768_b200.config import CleanPolicy, PipelineConfig, ViewSource
    _write(tmp, rows, [(r[0], r[3]) for r in rows if r[3] is not None])
    base = dict(views=(ViewSource("events", tmp / "events.fbxc", None,
                                  CleanPolicy(fills={"query": ""})),),
                driver="events", basic_path=tmp / "basic.fbxc",
                operators=(OperatorSpec(name="q_sig", inputs=("query",), outputs=("q_sig",),
                                        body=FunctionRef("hash:11")),),
                tables={}, features={"q_sig": 3, "basic_a": 7}, batch_size=2,
                staging_dir=tmp / "staging")
    base.update(kw)
    return PipelineConfig(**base)


def _expected_digest(rows=TINY) -> int:
    d = 0
    for iid, label, query, basic_a in rows:
        if basic_a is None:
            continue
        sig = _fnv((11).to_bytes(2, "big") + query.encode())  # hash:11 over the query
        msg = iid.to_bytes(8, "little") + bytes([label & 1])
        for slot, sign in sorted({(3, sig), (7, basic_a)}):
            msg += slot.to_bytes(2, "little") + sign.to_bytes(8, "little")
        d ^= _fnv(msg)
    return d


def _run(config, mode):
    from paper_2210_07768_b200.engine import run_pipeline
    return run_pipeline(config, mode=mode)


def test_tiny_digest_from_first_principles(tmp_path):
    cfg = _config(tmp_path)
    for mode in ("staged", "pipelined"):
        rep = _run(cfg, mode)
        assert rep.digest == _expected_digest(), mode
        assert (rep.instances, rep.batches, rep.signs) == (3, 2, 6), mode


def test_tiny_intermediates(tmp_path):
    cfg = _config(tmp_path)
    staged = _run(cfg, "staged")
    assert staged.intermediate_files == ("cleaned_events.fbxc", "extracted.fbxc",
                                         "merged.fbxc")
    on_disk = sum(f.stat().st_size for f in cfg.staging_dir.iterdir())
    assert staged.intermediate_bytes_written == on_disk > 0
    piped = _run(cfg, "pipelined")
    assert piped.intermediate_bytes_written == 0 and piped.intermediate_files == ()


def test_staged_needs_staging_dir_pipelined_does_not(tmp_path):
    from paper_2210_07768_b200.config import ConfigError
    cfg = _config(tmp_path, staging_dir=None)
    with pytest.raises(ConfigError, match="staging_dir"):
        _run(cfg, "staged")
    _run(cfg, "pipelined")


def test_mode_dispatch_and_override(tmp_path):
    from paper_2210_07768_b200.config import ConfigError
    from paper_2210_07768_b200.engine import run_pipeline
    cfg = _config(tmp_path, mode="staged")
    assert run_pipeline(cfg).mode == "staged"
    assert run_pipeline(cfg, mode="pipelined").mode == "pipelined"
    with pytest.raises(ConfigError, match="mode"):
        run_pipeline(cfg, mode="warp")


def test_corrupt_driver_body_fails_staged_clean(tmp_path):
    from paper_2210_07768_b200.columns import ChecksumError
    from paper_2210_07768_b200.config import StageError
    cfg = _config(tmp_path)
    blob = bytearray((tmp_path / "events.fbxc").read_bytes())
    blob[-20] ^= 0xFF  # a body byte: the full read's checksum catches it
    (tmp_path / "events.fbxc").write_bytes(blob)
    with pytest.raises(StageError) as exc:
        _run(cfg, "staged")
    assert exc.value.stage == "clean" and isinstance(exc.value.__cause__, ChecksumError)


def test_null_label_fails_emit(tmp_path):
    from paper_2210_07768_b200.config import EmitError, StageError
    cfg = _config(tmp_path, rows=[(1, None, "x", 5)])
    with pytest.raises(StageError) as exc:
        _run(cfg, "staged")
    assert exc.value.stage == "emit" and isinstance(exc.value.__cause__, EmitError)
    with pytest.raises(StageError) as exc2:
        _run(cfg, "pipelined")
    assert exc2.value.stage in {"merge", "emit"}
    assert isinstance(exc2.value.__cause__, EmitError)


def test_duplicate_driver_ids_fail_merge(tmp_path):
    from paper_2210_07768_b200.config import StageError
    cfg = _config(tmp_path, rows=[(5, 0, "a", 1), (5, 1, "b", None)])
    for mode in ("staged", "pipelined"):
        with pytest.raises(StageError) as exc:
            _run(cfg, mode)
        assert exc.value.stage == "merge", mode


def test_missing_basic_file_is_a_config_error(tmp_path):
    from paper_2210_07768_b200.config import ConfigError
    cfg = _config(tmp_path)
    (tmp_path / "basic.fbxc").unlink()
    for mode in ("staged", "pipelined"):
        with pytest.raises(ConfigError, match="basic"):
            _run(cfg, mode)


def test_giant_batch_size_is_one_batch(tmp_path):
    cfg = _config(tmp_path, batch_size=10 ** 6)
    rep = _run(cfg, "pipelined")
    assert rep.batches == 1 and rep.instances == 3 and rep.digest == _expected_digest()


def test_everything_filtered_is_an_empty_run(tmp_path):
    from paper_2210_07768_b200.config import CleanPolicy, parse_filter
    cfg = _config(tmp_path)
    strict = dataclasses.replace(cfg.views[0], policy=CleanPolicy(
        fills={"query": ""}, filter=parse_filter("instance_id > 999999")))
    cfg = dataclasses.replace(cfg, views=(strict,))
    for mode in ("staged", "pipelined"):
        rep = _run(cfg, mode)
        assert (rep.batches, rep.instances, rep.digest, rep.rows_filtered) == (0, 0, 0, 4), mode


def test_worker_count_and_fusion_leave_results_unchanged(tmp_path):
    cfg = _config(tmp_path)
    base = _run(cfg, "pipelined")
    for kw in ({"workers": 1}, {"workers": 4}, {"fusion": "unfused"}):
        rep = _run(dataclasses.replace(cfg, **kw), "pipelined")
        assert (rep.digest, rep.instances, rep.signs) == (base.digest, base.instances,
                                                          base.signs), kw


def test_stage_timing_keys(tmp_path):
    """pkg/tests/test_pipeline.py:576-582: the staged run times exactly its five
    stages; the pipelined run reports at least the reference's seven keys."""
    from conftest import corpus
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.workloads import workload_config
    _, d = corpus(2000, 300, 7)
    cfg = config_from_dict(dict(workload_config("default"), staging_dir=str(tmp_path / "s")), d)
    assert set(_run(cfg, "staged").stage_seconds) == {"clean", "join", "extract", "merge",
                                                      "emit"}
    keys = {"prepare", "read", "clean", "join", "extract", "merge", "emit"}
    assert keys <= set(_run(cfg, "pipelined").stage_seconds)
    assert keys <= set(_run(dataclasses.replace(cfg, batch_size=4096), "pipelined").stage_seconds)
