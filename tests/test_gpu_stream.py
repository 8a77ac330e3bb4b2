"""GPU: the drop-in run_pipelined over files -- the driver streamed from its FBXC
file in slices (parallel pread -> pinned ring -> H2D -> fused kernel, CSR in a
one-slice ring) -- against the reference goldens and the oracle, failures
placed like the reference across slice boundaries."""

from __future__ import annotations

import pytest

import featurebox_oracle as O
from conftest import corpus, golden_run
from test_gpu_edge import (PLACEMENT, POOL_FEATS, POOL_OPS, _config, _views, _write_views)

pytestmark = pytest.mark.gpu

DAGS = ("default", "fig4", "sign_heavy", "cross_heavy", "lookup_heavy")


def _cfg(dag, d, batch_size=512):
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.workloads import workload_config
    return config_from_dict(workload_config(dag, batch_size=batch_size), d)


@pytest.mark.parametrize("dag", DAGS)
@pytest.mark.parametrize("slice_rows", [4096, 1 << 18])
def test_streamed_run_pipelined_matches_goldens(dag, slice_rows, goldens):
    from paper_2210_07768_b200.engine import run_pipelined
    _, d = corpus(20000, 2000, 7)
    rep = run_pipelined(_cfg(dag, d), slice_rows=slice_rows)
    g = golden_run(goldens, 20000, 7, dag)
    assert f"0x{rep.digest:016x}" == g["digest"]
    assert (rep.instances, rep.signs, rep.batches) == (g["instances"], g["signs"], g["batches"])
    assert (rep.rows_dropped, rep.rows_filtered) == (g["rows_dropped"], g["rows_filtered"])
    assert rep.bytes_h2d > 0 and rep.launches > 0
    for k in ("prepare", "read", "transfer", "extract"):
        assert k in rep.stage_seconds


def test_file_run_memory_is_one_slice(goldens):
    """Bounded memory: the CSR arena and the staging buffers hold one slice."""
    from paper_2210_07768_b200.engine import DeviceView, Engine, _prepared
    from paper_2210_07768_b200.stream import FileRun
    _, d = corpus(20000, 2000, 7)
    cfg = _cfg("sign_heavy", d)
    prep = _prepared(cfg)
    dvs = {"user_profile": DeviceView.from_file(cfg.view("user_profile").path,
                                                cfg.view("user_profile").columns),
           "basic": DeviceView.from_file(cfg.basic_path, cfg.basic_columns)}
    eng = Engine(prep, device_views=dvs)
    fr = FileRun(prep, cfg.view("user_events").path, cfg.view("user_events").columns,
                 slice_rows=2048)
    eng.reserve(fr.n, fr.slice_rows, ring=True)
    eng.begin_run(fr.n)
    t = fr.run(eng)
    st = eng._read_state()
    eng.check_run(st)
    g = golden_run(goldens, 20000, 7, "sign_heavy")
    assert f"0x{st['digest']:016x}" == g["digest"] and st["instances"] == g["instances"]
    # 2048-row slices, the last one split into a short tail (FileRun's taper)
    assert t["slices"] == len(fr.bounds) == 11 and fr.bounds[-1] == (19456, 20000)
    assert eng.o_ids.numel() <= 2048 + 1 and eng.o_sign.numel() <= 2048 * 13 + 1
    assert len(fr.host) == 3 and fr.cap < 2048 * 200
    # the last slice's CSR sits at the start of the ring with launch-local offsets
    assert int(eng.o_off[0].item()) == 0


def _oracle(raw, drv, prof, bas, tmp):
    tables, sizes = O.load_tables(raw.get("tables", {}), tmp)
    try:
        return O.run_pipelined(raw, {"ev": drv, "pr": prof}, bas, tables, sizes), None
    except O.OracleError as e:
        return None, e


def _streamed(raw, tmp, slice_rows):
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.engine import run_pipelined
    try:
        return run_pipelined(config_from_dict(raw, tmp), slice_rows=slice_rows), None
    except Exception as e:  # noqa: BLE001
        return None, e


@pytest.mark.parametrize("case", sorted(PLACEMENT))
@pytest.mark.parametrize("batch_size,slice_rows", [(100, 300), (512, 512), (64, 1024)])
def test_streamed_failure_placement(case, batch_size, slice_rows, tmp_path):
    drv, prof, bas = PLACEMENT[case](*_views(2000, 5))
    _write_views(tmp_path, drv, prof, bas)
    ops = [{"name": "c", "inputs": ["query"], "outputs": ["c"], "body": {"fn": "hash:3"}}]
    raw = _config(batch_size, ops, {"c": 3}, filt="age != -12345")
    _, ref_err = _oracle(raw, drv, prof, bas, tmp_path)
    _, got_err = _streamed(raw, tmp_path, slice_rows)
    assert ref_err is not None and got_err is not None
    assert (got_err.stage, got_err.batch_index) == (ref_err.stage, ref_err.chunk)


@pytest.mark.parametrize("pool,lpg,batch_size", [(128, 256, 512), (1024, 7, 64), (4096, 256, 512),
                                                 (8 << 20, 256, 512), (3200, 7, 64)])
def test_streamed_pool_bytes(pool, lpg, batch_size, tmp_path):
    """The reference arena's PoolExhausted settled per slice (fbx_pool_account
    after each launch of the ring)."""
    drv, prof, bas = _views(2000, 9)
    _write_views(tmp_path, drv, prof, bas)
    raw = _config(batch_size, POOL_OPS, POOL_FEATS, filt="age != -12345")
    raw["device"] = {"budget_bytes": 65536, "pool_bytes": pool, "lanes_per_group": lpg}
    ref, ref_err = _oracle(raw, drv, prof, bas, tmp_path)
    got, got_err = _streamed(raw, tmp_path, 4 * batch_size)
    if ref_err is None:
        assert got_err is None, got_err
        assert (got.digest, got.instances, got.signs) == (ref.digest, ref.instances, ref.signs)
        return
    assert got_err is not None
    assert (got_err.stage, got_err.batch_index) == (ref_err.stage, ref_err.chunk)
    lay = got_err.__cause__
    assert (lay.layer_index, lay.node) == (ref_err.layer, ref_err.node)
    if type(ref_err.cause).__name__ == "PoolExhausted":
        assert (lay.__cause__.requested, lay.__cause__.remaining) == \
            (ref_err.cause.requested, ref_err.cause.remaining)


@pytest.mark.parametrize("batch_size,seed", [(512, 1), (64, 2), (7, 3), (1500, 4), (20000, 6)])
def test_streamed_adversarial_records(batch_size, seed, tmp_path):
    """Adversarial records (JSON corners, nulls, filters) through the file stream;
    batch_size > 1024 and a single whole-file chunk take the device-resident path."""
    from test_gpu_edge import FEATS, OPS
    drv, prof, bas = _views(3000, seed)
    _write_views(tmp_path, drv, prof, bas)
    raw = _config(batch_size, OPS, FEATS)
    ref, ref_err = _oracle(raw, drv, prof, bas, tmp_path)
    got, got_err = _streamed(raw, tmp_path, 1024)
    if ref_err is not None:
        assert got_err is not None and got_err.stage == ref_err.stage
        return
    assert got_err is None, got_err
    assert (got.digest, got.instances, got.signs) == (ref.digest, ref.instances, ref.signs)
    assert (got.rows_dropped, got.rows_filtered) == (ref.malformed, ref.filtered)


@pytest.mark.parametrize("which", ["basic.fbxc", "pr.fbxc"])
def test_streamed_checksum_error_is_prepare_failure(which, tmp_path):
    """A corrupted side / basic body (full read) fails prepare with the
    reference's ChecksumError -- checked on the device, raised after the stream."""
    from paper_2210_07768_b200.columns import ChecksumError
    from paper_2210_07768_b200.config import StageError
    drv, prof, bas = _views(2000, 5)
    _write_views(tmp_path, drv, prof, bas)
    f = tmp_path / which
    raw = bytearray(f.read_bytes())
    raw[-9] ^= 0x40  # a body byte (the last 4 bytes are the CRC trailer)
    f.write_bytes(bytes(raw))
    ops = [{"name": "c", "inputs": ["query"], "outputs": ["c"], "body": {"fn": "hash:3"}}]
    _, err = _streamed(_config(512, ops, {"c": 3}, filt="age != -12345"), tmp_path, 512)
    assert isinstance(err, StageError) and err.stage == "prepare"
    assert isinstance(err.__cause__, ChecksumError)


@pytest.mark.parametrize("rows", [0, 1, 511, 513])
def test_streamed_tiny_and_empty_logs(rows, tmp_path):
    """Empty and tiny driver files through the file stream (one partial chunk,
    a chunk boundary, no rows at all) equal the oracle."""
    drv, prof, bas = _views(max(rows, 1), 3)
    if rows == 0:
        drv = drv.slice(0, 0)
    _write_views(tmp_path, drv, prof, bas)
    ops = [{"name": "c", "inputs": ["query"], "outputs": ["c"], "body": {"fn": "hash:3"}}]
    raw = _config(512, ops, {"c": 3}, filt="age != -12345")
    ref, ref_err = _oracle(raw, drv, prof, bas, tmp_path)
    got, got_err = _streamed(raw, tmp_path, 512)
    if ref_err is not None:
        assert got_err is not None and got_err.stage == ref_err.stage
        return
    assert got_err is None, got_err
    assert (got.digest, got.instances, got.signs, got.batches) == \
        (ref.digest, ref.instances, ref.signs, -(-ref.instances // 512))
