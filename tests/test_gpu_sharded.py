"""GPU: one log record-sharded over G ranks (sharded.py) gives the single run's
result -- the reference goldens' digest and counters -- and raises the single
run's first failure (stage, chunk, cause, message), with repeated ids and label
failures straddling the rank boundaries.  The G shards run one after another on
this device through the same fold and wire format the torchrun path uses
(``run_shards_local``)."""

from __future__ import annotations

import pytest

import featurebox_oracle as O
from conftest import corpus, golden_run
from test_gpu_edge import PLACEMENT, _chain, _config, _set_ids, _set_labels, _views, _write_views

pytestmark = pytest.mark.gpu

OPS = [{"name": "c", "inputs": ["query"], "outputs": ["c"], "body": {"fn": "hash:3"}}]


def _cfg(dag, d, batch_size=512):
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.workloads import workload_config
    return config_from_dict(workload_config(dag, batch_size=batch_size), d)


@pytest.mark.parametrize("dag", ["default", "sign_heavy", "lookup_heavy"])
@pytest.mark.parametrize("world", [1, 2, 3, 7])
def test_sharded_run_matches_goldens(dag, world, goldens):
    from paper_2210_07768_b200.sharded import run_shards_local
    _, d = corpus(20000, 2000, 7)
    rep = run_shards_local(_cfg(dag, d), world, slice_rows=4096)
    g = golden_run(goldens, 20000, 7, dag)
    assert f"0x{rep.digest:016x}" == g["digest"]
    assert (rep.instances, rep.signs, rep.batches) == (g["instances"], g["signs"], g["batches"])
    assert (rep.rows_dropped, rep.rows_filtered) == (g["rows_dropped"], g["rows_filtered"])


def _oracle_err(raw, drv, prof, bas, tmp):
    tables, sizes = O.load_tables(raw.get("tables", {}), tmp)
    try:
        O.run_pipelined(raw, {"ev": drv, "pr": prof}, bas, tables, sizes)
    except O.OracleError as e:
        return e
    return None


def _sharded(raw, tmp, world, slice_rows):
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.sharded import run_shards_local
    try:
        return run_shards_local(config_from_dict(raw, tmp), world, slice_rows=slice_rows), None
    except Exception as e:  # noqa: BLE001
        return None, e


BOUNDARY = {  # rank boundary of world 2 / bs 100: row 1000 (rows that reach the merge)
    "dup_across_boundary": _set_ids([(1003, 998)]),
    "dup_of_id_zero": lambda d, p, b: _zero_ids(d, p, b, (4, 1502)),
    "range_then_null_one_batch": _chain(_set_labels([998], 7), _set_labels([1006], None)),
    "null_then_range": _chain(_set_labels([1006], 7), _set_labels([998], None)),
    "range_only_near_boundary": _set_labels([999], 2),
}


def _zero_ids(drv, prof, bas, rows):
    from paper_2210_07768_b200.columns import ColumnImage, Kind
    ids = drv.columns["instance_id"].to_pylist()
    for r in rows:
        ids[r] = 0
    drv.columns["instance_id"] = ColumnImage.from_values(Kind.INT64, ids)
    return drv, prof, bas


@pytest.mark.parametrize("case", sorted(PLACEMENT) + sorted(BOUNDARY))
@pytest.mark.parametrize("world,batch_size", [(2, 100), (3, 512), (4, 64), (5, 100)])
def test_sharded_failure_is_the_single_runs(case, world, batch_size, tmp_path):
    mut = PLACEMENT.get(case) or BOUNDARY[case]
    drv, prof, bas = mut(*_views(2000, 5))
    _write_views(tmp_path, drv, prof, bas)
    raw = _config(batch_size, OPS, {"c": 3}, filt="age != -12345")
    ref_err = _oracle_err(raw, drv, prof, bas, tmp_path)
    _, got_err = _sharded(raw, tmp_path, world, 2 * batch_size)
    assert ref_err is not None, "the mutation does not fail the reference"
    assert got_err is not None, "the sharded run did not fail"
    assert (got_err.stage, got_err.batch_index) == (ref_err.stage, ref_err.chunk)
    assert type(got_err.__cause__).__name__ == type(ref_err.cause).__name__
    assert str(got_err.__cause__) == str(ref_err.cause)


@pytest.mark.parametrize("case", ["range_then_null_one_batch", "dup_of_id_zero"])
@pytest.mark.parametrize("batch_size", [100, 512, 1500])
def test_single_run_failure_cause(case, batch_size, tmp_path):
    """The single-GPU run: a null label wins over an earlier non-0/1 label of
    the same batch (also from the merged order of batch_size > 1024), and a
    repeated id 0 is reported as 0 -- same cause and message as the reference."""
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.engine import run_pipelined
    drv, prof, bas = BOUNDARY[case](*_views(2000, 5))
    _write_views(tmp_path, drv, prof, bas)
    raw = _config(batch_size, OPS, {"c": 3}, filt="age != -12345")
    ref_err = _oracle_err(raw, drv, prof, bas, tmp_path)
    with pytest.raises(Exception) as ei:
        run_pipelined(config_from_dict(raw, tmp_path))
    got = ei.value
    assert (got.stage, got.batch_index) == (ref_err.stage, ref_err.chunk)
    assert type(got.__cause__).__name__ == type(ref_err.cause).__name__
    assert str(got.__cause__) == str(ref_err.cause)


@pytest.mark.parametrize("rows,world", [(600, 4), (1, 3), (0, 2), (1024, 2)])
def test_sharded_more_ranks_than_chunks(rows, world, tmp_path):
    """Ranks left without chunks contribute nothing; the result is the single run's."""
    drv, prof, bas = _views(max(rows, 1), 3)
    if rows == 0:
        drv = drv.slice(0, 0)
    _write_views(tmp_path, drv, prof, bas)
    raw = _config(512, OPS, {"c": 3}, filt="age != -12345")
    tables, sizes = O.load_tables({}, tmp_path)
    try:
        ref = O.run_pipelined(raw, {"ev": drv, "pr": prof}, bas, tables, sizes)
    except O.OracleError as e:
        _, got_err = _sharded(raw, tmp_path, world, 512)
        assert got_err is not None and got_err.stage == e.stage
        return
    got, got_err = _sharded(raw, tmp_path, world, 512)
    assert got_err is None, got_err  # one chunk: the whole log on every rank
    assert (got.digest, got.instances, got.signs) == (ref.digest, ref.instances, ref.signs)


# ---- run_sharded itself: two processes on this device, gloo for the exchange ----

def _rank_main(rank, world, port, d, raw, q, backend="gloo"):
    import os
    import sys
    from pathlib import Path
    sys.path[:0] = [str(Path(__file__).parent), str(Path(__file__).parent.parent / "oracle")]
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.sharded import run_sharded
    try:
        rep = run_sharded(config_from_dict(raw, Path(d)), slice_rows=1024)
        q.put((rank, ("ok", rep.digest, rep.instances, rep.signs, rep.batches)))
    except Exception as e:  # noqa: BLE001
        q.put((rank, ("err", e.stage, e.batch_index, type(e.__cause__).__name__,
                      str(e.__cause__))))
    finally:
        dist.destroy_process_group()


def _spawn(world, d, raw, backend="gloo"):
    import multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_rank_main, args=(r, world, port, str(d), raw, q, backend))
          for r in range(world)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    return got


def test_run_sharded_two_processes_matches_goldens(goldens):
    from paper_2210_07768_b200.workloads import workload_config
    _, d = corpus(20000, 2000, 7)
    got = _spawn(2, d, workload_config("sign_heavy"))
    g = golden_run(goldens, 20000, 7, "sign_heavy")
    for r in (0, 1):
        assert got[r][0] == "ok", got[r]
        assert f"0x{got[r][1]:016x}" == g["digest"]
        assert got[r][2:] == (g["instances"], g["signs"], g["batches"])


@pytest.mark.parametrize("case", ["dup_across_boundary", "range_then_null_one_batch"])
def test_run_sharded_two_processes_fail_alike(case, tmp_path):
    drv, prof, bas = BOUNDARY[case](*_views(2000, 5))
    _write_views(tmp_path, drv, prof, bas)
    raw = _config(100, OPS, {"c": 3}, filt="age != -12345")
    ref_err = _oracle_err(raw, drv, prof, bas, tmp_path)
    got = _spawn(2, tmp_path, raw)
    want = ("err", ref_err.stage, ref_err.chunk, type(ref_err.cause).__name__, str(ref_err.cause))
    assert got[0] == got[1] == want


def test_run_sharded_nccl_one_rank(goldens):
    """The NCCL exchange path (device tensors) with the one GPU of this box."""
    from paper_2210_07768_b200.workloads import workload_config
    _, d = corpus(20000, 2000, 7)
    got = _spawn(1, d, workload_config("lookup_heavy"), backend="nccl")
    g = golden_run(goldens, 20000, 7, "lookup_heavy")
    assert got[0][0] == "ok", got[0]
    assert f"0x{got[0][1]:016x}" == g["digest"]
    assert got[0][2:] == (g["instances"], g["signs"], g["batches"])


@pytest.mark.parametrize("pool,lpg,batch_size", [(128, 256, 512), (1024, 7, 64), (4096, 256, 512),
                                                 (3200, 7, 64)])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_pool_bytes(pool, lpg, batch_size, world, tmp_path):
    """The reference arena's PoolExhausted (requested, remaining) at the single
    run's (chunk, layer, node) when the failing chunk sits on any rank."""
    from test_gpu_edge import POOL_FEATS, POOL_OPS
    drv, prof, bas = _views(2000, 9)
    _write_views(tmp_path, drv, prof, bas)
    raw = _config(batch_size, POOL_OPS, POOL_FEATS, filt="age != -12345")
    raw["device"] = {"budget_bytes": 65536, "pool_bytes": pool, "lanes_per_group": lpg}
    tables, sizes = O.load_tables({}, tmp_path)
    try:
        ref, ref_err = O.run_pipelined(raw, {"ev": drv, "pr": prof}, bas, tables, sizes), None
    except O.OracleError as e:
        ref, ref_err = None, e
    got, got_err = _sharded(raw, tmp_path, world, 2 * batch_size)
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
