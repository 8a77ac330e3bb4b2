"""CPU: the record-sharded run's fold (sharded.combine_outcomes + exchange) places
the run's first failure where the reference's single pass over the whole log
raises it (pipeline.py:1040-1090: per chunk the row-level failures, then the
merge's check_unique_ids, then the _Emitter flushes; the final flush last).

A log is modelled row by row (id, label, whether the row survives to the merge,
whether it fails its extract); each rank's ShardOutcome is computed from its
own rows only -- what its engine reports -- and the fold must give the single
pass's (stage, chunk, cause).  The exchange runs over gloo with world size 2."""

from __future__ import annotations

import os
import random

import pytest

from paper_2210_07768_b200 import codegen, placement
from paper_2210_07768_b200.distributed import shard_rows
from paper_2210_07768_b200.sharded import NONE, ShardOutcome, combine_outcomes

ROW_ERR = codegen.ERR["value"]


def _log(seed):
    rng = random.Random(seed)
    n = rng.randrange(0, 400)
    bs = rng.choice([1, 3, 7, 16, 50, 64, 100])
    pool = rng.randrange(max(2, n // 3), 4 * n + 8)
    rows = []
    for _ in range(n):
        r = rng.random()
        label = None if r < 0.004 else (rng.choice([2, 7, -1]) if r < 0.008 else rng.randrange(2))
        rows.append({"id": rng.randrange(pool) - pool // 2, "label": label,
                     "alive": rng.random() < 0.9, "err": rng.random() < 0.0015})
    return rows, bs


def single_pass(rows, bs):
    """The reference's one pass: (stage, chunk, kind, detail) of its failure, or None."""
    seen, buf = set(), []
    for c in range(0, -(-len(rows) // bs)):
        chunk = rows[c * bs:(c + 1) * bs]
        if any(r["err"] for r in chunk):
            return ("extract", c, "value", None)
        alive = [r for r in chunk if r["alive"]]
        for r in alive:
            if r["id"] in seen:
                return ("merge", c, "dup_id", r["id"])
            seen.add(r["id"])
        buf += alive
        while len(buf) >= bs:
            batch, buf = buf[:bs], buf[bs:]
            f = _batch_failure(batch)
            if f:
                return ("merge", c) + f
    f = _batch_failure(buf) if buf else None
    return ("emit", None) + f if f else None


def _batch_failure(batch):
    if any(r["label"] is None for r in batch):
        return ("null_label", None)
    for r in batch:
        if r["label"] not in (0, 1):
            return ("label_range", r["label"])
    return None


def shard_outcome(rows, bs, lo, hi, lower_ids=None):
    """What a rank's engine reports for rows [lo, hi): its own first row-level
    failure, first in-range repeat, first row whose id a lower rank holds, first
    null / non-0/1 label by range-local emission position, per-chunk counts."""
    err = NONE
    for i in range(lo, hi):
        if rows[i]["err"]:
            err = placement.key_of(i // bs, "extract", ROW_ERR)
            break
    seen, dup_row, dup_id, cross_row, cross_id = set(), NONE, 0, NONE, 0
    null_pos = range_pos = NONE
    range_label, pos, ends = 0, 0, []
    for i in range(lo, hi):
        r = rows[i]
        if r["alive"]:
            if r["id"] in seen and dup_row == NONE:
                dup_row, dup_id = i, r["id"]
            if lower_ids is not None and r["id"] in lower_ids and cross_row == NONE:
                cross_row, cross_id = i, r["id"]
            seen.add(r["id"])
            if r["label"] is None and null_pos == NONE:
                null_pos = pos
            if r["label"] is not None and r["label"] not in (0, 1) and range_pos == NONE:
                range_pos, range_label = pos, r["label"]
            pos += 1
        if (i + 1) % bs == 0 or i + 1 == hi:
            ends.append(pos)
    return ShardOutcome(lo, hi, pos, 0, 0, 0, 0, pos, err, 0, dup_row, dup_id, cross_row,
                        cross_id, null_pos, range_pos, range_label, NONE, 1, 0, tuple(ends))


def _ids(rows, lo, hi):
    return {r["id"] for r in rows[lo:hi] if r["alive"]}


def _decode(key, detail):
    stage = {v: k for k, v in codegen.STAGE.items()}[(key >> 28) & 0xF]
    kind = {v: k for k, v in codegen.ERR.items()}[key & 0xFF]
    chunk = None if stage == "emit" else key >> 32
    det = detail if kind in ("dup_id", "label_range") else None
    return stage, chunk, kind, det


def _fold(rows, bs, world):
    outs, lower = [], set()
    n = len(rows)
    for r in range(world):
        lo, hi = shard_rows(n, bs, r, world)
        o = shard_outcome(rows, bs, lo, hi, lower if r else None)
        width = max(-(-(b - a) // bs) for a, b in (shard_rows(n, bs, q, world)
                                                    for q in range(world)))
        outs.append(ShardOutcome.from_vector(o.to_vector(width)))
        lower |= _ids(rows, lo, hi)
    return combine_outcomes(outs, bs)


@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
def test_fold_places_the_single_pass_failure(world):
    hits = 0
    for seed in range(400):
        rows, bs = _log(seed)
        want = single_pass(rows, bs)
        comb = _fold(rows, bs, world)
        got = None if comb.key == NONE else _decode(comb.key, comb.detail)
        assert got == want, (seed, world, bs, got, want)
        hits += want is not None
        assert comb.instances == sum(r["alive"] for r in rows) or want is not None
    assert hits > 50  # the corpus exercises the failures


def test_null_beats_an_earlier_range_label_across_ranks():
    """A batch straddling two ranks: rank 0 holds a non-0/1 label early in it,
    rank 1 a null later in it -- the batch fails with the null (emit_minibatch
    before MiniBatch.validate), at the chunk whose merge completes the batch."""
    bs = 10
    rows = [{"id": i, "label": 0, "alive": True, "err": False} for i in range(40)]
    for i in (3, 5, 7, 12, 14, 16):  # rank 0's last chunk ends early in instances
        rows[i]["alive"] = False
    rows[18]["label"] = 9        # rank 0 (rows 0-19), batch 1
    rows[21]["label"] = None     # rank 1 (rows 20-39), still batch 1
    want = single_pass(rows, bs)
    assert want[2] == "null_label"
    comb = _fold(rows, bs, 2)
    assert _decode(comb.key, comb.detail) == want


def test_cross_rank_repeat_is_found_at_its_row():
    bs = 8
    rows = [{"id": i, "label": 1, "alive": True, "err": False} for i in range(64)]
    rows[50]["id"] = 2   # repeats row 2 (rank 0) on rank 3 of 4
    rows[60]["id"] = 55  # an in-range repeat, later
    want = single_pass(rows, bs)
    assert want == ("merge", 6, "dup_id", 2)
    comb = _fold(rows, bs, 4)
    assert _decode(comb.key, comb.detail) == want


def test_wire_format_round_trip():
    o = ShardOutcome(512, 1024, 7, 99, (1 << 64) - 5, 1, 2, 7, NONE, 0, NONE, 0, 700, -3,
                     NONE, 4, -9, NONE, 3, 12345, (3, 7))
    v = o.to_vector(5)
    assert len(v) == ShardOutcome.HEAD + 1 + 5
    assert ShardOutcome.from_vector(v) == o


# ---- the exchange over gloo, world size 2 ------------------------------------

class _FakeShard:
    """A rank's side of the exchange without a device: ids and outcome from
    the row model (the engine computes the same on the GPU)."""

    def __init__(self, rows, bs, rank, world):
        import torch
        self.rows, self.bs = rows, bs
        self.n_total = len(rows)
        self.lo, self.hi = shard_rows(self.n_total, bs, rank, world)
        ids = sorted(_ids(rows, self.lo, self.hi))
        self.ids = torch.tensor(ids or [0], dtype=torch.int64)
        self.n_ids = len(ids)
        self.device = torch.device("cpu")
        self.lower = None

    def seen_before(self, prior):
        self.lower = set(int(x) for x in prior.tolist())

    def outcome(self):
        return shard_outcome(self.rows, self.bs, self.lo, self.hi, self.lower)


def _gloo_worker(rank, world, port, seeds, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2210_07768_b200.sharded import exchange
    try:
        res = []
        for seed in seeds:
            rows, bs = _log(seed)
            comb = combine_outcomes(exchange(_FakeShard(rows, bs, rank, world), bs), bs)
            got = None if comb.key == NONE else _decode(comb.key, comb.detail)
            res.append((seed, got, single_pass(rows, bs), comb.instances))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_exchange_over_gloo_world2():
    import multiprocessing as mp
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    seeds = list(range(60))
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, seeds, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    assert got[0] == got[1]  # every rank folds to the same result
    for seed, g, want, _ in got[0]:
        assert g == want, (seed, g, want)
