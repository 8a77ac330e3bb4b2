"""One log, record-sharded over G GPUs, with the single run's exact result.

``run_sharded`` is ``run_pipelined`` (pipeline.py:952-1114) over a driver log cut
into G contiguous ranges of whole chunks (``distributed.shard_rows``; chunk
boundaries are the reference's read boundaries, pipeline.py:994).  Rank r
streams its range through its own engine (``stream.FileRun`` with ``rows=``);
every operator is row-local, so the ranks' CSRs concatenate to the single-run
emission order and the counters add up.  Two things in the reference are global
across chunks, and they are what the ranks exchange -- no per-record traffic:

* ``check_unique_ids``' ``seen`` set (pipeline.py:1071-1072, viewpipe.py:562-576):
  each rank finds its first in-range repeat on the device as a single run does
  (``fbx_dup_resolve``); the ranks then all-gather their distinct instance ids
  (``fbx_idset_entries``: 8 B per distinct id) and rank r finds the first of
  its rows whose id a lower rank holds (``fbx_seen_before``: sort + binary
  search on the device);
* the mini-batch boundaries (``_Emitter``, pipeline.py:748-777): the kernel
  keeps each rank's first null and first non-0/1 label by emission position
  (fbx_core.cuh ``raise_emit``); shifted by the instances of the lower ranks
  they are run-global positions, and the per-chunk instance counts of every
  rank place the flush that raises.

Then one all-gather of a small outcome vector per rank (``ShardOutcome``), and
every rank folds the outcomes the same way (``combine_outcomes``): counters
summed, digest XOR, the failure with the smallest error key (placement.py)
raised on every rank -- the StageError the single run raises.  Three
collectives per run (id counts, ids, outcomes), NCCL under torchrun.

``run_shards_local`` runs the G shards one after another on one device and
folds them through the same code: the single-GPU check of the sharded path.
A log that does not stream (one chunk, or batch_size > 1024: the
device-resident run) runs whole on every rank.
"""

from __future__ import annotations

from dataclasses import dataclass, fields

import numpy as np

from . import placement, runtime
from .distributed import shard_rows

NONE = placement.NONE
MASK64 = (1 << 64) - 1


@dataclass
class ShardOutcome:
    """What one rank contributes to the run (``NONE`` = nothing)."""
    row_lo: int
    row_hi: int
    instances: int
    signs: int
    digest: int
    malformed: int
    filtered: int
    joined: int
    error_key: int        # the range's first row-level failure (global chunk keys)
    error_detail: int
    dup_row: int          # first row repeating an id of an earlier row of the range
    dup_id: int
    cross_row: int        # first row whose id a lower rank holds
    cross_id: int
    null_pos: int         # first null label, range-local emission position
    range_pos: int        # first non-0/1 label, range-local emission position
    range_label: int
    read_chunk: int       # the chunk whose read failed
    launches: int
    bytes_h2d: int
    chunk_ends: tuple = ()  # range-local inclusive instance count per chunk

    HEAD = 20

    def to_vector(self, width: int) -> list[int]:
        """int64 words (u64 values two's complement): the head, the number of
        chunk ends, the chunk ends, zeros up to ``width`` ends (the widest rank)."""
        head = [getattr(self, f.name) for f in fields(self)][:self.HEAD]
        ends = [int(e) for e in self.chunk_ends]
        return [_s64(v) for v in head] + [len(ends)] + ends + [0] * (width - len(ends))

    @classmethod
    def from_vector(cls, v) -> "ShardOutcome":
        v = [int(x) for x in v]
        head = [x & MASK64 if f.name not in ("dup_id", "cross_id", "range_label") else x
                for f, x in zip(fields(cls), v[:cls.HEAD])]
        n = v[cls.HEAD]
        return cls(*head, chunk_ends=tuple(v[cls.HEAD + 1:cls.HEAD + 1 + n]))


def _s64(v: int) -> int:
    v &= MASK64
    return v - (1 << 64) if v >> 63 else v


@dataclass
class Combined:
    instances: int
    signs: int
    digest: int
    malformed: int
    filtered: int
    joined: int
    launches: int
    bytes_h2d: int
    key: int       # the run's first failure (placement.NONE: none)
    detail: int
    who: int       # the rank whose failure it is (the read failure's original cause)
    inst_base: list


def combine_outcomes(outs: list[ShardOutcome], batch_size: int) -> Combined:
    """Fold the ranks' outcomes (rank order) into the single run's result and
    first failure: the smallest of every rank's row-level failure, the first
    repeated id over all ranks (in-range and cross-rank repeats, by row), and
    the first label failure at run-global emission positions, placed at the
    merge of the chunk that flushes its batch."""
    inst_base, acc = [], 0
    for o in outs:
        inst_base.append(acc)
        acc += o.instances
    key, detail, who = NONE, 0, -1
    for r, o in enumerate(outs):
        if o.error_key < key:
            key, detail, who = o.error_key, o.error_detail, r
        if o.read_chunk != NONE:
            rk = placement.key_of(o.read_chunk, "read", 0)
            if rk < key:
                key, detail, who = rk, -1, r
    row, ident, drank = NONE, 0, -1
    for r, o in enumerate(outs):
        for rr, ii in ((o.dup_row, o.dup_id), (o.cross_row, o.cross_id)):
            if rr < row:
                row, ident, drank = rr, ii, r
    if row != NONE:
        dk = placement.dup_key(row, batch_size)
        if dk < key:
            key, detail, who = dk, ident, drank
    gnull = grange = NONE
    glabel, lrank = 0, -1
    for r, o in enumerate(outs):
        if gnull == NONE and o.null_pos != NONE:
            gnull = inst_base[r] + o.null_pos
        if grange == NONE and o.range_pos != NONE:
            grange, glabel, lrank = inst_base[r] + o.range_pos, o.range_label, r
    lf = placement.label_failure(gnull, grange, batch_size)
    if lf is not None:
        ends = np.concatenate([np.asarray(o.chunk_ends, dtype=np.int64) + inst_base[r]
                               for r, o in enumerate(outs)] or [np.zeros(0, np.int64)])
        lk = placement.label_key(lf, ends, outs[0].row_lo // batch_size, batch_size)
        if lk < key:
            key, detail, who = lk, glabel if lf[1] else 0, lrank
    dig = 0
    for o in outs:
        dig ^= o.digest
    return Combined(acc, sum(o.signs for o in outs), dig, sum(o.malformed for o in outs),
                    sum(o.filtered for o in outs), sum(o.joined for o in outs),
                    sum(o.launches for o in outs), sum(o.bytes_h2d for o in outs), key, detail,
                    who, inst_base)


class ShardReadError(RuntimeError):
    """Another rank's driver read failed (the original error is raised there)."""


# ---------------------------------------------------------------------------
# device side of one shard
# ---------------------------------------------------------------------------

class _Shard:
    def __init__(self, config, rank: int, world: int, slice_rows: int):
        from .columns import open_view
        from .config import StageError
        from .engine import _stream_pipelined
        try:
            n = open_view(config.view(config.driver).path).row_count
        except Exception as exc:  # noqa: BLE001
            raise StageError("prepare", None, exc) from exc
        self.n_total = n
        self.rows = shard_rows(n, config.batch_size, rank, world)
        self.run = _stream_pipelined(config, slice_rows, self.rows)
        eng = self.run.engine
        self.eng, self.torch, self.device = eng, eng.torch, eng.device
        self.st = self.run.state
        self.n_chunks = -(-(self.rows[1] - self.rows[0]) // config.batch_size)
        # the distinct ids of the range with the first row holding each
        cap = eng._idset_cap
        t = self.torch
        self.ids = t.empty(cap + 1, dtype=t.int64, device=eng.device)
        self.id_rows = t.empty(cap + 1, dtype=t.int64, device=eng.device)
        cnt = t.zeros(1, dtype=t.int64, device=eng.device)
        runtime.call("fbx_idset_entries", eng.idset.data_ptr(), eng.idset_w.data_ptr(),
                     eng.idset_d.data_ptr(), cap, self.ids.data_ptr(),
                     self.id_rows.data_ptr(), cnt.data_ptr(), eng._stream())
        self.n_ids = int(cnt.item())
        self.cross = (NONE, 0)

    def seen_before(self, prior):
        """The first row of the range whose id is in ``prior`` (the lower
        ranks' ids, a device int64 tensor)."""
        eng, t = self.eng, self.torch
        out = t.empty(2, dtype=t.int64, device=eng.device)
        prior = prior.to(eng.device).contiguous()
        runtime.call("fbx_seen_before", self.ids.data_ptr(), self.id_rows.data_ptr(),
                     self.n_ids, prior.data_ptr(), prior.numel(), out.data_ptr(), eng._stream())
        row, ident = (int(x) for x in out.cpu().tolist())
        self.cross = (NONE, 0) if row == -1 else (row, ident)

    def outcome(self) -> ShardOutcome:
        eng, st, c = self.eng, self.st, self.run.counters
        dup_row, dup_id = eng._dup_row() if st["dup_seen"] else (NONE, 0)
        ends = [int(x) for x in eng._global_incl(0, eng._run_tiles)] if eng._run_tiles else []
        # a read failure stops the range early: no instances after it
        ends += [ends[-1] if ends else 0] * (self.n_chunks - len(ends))
        rf = self.run.read_failure
        return ShardOutcome(
            self.rows[0], self.rows[1], c.instances, c.signs, c.digest, c.malformed, c.filtered,
            c.joined, st["error_key"], st["error_detail"], dup_row, dup_id, self.cross[0],
            self.cross[1], st["emit_null_pos"], st["emit_range_pos"], st["emit_range_label"],
            NONE if rf is None else rf.batch_index, self.run.launches, self.run.bytes_h2d,
            tuple(ends))

    def finish(self, outs: list[ShardOutcome], rank: int):
        """Raise the run's first failure on this rank, else its RunReport."""
        from .config import StageError
        from .engine import Counters
        comb = combine_outcomes(outs, self.run.config.batch_size)
        if comb.key != NONE:
            if comb.detail == -1 and (comb.key >> 28) & 0xF == 1:  # a read failure
                if comb.who == rank:
                    raise self.run.read_failure
                chunk = comb.key >> 32
                raise StageError("read", chunk,
                                 ShardReadError(f"rank {comb.who}: driver read failed at chunk "
                                                f"{chunk}"))
            self.eng.raise_key(comb.key, comb.detail, self.st)
        c = Counters(comb.digest, comb.instances, comb.signs, comb.malformed, comb.filtered,
                     comb.joined)
        return self.run.to_report(counters=c, launches=comb.launches, bytes_h2d=comb.bytes_h2d)


# ---------------------------------------------------------------------------
# entry points
# ---------------------------------------------------------------------------

def run_sharded(config, group=None, slice_rows: int = 1 << 19):
    """``run_pipelined`` over this rank's record shard of the driver log
    (torch.distributed initialised: one process per GPU); every rank returns
    the single run's RunReport -- or raises its first failure."""
    import torch.distributed as dist
    from .engine import driver_streams, run_pipelined
    if not driver_streams(config):  # one chunk, or batch_size > 1024: whole on every rank
        return run_pipelined(config, slice_rows=slice_rows)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    sh = _Shard(config, rank, world, slice_rows)
    return sh.finish(exchange(sh, config.batch_size, group), rank)


def exchange(sh, batch_size: int, group=None) -> list[ShardOutcome]:
    """The three collectives of a sharded run: the ranks' distinct-id counts,
    their ids (padded to the largest count; rank r checks its rows against
    the lower ranks' ids), their outcomes.  NCCL moves device tensors; any
    other backend host ones."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = sh.device if dist.get_backend(group) == "nccl" else torch.device("cpu")
    cnt = torch.tensor([sh.n_ids], dtype=torch.int64, device=dev)
    counts = [torch.empty_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(x.item()) for x in counts]
    mine = torch.zeros(max(counts + [1]), dtype=torch.int64, device=dev)
    mine[:sh.n_ids] = sh.ids[:sh.n_ids].to(dev)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    prior = [p[:k] for p, k in zip(parts[:rank], counts[:rank]) if k]
    if prior:
        sh.seen_before(torch.cat(prior))
    del parts, mine
    width = max(-(-(b - a) // batch_size)
                for a, b in (shard_rows(sh.n_total, batch_size, q, world) for q in range(world)))
    vec = torch.tensor(sh.outcome().to_vector(width), dtype=torch.int64, device=dev)
    outs = [torch.empty_like(vec) for _ in range(world)]
    dist.all_gather(outs, vec, group=group)
    return [ShardOutcome.from_vector(o.cpu().tolist()) for o in outs]


def run_shards_local(config, world: int, slice_rows: int = 1 << 19):
    """The G shards of ``run_sharded`` one after another on this device, folded
    through the same exchange and combine (rank 0's view of the run)."""
    import torch
    from .engine import driver_streams, run_pipelined
    if not driver_streams(config):
        return run_pipelined(config, slice_rows=slice_rows)
    shards = [_Shard(config, r, world, slice_rows) for r in range(world)]
    for r in range(1, world):
        prior = [s.ids[:s.n_ids] for s in shards[:r] if s.n_ids]
        if prior:
            shards[r].seen_before(torch.cat(prior))
    outs = [s.outcome() for s in shards]
    n_chunks = max(s.n_chunks for s in shards)
    outs = [ShardOutcome.from_vector(o.to_vector(n_chunks)) for o in outs]  # the wire format
    return shards[0].finish(outs, 0)
