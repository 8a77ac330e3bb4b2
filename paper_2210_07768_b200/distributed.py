"""Record-sharded multi-GPU execution (SURVEY.md §8 e).

Every operator is row-local, so the 8-GPU box runs one record shard per GPU
with no per-record communication.  Each rank owns a contiguous range of driver
chunks (chunk boundaries are the reference's read boundaries, pipeline.py:994),
so the concatenation of the ranks' CSRs in rank order is the single-GPU
emission order.  The only collective is one all-gather of the per-shard
counters ``[records, instances, signs, digest, malformed, filtered]`` after the
shard finishes; each rank turns it into its global CSR base offsets (an
exclusive scan over ranks) and the run digest (XOR -- NCCL has no XOR
reduction, so it is folded after the gather).
"""

from __future__ import annotations

from dataclasses import dataclass

FIELDS = ("records", "instances", "signs", "digest", "malformed", "filtered")
MASK64 = (1 << 64) - 1


def shard_rows(n_rows: int, batch_size: int, rank: int, world: int) -> tuple[int, int]:
    """Rank's row range: contiguous whole chunks, balanced to +-1 chunk."""
    if not 0 <= rank < world:
        raise ValueError("rank outside world")
    chunks = (n_rows + batch_size - 1) // batch_size
    per, extra = divmod(chunks, world)
    c0 = rank * per + min(rank, extra)
    c1 = c0 + per + (1 if rank < extra else 0)
    return min(c0 * batch_size, n_rows), min(c1 * batch_size, n_rows)


@dataclass
class ShardResult:
    records: int
    instances: int
    signs: int
    digest: int
    malformed: int = 0
    filtered: int = 0

    def to_list(self) -> list[int]:
        d = self.digest & MASK64
        return [self.records, self.instances, self.signs,
                d - (1 << 64) if d >> 63 else d, self.malformed, self.filtered]

    @classmethod
    def from_list(cls, v) -> "ShardResult":
        v = [int(x) for x in v]
        return cls(v[0], v[1], v[2], v[3] & MASK64, v[4], v[5])


@dataclass
class RunTotals:
    records: int
    instances: int
    signs: int
    digest: int
    malformed: int
    filtered: int
    inst_base: list[int]   # per-rank exclusive prefix of instances
    sign_base: list[int]   # per-rank exclusive prefix of signs


def combine(shards: list[ShardResult]) -> RunTotals:
    """Fold gathered shard results (rank order) into run totals."""
    ib, sb, i, s, dig = [], [], 0, 0, 0
    for r in shards:
        ib.append(i)
        sb.append(s)
        i += r.instances
        s += r.signs
        dig ^= r.digest
    return RunTotals(sum(r.records for r in shards), i, s, dig,
                     sum(r.malformed for r in shards), sum(r.filtered for r in shards), ib, sb)


def all_gather_results(local: ShardResult, group=None, device=None) -> RunTotals:
    """The one collective: all-gather 6 int64 per rank (NCCL or gloo)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(local.to_list(), dtype=torch.int64, device=device)
    world = dist.get_world_size(group)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    return combine([ShardResult.from_list(p.cpu().tolist()) for p in parts])
