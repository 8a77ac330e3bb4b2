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

Two ways to split a workload (``bench.py`` uses both):

* one log cut into contiguous chunk ranges (``shard_rows``): the ranks' CSRs
  concatenate to the single-GPU emission order.  ``sharded.run_sharded`` runs it
  with the single run's result AND failures: the instance-id uniqueness check
  (pipeline.py:1071-1072) across ranks and the mini-batch boundaries are
  exchanged after the shards finish (sharded.py);
* independent logs (SURVEY.md §8 d: C5's 1M-record shards, each its own
  reference pipeline with ids restarting at 0): shard k goes to rank k mod G
  (``assign_shards``), every shard is checked against the reference's digest
  of that shard, and the run digest is the XOR of the shard digests.
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


def assign_shards(n_shards: int, seed0: int, rank: int, world: int) -> list[int]:
    """Seeds of the independent shards rank owns: shard k -> rank k mod world."""
    if not 0 <= rank < world:
        raise ValueError("rank outside world")
    return [seed0 + k for k in range(n_shards) if k % world == rank]


def weak_seeds(seed: int, rank: int) -> list[int]:
    """Weak scaling: every rank extracts its own log, seed + rank."""
    return [seed + rank]


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


def gather_parity(checked: int, n_shards: int, golden_xor: int, run_digest: int,
                  group=None, device=None) -> dict:
    """All-gather of the per-rank parity tallies (shards checked against the
    reference, shards owned, XOR of the reference digests of the checked
    shards) -> one summary; raises when every shard was checked but the run
    digest differs from the reference XOR."""
    import torch
    import torch.distributed as dist
    gx = golden_xor & MASK64
    t = torch.tensor([checked, n_shards, gx & ((1 << 63) - 1), gx >> 63], dtype=torch.int64,
                     device=device)
    if dist.is_available() and dist.is_initialized():
        parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
        dist.all_gather(parts, t, group=group)
    else:
        parts = [t]
    n_checked = sum(int(p[0]) for p in parts)
    n_all = sum(int(p[1]) for p in parts)
    x = 0
    for p in parts:
        x ^= int(p[2]) | (int(p[3]) << 63)
    if n_checked == n_all and n_all and x != run_digest & MASK64:
        raise RuntimeError(f"run digest 0x{run_digest & MASK64:016x} != XOR of the reference "
                           f"shard digests 0x{x:016x}")
    return {"shards_checked": f"{n_checked}/{n_all} shard digests = reference",
            "reference_xor": f"0x{x:016x}" if n_checked == n_all else None,
            "checked": n_checked, "shards": n_all}
