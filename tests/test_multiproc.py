"""CPU, world_size 2 over gloo: the record-sharded run's only collective
(all-gather of per-shard counters) reproduces the single-process run."""

from __future__ import annotations

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_07768_b200.distributed import (ShardResult, all_gather_results, combine,
                                               shard_rows)


def test_shard_rows_partition_whole_chunks():
    for n in (0, 1, 511, 512, 513, 20000, 1_000_000):
        for world in (1, 2, 3, 8):
            spans = [shard_rows(n, 512, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and (a % 512 == 0 or a == n)
            for a, b in spans:
                assert a <= b


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "oracle"), str(root / "tests")]
    import featurebox_oracle as O
    from conftest import corpus
    from paper_2210_07768_b200.workloads import workload_config
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c, d = corpus(2000, 300, 7)
    lo, hi = shard_rows(c.driver.row_count, 512, rank, world)
    cfg = workload_config("default")
    r = O.run_pipelined(cfg, {"user_events": c.driver.slice(lo, hi),
                              "user_profile": c.profile}, c.basic, *O.load_tables(cfg["tables"], d))
    tot = all_gather_results(ShardResult(hi - lo, r.instances, r.signs, r.digest, r.malformed,
                                         r.filtered))
    q.put((rank, tot.digest, tot.instances, tot.signs, tot.records, tot.inst_base))
    dist.destroy_process_group()


def test_gloo_world2_matches_single_process(goldens):
    from conftest import golden_run
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    g = golden_run(goldens, 2000, 7, "default")
    for rank, digest, inst, signs, records, base in out:
        assert f"0x{digest:016x}" == g["digest"]
        assert (inst, signs, records) == (g["instances"], g["signs"], 2000)
        assert base[0] == 0 and len(base) == 2


def test_combine_is_rank_ordered_prefix():
    t = combine([ShardResult(10, 3, 9, 5), ShardResult(10, 4, 8, 6), ShardResult(5, 1, 2, 3)])
    assert t.inst_base == [0, 3, 7] and t.sign_base == [0, 9, 17]
    assert t.digest == 5 ^ 6 ^ 3 and t.records == 25


def test_assign_shards_partition():
    from paper_2210_07768_b200.distributed import assign_shards
    for n in (1, 7, 100):
        for world in (1, 2, 3, 8):
            got = sorted(s for r in range(world) for s in assign_shards(n, 1000, r, world))
            assert got == list(range(1000, 1000 + n))


def _shard(seed):
    import tempfile
    from pathlib import Path
    from paper_2210_07768_b200.corpus import make_corpus, write_corpus
    c = make_corpus(600, 100, seed)
    d = Path(tempfile.mkdtemp(prefix=f"fbxshard{seed}_"))
    write_corpus(c, d)
    return c, d


def _c5_worker(rank, world, port, q, corrupt):
    """bench.py's C5 path on CPU: shard assignment, per-shard results (oracle in
    the engine's seat), the counters all-gather and the parity all-gather."""
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "oracle")]
    import featurebox_oracle as O
    from paper_2210_07768_b200.distributed import (ShardResult, all_gather_results,
                                                   assign_shards, combine, gather_parity)
    from paper_2210_07768_b200.workloads import workload_config
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = workload_config("default")
    mine, gx = [], 0
    for sd in assign_shards(5, 100, rank, world):
        c, d = _shard(sd)
        r = O.run_pipelined(cfg, {"user_events": c.driver, "user_profile": c.profile}, c.basic,
                            *O.load_tables(cfg["tables"], d))
        mine.append(ShardResult(600, r.instances, r.signs, r.digest, r.malformed, r.filtered))
        gx ^= r.digest  # the "golden" of this shard
    loc = combine(mine)
    digest = loc.digest ^ (1 if (corrupt and rank == 1) else 0)
    tot = all_gather_results(ShardResult(loc.records, loc.instances, loc.signs, digest,
                                         loc.malformed, loc.filtered))
    try:
        gp = gather_parity(len(mine), len(mine), gx, tot.digest)
        q.put((rank, tot.digest, tot.records, gp["shards_checked"]))
    except RuntimeError as exc:
        q.put((rank, None, None, str(exc)))
    dist.destroy_process_group()


@pytest.mark.parametrize("corrupt", [False, True])
def test_gloo_world2_c5_shards(corrupt):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root / "oracle")]
    import featurebox_oracle as O
    from paper_2210_07768_b200.workloads import workload_config
    cfg = workload_config("default")
    want = 0
    for sd in range(100, 105):
        c, d = _shard(sd)
        want ^= O.run_pipelined(cfg, {"user_events": c.driver, "user_profile": c.profile},
                                c.basic, *O.load_tables(cfg["tables"], d)).digest
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c5_worker, args=(r, 2, port, q, corrupt)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, digest, records, msg in out:
        if corrupt:
            assert digest is None and "XOR of the reference" in msg
        else:
            assert digest == want and records == 3000 and msg == "5/5 shard digests = reference"
