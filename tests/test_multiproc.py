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
