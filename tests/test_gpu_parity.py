"""GPU parity: the fused CUDA path against the reference's golden outputs and
the CPU oracle.  Bit-exact for ids, labels, offsets, slots and signs."""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN, corpus, golden_run

pytestmark = pytest.mark.gpu

DAGS = ("default", "fig4", "sign_heavy", "cross_heavy", "lookup_heavy")


def _run(rows, users, seed, dag, ops_only=False, batch_size=512, views=2, collect=True,
         max_rows_per_launch=1 << 22, raw=None):
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.engine import run_views
    from paper_2210_07768_b200.workloads import workload_config
    c, d = corpus(rows, users, seed, views)
    if raw is None:
        if views == 2:
            raw = workload_config(dag, batch_size=batch_size, ops_only=ops_only)
        else:
            raw = json.loads((d / "pipeline.json").read_text())
            raw["batch_size"] = batch_size
    cfg = config_from_dict(raw, d)
    vs = {"user_events": c.driver}
    if c.profile is not None:
        vs["user_profile"] = c.profile
    return run_views(cfg, vs, c.basic, collect=collect,
                     max_rows_per_launch=max_rows_per_launch)


@pytest.mark.parametrize("dag", DAGS)
def test_csr_matches_reference_minibatches(dag, goldens):
    res = _run(2000, 300, 7, dag)
    g = golden_run(goldens, 2000, 7, dag)
    rep = res.report
    assert f"0x{rep.digest:016x}" == g["digest"]
    assert (rep.instances, rep.signs, rep.batches) == (g["instances"], g["signs"], g["batches"])
    assert (rep.rows_dropped, rep.rows_filtered) == (g["rows_dropped"], g["rows_filtered"])
    ref = np.load(GOLDEN / f"csr_{dag}.npz")
    for k in ("ids", "labels", "offsets", "slots", "signs"):
        np.testing.assert_array_equal(res.csr[k], ref[k], err_msg=k)


@pytest.mark.parametrize("dag", DAGS)
@pytest.mark.parametrize("ops_only", [False, True])
def test_digest_20k(dag, ops_only, goldens):
    rep = _run(20000, 2000, 7, dag, ops_only=ops_only, collect=False).report
    g = golden_run(goldens, 20000, 7, dag, ops_only)
    assert f"0x{rep.digest:016x}" == g["digest"]
    assert (rep.instances, rep.signs, rep.batches) == (g["instances"], g["signs"], g["batches"])
    assert (rep.rows_dropped, rep.rows_filtered) == (g["rows_dropped"], g["rows_filtered"])


def test_single_view_corpus(goldens):
    rep = _run(1200, 200, 11, "default", views=1, collect=False).report
    g = golden_run(goldens, 1200, 11, "default", views=1)
    assert f"0x{rep.digest:016x}" == g["digest"]
    assert (rep.instances, rep.signs) == (g["instances"], g["signs"])


def test_multi_launch_equals_single_launch():
    a = _run(20000, 2000, 7, "sign_heavy")
    b = _run(20000, 2000, 7, "sign_heavy", max_rows_per_launch=4096)
    assert a.report.digest == b.report.digest
    for k in ("ids", "labels", "offsets", "slots", "signs"):
        np.testing.assert_array_equal(a.csr[k], b.csr[k], err_msg=k)


@pytest.mark.parametrize("dag,zero_copy", [("sign_heavy", True), ("cross_heavy", False),
                                           ("default", True)])
def test_streamed_e2e_equals_device_resident(dag, zero_copy, goldens):
    """Host buffers -> overlapped H2D / fused kernels / D2H with the look-back
    continuing across launches == the single device-resident launch."""
    from paper_2210_07768_b200 import engine as E
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.workloads import workload_config
    c, d = corpus(20000, 2000, 7)
    views = {"user_events": c.driver, "user_profile": c.profile}
    prep = E.prepare(config_from_dict(workload_config(dag), d), views, c.basic)
    eng = E.Engine(prep, views, c.basic)
    eng.begin_run(c.driver.row_count)
    sr = E.StreamedRun(eng, c.driver, slice_rows=3000, zero_copy=zero_copy)
    tot = sr.run()
    g = golden_run(goldens, 20000, 7, dag)
    assert f"0x{tot.digest:016x}" == g["digest"]
    assert (tot.instances, tot.signs) == (g["instances"], g["signs"])
    got = sr.csr(tot)
    ref = _run(20000, 2000, 7, dag).csr
    for k in ("ids", "labels", "offsets", "slots", "signs"):
        np.testing.assert_array_equal(got[k], ref[k], err_msg=k)


def test_streamed_runs_back_to_back_two_engines(goldens):
    """start()/finish() pipelining: run k+1's H2D and kernels are enqueued before
    run k drains; every run's CSR still equals the device-resident result."""
    from paper_2210_07768_b200 import engine as E
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.workloads import workload_config
    c, d = corpus(20000, 2000, 7)
    views = {"user_events": c.driver, "user_profile": c.profile}
    cfg = config_from_dict(workload_config("sign_heavy"), d)
    engs = [E.Engine(E.prepare(cfg, views, c.basic), views, c.basic) for _ in range(2)]
    for taper in (False, True):
        srs = [E.StreamedRun(e, c.driver, slice_rows=4096, taper=taper) for e in engs]
        ref = _run(20000, 2000, 7, "sign_heavy").csr
        g = golden_run(goldens, 20000, 7, "sign_heavy")
        srs[0].start()
        for k in range(5):
            if k + 1 < 5:
                srs[(k + 1) % 2].start()
            tot = srs[k % 2].finish()
            srs[k % 2].wait()
            assert f"0x{tot.digest:016x}" == g["digest"]
            got = srs[k % 2].csr(tot)
            for key in ("ids", "labels", "offsets", "slots", "signs"):
                np.testing.assert_array_equal(got[key], ref[key], err_msg=f"{key} run {k}")
        for r in srs:
            r.wait()


def test_streamed_slice_plan_covers_rows():
    """Tapered slices: chunk-aligned cuts covering every row exactly once."""
    from paper_2210_07768_b200 import engine as E
    c, d = corpus(20000, 2000, 7)
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.workloads import workload_config
    views = {"user_events": c.driver, "user_profile": c.profile}
    eng = E.Engine(E.prepare(config_from_dict(workload_config("default"), d), views, c.basic),
                   views, c.basic)
    for rows, taper in ((1000, True), (4096, True), (4096, False), (1 << 20, True)):
        sr = E.StreamedRun(eng, c.driver, slice_rows=rows, taper=taper)
        cuts = [a for a, _ in sr.bounds] + [sr.bounds[-1][1]]
        assert cuts[0] == 0 and cuts[-1] == 20000
        assert all(a < b for a, b in sr.bounds)
        assert all(x % eng.ir.chunk == 0 for x in cuts[:-1])


@pytest.mark.parametrize("knob", ["FBX_NVRTC_OPTS=-DFBX_POOL_WARP", "FBX_STAGE=0",
                                  "FBX_SORT_ROWS=0", "FBX_POOL_WARP_GRANTS=0"])
@pytest.mark.parametrize("dag", ["sign_heavy", "cross_heavy"])
def test_codegen_knobs_keep_parity(knob, dag, goldens, monkeypatch):
    """The remaining generator switches (fallback paths the kernel takes for other
    shapes: HBM-resident spans, unsorted rows, CTA-scan pool grants) stay bit-exact."""
    for kv in knob.split():
        k, v = kv.split("=", 1)
        monkeypatch.setenv(k, v)
    res = _run(20000, 2000, 7, dag, max_rows_per_launch=8192)
    g = golden_run(goldens, 20000, 7, dag)
    assert f"0x{res.report.digest:016x}" == g["digest"]
    assert (res.report.instances, res.report.signs) == (g["instances"], g["signs"])
    ref = _run(20000, 2000, 7, dag).csr
    for k in ("ids", "labels", "offsets", "slots", "signs"):
        np.testing.assert_array_equal(res.csr[k], ref[k], err_msg=k)


@pytest.mark.parametrize("n", [0, 1, 7, 255, 256, 257, 65535, 65536, 65537, 1_000_003,
                               1024 * 65536 + 4097, 3 * 1024 * 65536 + 5])
def test_crc32_device_matches_zlib(n):
    import zlib
    import torch
    from paper_2210_07768_b200.engine import crc32_device
    rng = np.random.default_rng(n)
    host = rng.integers(0, 256, size=n + 11, dtype=np.uint8)
    dev = torch.from_numpy(host).cuda()
    for off in (0, 3) if n else (0,):  # aligned and unaligned starts
        got = crc32_device(dev[off:off + n])
        assert got == zlib.crc32(host[off:off + n].tobytes()) & 0xFFFFFFFF, (n, off)


def test_fbxc_ingest_device_view_and_crc(tmp_path):
    """DeviceView.from_fbxc: one body copy, column views, device CRC (and the
    engine runs on it bit-exactly)."""
    from paper_2210_07768_b200 import engine as E
    from paper_2210_07768_b200.columns import ChecksumError, read_view
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.workloads import workload_config
    c, d = corpus(20000, 2000, 7)
    path = d / "user_events.fbxc"
    dv = E.DeviceView.from_fbxc(path)
    ref = E.DeviceView(read_view(path))
    for name, parts in ref.tensors.items():
        for part, t in parts.items():
            got = dv.tensors[name][part]
            assert torch_equal_prefix(got, t), (name, part)
    views = {"user_events": c.driver, "user_profile": c.profile}
    eng = E.Engine(E.prepare(config_from_dict(workload_config("sign_heavy"), d), views, c.basic),
                   views, c.basic)
    eng.bind_driver(dv)
    eng.reserve(c.driver.row_count)
    eng.begin_run(c.driver.row_count)
    eng.launch(0, c.driver.row_count, tile_base=0)
    res = eng.finish()
    want = _run(20000, 2000, 7, "sign_heavy").report.digest
    assert res.counters.digest == want
    raw = bytearray(path.read_bytes())
    raw[len(raw) // 2] ^= 0x40
    bad = tmp_path / "bad.fbxc"
    bad.write_bytes(bytes(raw))
    with pytest.raises(ChecksumError):
        E.DeviceView.from_fbxc(bad)


def torch_equal_prefix(a, b):
    n = min(a.numel(), b.numel())
    la = a.numel() if a.numel() < b.numel() else n
    return bool((a[:la] == b[:la]).all())


def test_device_minibatches_match_reference_batches(goldens):
    """CsrBatch.minibatches: the _Emitter's cut (every batch_size instances across
    chunks), as device views; concatenated they are the run's CSR."""
    from paper_2210_07768_b200 import engine as E
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.workloads import workload_config
    c, d = corpus(20000, 2000, 7)
    views = {"user_events": c.driver, "user_profile": c.profile}
    cfg = config_from_dict(workload_config("default"), d)
    eng = E.Engine(E.prepare(cfg, views, c.basic), views, c.basic)
    eng.bind_driver(E.DeviceView(c.driver))
    eng.reserve(c.driver.row_count)
    eng.begin_run(c.driver.row_count)
    eng.launch(0, c.driver.row_count, tile_base=0)
    batch = eng.finish()
    full = batch.to_numpy()
    mbs = list(batch.minibatches(cfg.batch_size))
    n = batch.counters.instances
    assert len(mbs) == -(-n // cfg.batch_size)
    assert sum(int(mb.ids.numel()) for mb in mbs) == n
    signs = np.concatenate([mb.signs.cpu().numpy().view(np.uint64) for mb in mbs])
    np.testing.assert_array_equal(signs, full["signs"])
    for k, mb in enumerate(mbs[:5]):
        o = mb.offsets.cpu().numpy()
        b0 = k * cfg.batch_size
        np.testing.assert_array_equal(o, full["offsets"][b0:b0 + len(o)].astype(np.int64)
                                      - int(full["offsets"][b0]))


def test_captured_run_graph_replays_bit_exact(goldens):
    """Engine.capture_run: reset + launches as one CUDA graph; every replay
    reproduces the reference digest and CSR."""
    from paper_2210_07768_b200 import engine as E
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.workloads import workload_config
    c, d = corpus(20000, 2000, 7)
    views = {"user_events": c.driver, "user_profile": c.profile}
    cfg = config_from_dict(workload_config("sign_heavy"), d)
    eng = E.Engine(E.prepare(cfg, views, c.basic), views, c.basic, max_rows_per_launch=8192)
    eng.bind_driver(E.DeviceView(c.driver))
    g = eng.capture_run(c.driver.row_count)
    gold = golden_run(goldens, 20000, 7, "sign_heavy")
    ref = _run(20000, 2000, 7, "sign_heavy").csr
    for _ in range(3):
        g.replay()
        res = eng.finish()
        assert f"0x{res.counters.digest:016x}" == gold["digest"]
        got = res.to_numpy()
        for k in ("ids", "offsets", "signs"):
            np.testing.assert_array_equal(got[k], ref[k], err_msg=k)


def test_reproduces_the_reference_published_100k_run(tmp_path):
    """The reference's own acceptance run (tests/test_acceptance.py: gen_corpus(rows=100_000,
    users=5_000, seed=11), its default pipeline.json, run_pipelined) published digest
    0xb2bcd7004cff26a0, 90,326 instances, 177 batches, 517,976 signs
    (pkg/test_output.txt:19, 25): reproduced end to end on the device."""
    from paper_2210_07768_b200 import load_config, run_pipelined
    from paper_2210_07768_b200.corpus import gen_corpus
    paths = gen_corpus(tmp_path, rows=100_000, users=5_000, seed=11)
    report = run_pipelined(load_config(paths["config"]))
    assert report.digest == 0xB2BCD7004CFF26A0
    assert report.instances == 90326
    assert report.signs == 517976
    assert report.batches == 177


@pytest.mark.parametrize("batch_size", [20_000, 100_000, 1025, 4096])
def test_batch_size_beyond_a_cta(batch_size):
    """SPEC.md:499 (reference): batch_size >= corpus size -> exactly one batch; and any
    batch_size > 1024 (chunks cut into 512-row sub-tiles, merged by instance id)."""
    import featurebox_oracle as O
    res = _run(20000, 2000, 7, "sign_heavy", batch_size=batch_size, max_rows_per_launch=8192)
    from paper_2210_07768_b200.workloads import workload_config
    c, d = corpus(20000, 2000, 7)
    raw = workload_config("sign_heavy", batch_size=batch_size)
    tables, sizes = O.load_tables(raw.get("tables", {}), d)
    ref = O.run_pipelined(raw, {"user_events": c.driver, "user_profile": c.profile}, c.basic,
                          tables, sizes)
    assert (res.report.digest, res.report.instances, res.report.signs) == \
        (ref.digest, ref.instances, ref.signs)
    assert res.report.batches == -(-ref.instances // batch_size)
    np.testing.assert_array_equal(res.csr["ids"], np.array(ref.ids, np.uint64))
    np.testing.assert_array_equal(res.csr["offsets"], np.array(ref.offsets, np.uint64))
    np.testing.assert_array_equal(res.csr["slots"], np.array(ref.slots, np.uint16))
    np.testing.assert_array_equal(res.csr["signs"], np.array(ref.values, np.uint64))


@pytest.mark.parametrize("batch_size,slice_rows", [(2048, 4096), (3000, 9000)])
def test_streamed_run_big_batches(batch_size, slice_rows):
    """StreamedRun with batch_size > 1024: each slice's chunks are merged on the
    device before their D2H; equals the device-resident run and the oracle digest."""
    from paper_2210_07768_b200 import engine as E
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.workloads import workload_config
    c, d = corpus(20000, 2000, 7)
    views = {"user_events": c.driver, "user_profile": c.profile}
    raw = workload_config("cross_heavy", batch_size=batch_size)
    eng = E.Engine(E.prepare(config_from_dict(raw, d), views, c.basic), views, c.basic)
    sr = E.StreamedRun(eng, c.driver, slice_rows=slice_rows)
    tot = sr.run()
    got = sr.csr(tot)
    ref = _run(20000, 2000, 7, "cross_heavy", batch_size=batch_size).csr
    for k in ("ids", "labels", "offsets", "slots", "signs"):
        np.testing.assert_array_equal(got[k], ref[k], err_msg=k)
