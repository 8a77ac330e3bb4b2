"""Benchmark: raw log records/s through the fused B200 extraction path.

Workload (BASELINE.json configs[1]): the 1M-record synthetic ads log
(gen_corpus rows=1,000,000 users=5,000 seed=11) through the sign-heavy DAG
 with the reference's full emit (basic merge
included).  A *step* is one pass of the hot path over the whole log: the
per-run side / basic index builds, then clean -> side join -> 18-node DAG ->
uniqueness check + basic merge -> sorted/deduplicated CSR + digests, replayed
as one captured CUDA graph (--no-graph: kernel by kernel).  Every shard's
digest is checked against the unmodified reference's (0xb30824efab77470b for
this log); the L2 is flushed between steps.  `e2e` is the reference-facing
run_pipelined(config) over the log's files, one call per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--dag sign_heavy]
    python bench.py --impl reference ...   # the unmodified reference on the host cores

N > 1 runs under torchrun: one record shard (its own 1M-row log, seed 11 + r)
per GPU, no per-record communication, one NCCL all-gather of the per-shard
{records, instances, signs, digest} at the end (SURVEY.md §8 e).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path


ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

GOLDEN_1M = {  # SURVEY.md Appendix B, 1M / 5000 / seed 11 (reference output, full emit)
    "default": (0xD81834ED0893E11E, 907463, 5203686),
    "fig4": (0xD75A8D50AF79290B, 907463, 4537315),
    "sign_heavy": (0xB30824EFAB77470B, 907463, 11586442),
    "cross_heavy": (0xE504098333D34E53, 907463, 8653476),
    "lookup_heavy": (0x5A153AB37CE08E96, 907463, 9074630),
}


def golden_for(dag: str, seed: int, rows: int, users: int, batch_size: int):
    """(digest, instances, signs) of the UNMODIFIED reference for one shard, or None.
    Seed 11: SURVEY Appendix B; other seeds: tests/golden/shard_goldens.json
    (tests/golden/make_shard_goldens.py, the reference run per shard)."""
    if rows != 1_000_000 or users != 5000 or batch_size != 512:
        return None
    if seed == 11 and dag in GOLDEN_1M:
        return GOLDEN_1M[dag]
    try:
        doc = json.loads((ROOT / "tests" / "golden" / "shard_goldens.json").read_text())
    except (OSError, ValueError):
        return None
    for r in doc.get("shards", []):
        if r["dag"] == dag and r["seed"] == seed:
            return int(r["digest"], 16), r["instances"], r["signs"]
    return None


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--dag", default="sign_heavy")
    ap.add_argument("--batch-size", type=int, default=512,
                    help="driver chunk (the reference's batch_size); the goldens are for 512")
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--users", type=int, default=5000)
    ap.add_argument("--seed", type=int, default=11)
    ap.add_argument("--cpu-sample-rows", type=int, default=24576)
    ap.add_argument("--ref-sample-rows", type=int, default=4096,
                    help="driver rows per host process per step of the reference arm")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--shards", type=int, default=0,
                    help="C5 mode: this many independent 1M-record shards (seeds "
                         "--shard-seed0 + k), split across ranks; 0 = one log per rank")
    ap.add_argument("--shard-seed0", type=int, default=1000)
    ap.add_argument("--shard-streams", type=int, default=3,
                    help="C5: streams the independent shards are spread over")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch each step's kernels one by one instead of replaying each "
                         "shard's step (index rebuild, run reset, fused launches) as one "
                         "captured CUDA graph (measured: the graph is 1.2-1.4 % faster)")
    ap.add_argument("--launch-rows", type=int, default=1 << 24)
    ap.add_argument("--e2e-slice-rows", type=int, default=1 << 18)
    ap.add_argument("--e2e-stream-slice-rows", type=int, default=1 << 20)
    ap.add_argument("--api-slice-rows", type=int, default=1 << 19,
                    help="driver slice of the drop-in run_pipelined file stream")
    ap.add_argument("--lookup-fillers", type=int, default=10_000_000,
                    help="lookup_heavy: never-matching query_dict fillers (SURVEY 8d: >= 1e7 so "
                         "the HBM table exceeds L2)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md): nvidia-smi during the timed region
# ---------------------------------------------------------------------------

class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.out = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.out, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.out.flush()
        rows = []
        for line in Path(self.out.name).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            for n, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        load = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port over a bounded sample on all host cores
# ---------------------------------------------------------------------------

_CPU_CTX = {}


def _cpu_worker(args):
    lo, hi = args
    sys.path.insert(0, str(ROOT / "oracle"))
    import featurebox_oracle as O
    ctx = _CPU_CTX
    drv = ctx["driver"].slice(lo, hi)
    basic = ctx["basic"].slice(lo, hi)  # gen_corpus: basic row i <-> driver row i
    t = time.perf_counter()
    O.run_pipelined(ctx["cfg"], {"user_events": drv, "user_profile": ctx["profile"]},
                    basic, ctx["tables"], ctx["sizes"])
    return hi - lo, time.perf_counter() - t


def cpu_baseline(corpus, raw_cfg, tables_dir, sample_rows, procs=None):
    import multiprocessing as mp
    sys.path.insert(0, str(ROOT / "oracle"))
    import featurebox_oracle as O
    procs = procs or os.cpu_count() or 1
    tables, sizes = O.load_tables(raw_cfg.get("tables", {}), tables_dir)
    _CPU_CTX.update(driver=corpus.driver, profile=corpus.profile, basic=corpus.basic,
                    cfg=raw_cfg, tables=tables, sizes=sizes)
    jobs = [(k * sample_rows, (k + 1) * sample_rows) for k in range(procs)]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    rows = sum(r for r, _ in res)
    slowest = max(t for _, t in res)
    return {"value": rows / slowest, "unit": "records/s", "cores": procs, "kind": "port",
            "sample": f"{procs} processes x {sample_rows} driver rows of the same log "
                      f"(oracle/featurebox_oracle.py, CPython); rate = rows / slowest "
                      f"process ({slowest:.1f}s, wall {wall:.1f}s)"}


# ---------------------------------------------------------------------------

# FNV-1a bytes hashed by the DAG per input record (measured on the
# reference corpus); the instance digests add 9 B per instance + 10 B per sign (exact)
DAG_HASHED_B_PER_REC = {"default": 44, "fig4": 57, "sign_heavy": 102, "cross_heavy": 119,
                        "lookup_heavy": 73}
FNV_INSTR_PER_BYTE = 4.75  # LOP3 xor + IMAD.WIDE + IMAD + LEA (+ byte extract), DESIGN §4


def algorithmic_bytes(corpus, counters, dict_probes_per_row: int = 0) -> dict:
    """Compulsory HBM bytes of one step (SURVEY.md §8 d): the driver
    columns, the basic columns the merge reads, the CSR written and, for
    lookup_heavy, one 32-B sector per probe of the >L2 query_dict.  Index and
    hash-table sectors are implementation traffic (they show in ``traffic``).

    dict_probes_per_row: lookups per live row into dictionaries larger than L2."""
    d = corpus.driver
    inp = sum(d.columns[c].nbytes() for c in d.order)
    b = corpus.basic
    basic = sum(b.columns[c].nbytes() for c in ("instance_id", "basic_a", "basic_b"))
    out = counters.instances * (8 + 1 + 8) + counters.signs * (2 + 8)
    dprobe = 32 * dict_probes_per_row * counters.joined
    return {"input": inp, "basic": basic, "dict_probe": dprobe, "output": out,
            "total": inp + basic + dprobe + out}


def int_ceiling_s(dag: str, records: int, counters, clock_mhz: float) -> float:
    """Integer-pipe floor of one step: the FNV-1a instructions alone at full issue
    on 148 SMs x 4 schedulers x 32 lanes (SURVEY.md §8 d)."""
    hashed = DAG_HASHED_B_PER_REC.get(dag, 0) * records + 9 * counters.instances + \
        10 * counters.signs
    return hashed * FNV_INSTR_PER_BYTE / (148 * 4 * 32 * clock_mhz * 1e6)


def relaunch_under_torchrun(args) -> int:
    """``bench.py --gpus N`` (N > 1) started as a plain process: start the N
    ranks itself (torchrun, one process per GPU, rendezvous on 127.0.0.1) and
    return their exit code.  Fails loudly when the box has fewer GPUs."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} needs {args.gpus} GPUs, this box has "
                                   f"{have}"}), flush=True)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator init (and NVLS use) in the log
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    print(f"[bench] starting {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def main():
    args = parse_args()
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        raise SystemExit(relaunch_under_torchrun(args))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    import torch
    from paper_2210_07768_b200 import engine as E
    from paper_2210_07768_b200 import runtime
    from paper_2210_07768_b200.config import config_from_dict
    from paper_2210_07768_b200.corpus import make_corpus_fast as make_corpus, write_corpus
    from paper_2210_07768_b200.workloads import workload_config, write_lookup_tables

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1 or "WORLD_SIZE" in os.environ:  # under torchrun: the NCCL path, any N
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    # what this rank extracts per step: one log (seed 11 + rank, weak scaling)
    # or, in C5 mode, its share of independent 1M-record shards (seeds 1000+k)
    from paper_2210_07768_b200.distributed import assign_shards, weak_seeds
    if args.shards:
        seeds = assign_shards(args.shards, args.shard_seed0, rank, world)
    else:
        seeds = weak_seeds(args.seed, rank)
    raw = workload_config(args.dag, batch_size=args.batch_size)
    t0 = time.time()
    shards, gen_s, prep_s = [], 0.0, 0.0
    for sd in seeds:
        t0 = time.time()
        corpus = make_corpus(args.rows, args.users, sd)
        gen_s += time.time() - t0
        tmp = Path(tempfile.mkdtemp(prefix="fbxbench"))
        write_corpus(corpus, tmp)
        if args.dag == "lookup_heavy":
            write_lookup_tables(tmp, args.users, args.lookup_fillers)
        cfg = config_from_dict(raw, tmp)
        views = {"user_events": corpus.driver, "user_profile": corpus.profile}
        t1 = time.time()
        prep = E.prepare(cfg, views, corpus.basic)
        eng = E.Engine(prep, views, corpus.basic, device=str(dev),
                       max_rows_per_launch=args.launch_rows)
        eng.bind_driver(E.DeviceView(corpus.driver, device=dev))
        eng.reserve(corpus.driver.row_count, eng.max_rows)
        prep_s += time.time() - t1
        shards.append((corpus, eng, tmp, cfg))
    corpus, eng, tmp, cfg = shards[0]
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    launches = [0]

    # C5: independent shards on several streams, so one shard's index builds
    # (latency-bound, few CTAs) overlap another shard's fused kernel
    nstreams = max(1, min(args.shard_streams, len(shards)))
    streams = [stream] + [torch.cuda.Stream(dev) for _ in range(nstreams - 1)]

    def run_shard(eng, n, ev=None, iev=None, s=None):
        """One run over a shard, as the reference runs it (pipeline.py:952-1094):
        the per-run prepare phase -- the side-view and basic-view indices rebuilt
        on the device from their resident images (:970-980) -- then the run's id
        set cleared and launches of at most --launch-rows rows, the look-back
        continuing across them."""
        s = stream if s is None else s
        with torch.cuda.stream(s):
            if iev is not None:
                iev[0].record(s)
            launches[0] += eng.rebuild_indices(s.cuda_stream)
            if iev is not None:
                iev[1].record(s)
            launches[0] += eng.begin_run(n)  # k_idset_clear + k_state_reset
            if ev is not None:
                ev[0].record(s)
            for lo in range(0, n, eng.max_rows):
                eng.launch(lo, min(lo + eng.max_rows, n), s.cuda_stream,
                           tile_base=eng.tile_of_row(lo))
                launches[0] += 1  # fbx_pipeline
            if ev is not None:
                ev[1].record(s)

    # ---- warmup + correctness of every shard ---------------------------------
    for _ in range(max(args.warmup, 3)):
        for corp, e, _, _ in shards:
            run_shard(e, corp.driver.row_count)
    results = [e.finish().counters for _, e, _, _ in shards]
    # every shard on every rank against the unmodified reference's own run of it
    checked = 0
    golden_xor = 0
    for sd, c in zip(seeds, results):
        want = golden_for(args.dag, sd, args.rows, args.users, args.batch_size)
        if want is None:
            continue
        if (c.digest, c.instances, c.signs) != want:
            raise SystemExit(f"parity failure on rank {rank} shard seed {sd}: got digest "
                             f"0x{c.digest:016x} / {c.instances} / {c.signs}, want "
                             f"0x{want[0]:016x} / {want[1]} / {want[2]}")
        checked += 1
        golden_xor ^= want[0]
    ab = None
    for (corp, _, _, _), cc in zip(shards, results):
        big = 1 if (args.dag == "lookup_heavy" and args.lookup_fillers * 64 > (126 << 20)) else 0
        b = algorithmic_bytes(corp, cc, big)
        ab = b if ab is None else {k: ab[k] + b[k] for k in ab}

    # ---- timed device-resident steps ---------------------------------------
    K = args.steps
    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in shards] for _ in range(K)]
    ievs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
             for _ in shards] for _ in range(K)]
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(K)]
    graphs = []
    if args.graph:
        # one CUDA graph per shard: its whole step (memsets, index build, run reset,
        # fused launches) replayed as one launch; timing events recorded inside it
        # (external events), read back after every step
        torch.cuda.synchronize(dev)
        launches[0] = 0
        cap = torch.cuda.Stream(dev)  # capture needs a non-default stream
        for j, (corp, e, _, _) in enumerate(shards):
            gev = tuple(torch.cuda.Event(enable_timing=True, external=True) for _ in range(2))
            giev = tuple(torch.cuda.Event(enable_timing=True, external=True) for _ in range(2))
            g = torch.cuda.CUDAGraph()
            cap.wait_stream(torch.cuda.current_stream(dev))
            # thread_local: the NCCL watchdog's event queries (torchrun) must not
            # invalidate the capture
            with torch.cuda.graph(g, stream=cap, capture_error_mode="thread_local"):
                run_shard(e, corp.driver.row_count, gev, giev, cap)
            graphs.append((g, gev, giev, streams[j % nstreams]))
        graph_launches = launches[0]
        torch.cuda.synchronize(dev)
    clocks = Clocks(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    launches[0] = 0
    kern_total = index_total = 0.0
    for k in range(K):
        runtime.l2_flush(flush.data_ptr(), flush.numel(), stream.cuda_stream)  # L2 flush
        step_ev[k][0].record(stream)
        for s in streams[1:]:
            s.wait_stream(stream)
        if graphs:
            for g, _, _, s in graphs:
                with torch.cuda.stream(s):
                    g.replay()
        else:
            for j, ((corp, e, _, _), ev, iev) in enumerate(zip(shards, evs[k], ievs[k])):
                run_shard(e, corp.driver.row_count, ev, iev, streams[j % nstreams])
        for s in streams[1:]:
            stream.wait_stream(s)
        step_ev[k][1].record(stream)
        if graphs:  # the graph's events are re-recorded by the next replay
            torch.cuda.synchronize(dev)
            kern_total += sum(a.elapsed_time(b) for _, (a, b), _, _ in graphs)
            index_total += sum(a.elapsed_time(b) for _, _, (a, b), _ in graphs)
            launches[0] += graph_launches
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    if dist:
        dist.barrier()
    total_ms = sum(a.elapsed_time(b) for a, b in step_ev)
    if not graphs:
        kern_total = sum(a.elapsed_time(b) for row in evs for a, b in row)
        index_total = sum(a.elapsed_time(b) for row in ievs for a, b in row)
    results = [e.finish().counters for _, e, _, _ in shards]
    tot = torch.tensor([total_ms, kern_total], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms, kern_total = float(tot[0]), float(tot[1])
    # the one collective: all-gather of per-shard counters (distributed.py)
    from paper_2210_07768_b200.distributed import ShardResult, all_gather_results, combine
    mine = combine([ShardResult(corp.driver.row_count, r.instances, r.signs, r.digest,
                                r.malformed, r.filtered)
                    for (corp, _, _, _), r in zip(shards, results)])
    shard = ShardResult(mine.records, mine.instances, mine.signs, mine.digest, mine.malformed,
                        mine.filtered)
    totals = all_gather_results(shard, device=dev) if dist else combine([shard])
    run_digest = totals.digest
    from paper_2210_07768_b200.distributed import gather_parity
    try:
        gp = gather_parity(checked, len(seeds), golden_xor, run_digest, device=dev)
    except RuntimeError as exc:
        raise SystemExit(f"parity failure: {exc}")
    parity = {"digest": f"0x{run_digest:016x}", "instances": totals.instances,
              "signs": totals.signs, "shards_checked": gp["shards_checked"],
              "reference_xor": gp["reference_xor"],
              "source": "tests/golden/shard_goldens.json + SURVEY Appendix B (unmodified "
                        "reference run per shard)"}
    records_all = totals.records
    value = records_all * K / (total_ms / 1e3)
    ms_per_step = total_ms / K
    kern_avg_s = kern_total / K / 1e3
    n = corpus.driver.row_count
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except (OSError, ValueError):
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = ab["total"] / kern_avg_s / 1e9
    clk_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    hbm_floor = ab["total"] / (peak * 1e9)
    int_floor = sum(int_ceiling_s(args.dag, corp.driver.row_count, cc, clk_mhz)
                    for (corp, _, _, _), cc in zip(shards, results))
    # the generated plan's text: the same under ncu (FBX_DUMP_SOURCE renames the NVRTC
    # source, and -lineinfo carries the name into the cubin) and in a plain run
    plan_sha = hashlib.sha256(eng.prepared.program.source.encode()).hexdigest()[:16]
    roofline = {"bound": "hbm" if hbm_floor >= int_floor else "int",
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": None,
                "bytes_per_launch": ab, "kernel_ms": round(kern_avg_s * 1e3, 4),
                "index_build_ms": round(index_total / K, 4),
                "ceilings_ms": {"hbm": round(hbm_floor * 1e3, 4),
                                "int_pipe_fnv": round(int_floor * 1e3, 4)},
                "limiter": "instruction issue (see profiles/: inst_executed, issue_active)",
                **({"note": f"shards on {nstreams} streams: kernel events overlap other "
                            "shards' index builds, so kernel_ms / frac are conservative"}
                   if nstreams > 1 else {}),
                "plan_sha": plan_sha,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.65 TB/s"}
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        try:
            t = json.loads(prof.read_text()).get(args.dag)
            if t and t.get("plan_sha") == plan_sha:  # same plan, measured by ncu
                roofline["traffic"] = t["dram_bytes"]
                roofline["traffic_source"] = t.get("source")
        except (OSError, ValueError):
            pass

    # ---- e2e through the public API with host buffers ----------------------
    e2e = None
    if not args.no_e2e and len(shards) == 1:
        views = {"user_events": corpus.driver, "user_profile": corpus.profile}
        eng2 = E.Engine(E.prepare(cfg, views, corpus.basic), views, corpus.basic,
                        device=str(dev), max_rows_per_launch=args.launch_rows)
        e2e = measure_e2e(torch, E, eng, corpus, dev, stream, K, world, dist,
                          args.e2e_slice_rows, eng2, args.e2e_stream_slice_rows, cfg,
                          args.api_slice_rows)
        if e2e["digest"] != parity["digest"]:
            raise SystemExit(f"e2e parity failure: {e2e['digest']} != {parity['digest']}")

    if not args.no_e2e and len(shards) > 1:
        e2e = measure_e2e_shards(torch, E, shards, seeds, args, dev, world, dist, golden_xor,
                                 checked == len(seeds))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            if reference_installed():  # the unmodified reference on this very log's files
                (tmp / "cfg.json").write_text(json.dumps(raw))
                cpu = reference_cpu(tmp, args.ref_sample_rows, rows=args.rows)
            else:
                cpu = cpu_baseline(corpus, raw, tmp, args.cpu_sample_rows)
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "error": str(exc)[:200]}
    out = {
        "metric": "raw log records/sec extracted (device-resident input)",
        "value": round(value, 1), "unit": "records/s", "n_gpus": world, "steps": K,
        "warmup": max(args.warmup, 3), "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (gen_corpus restatement, byte-identical to the reference)",
        "config": {"workload": (f"{args.dag} DAG (SURVEY Appendix B), "
                                + (f"C5: {len(shards)} of {args.shards} independent "
                                   f"{args.rows}-record shards (seeds {args.shard_seed0}+k) "
                                   "on this rank" if args.shards else
                                   f"{args.rows} records/GPU, seed {args.seed}+rank")
                                + f", users {args.users}, full emit incl. basic merge"),
                   "batch_size": cfg.batch_size,
                   **({"query_dict_keys": 47296 + args.lookup_fillers}
                      if args.dag == "lookup_heavy" else {}),
                   "l2": "flushed between steps (512 MiB write, outside the timed events)",
                   "step_launch": ("one CUDA graph replay per shard (memsets, index build, "
                                   "run reset, fused launches)" if graphs else
                                   "kernels launched one by one"),
                   **({"shard_streams": nstreams} if len(shards) > 1 else {}),
                   "parallelism": f"record-sharded x{world}"},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches[0], "clocks": clk,
        "parity": parity,
        "setup_s": {"corpus": round(gen_s, 1), "prepare": round(prep_s, 1)},
        "records_per_step": records_all,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


def measure_e2e_shards(torch, E, shards, seeds, args, dev, world, dist, golden_xor,
                       all_checked: bool) -> dict:
    """C5 end to end: every shard of this rank is its own reference pipeline,
    run through the drop-in ``run_pipelined(config)`` over the shard's FBXC
    files (page cache), one call after the other -- per shard the side and
    basic views are read, CRC-checked and indexed on the device and the driver
    streamed through the pinned ring -- and every shard's digest checked
    against the unmodified reference's.  One untimed warm-up call compiles the
    plan.  Wall clock over all shards, max over ranks."""
    E.run_pipelined(shards[0][3], slice_rows=args.api_slice_rows)  # plan + module
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    reps = [E.run_pipelined(cfg, slice_rows=args.api_slice_rows) for _, _, _, cfg in shards]
    dt = time.perf_counter() - t0
    x, h2d = 0, 0
    for sd, rep in zip(seeds, reps):
        want = golden_for(args.dag, sd, args.rows, args.users, args.batch_size)
        if want is not None and (rep.digest, rep.instances, rep.signs) != want:
            raise SystemExit(f"C5 e2e parity failure, shard seed {sd}")
        x ^= rep.digest
        h2d += rep.bytes_h2d
    tt = torch.tensor([dt], dtype=torch.float64, device=dev)
    xs = torch.tensor([x & ((1 << 63) - 1), x >> 63], dtype=torch.int64, device=dev)
    if dist:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        parts = [torch.empty_like(xs) for _ in range(world)]
        dist.all_gather(parts, xs)
        x = 0
        for q in parts:
            x ^= int(q[0]) | (int(q[1]) << 63)
    records = sum(c.driver.row_count for c, _, _, _ in shards) * world
    if all_checked and dist is None and x != golden_xor:
        raise SystemExit("C5 e2e: shard digest XOR differs from the reference XOR")
    return {"value": round(records / float(tt[0]), 1), "unit": "records/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": (2 * runtime_state_bytes() + 8)
            * len(shards), "digest": f"0x{x:016x}", "seconds": round(float(tt[0]), 3),
            "path": f"{len(shards)} shards per rank, each its own run_pipelined(config) over "
                    "its FBXC files (page cache): side + basic views read, CRC-checked and "
                    "indexed on the device, the driver streamed through a pinned ring; "
                    "every shard's digest = the unmodified reference's; one step = all "
                    "shards once"}


def runtime_state_bytes() -> int:
    from paper_2210_07768_b200 import runtime
    return runtime.STATE_BYTES


def measure_e2e(torch, E, eng, corpus, dev, stream, K, world, dist, slice_rows=1 << 18,
                eng2=None, stream_slice_rows=1 << 20, cfg=None, api_slice_rows=1 << 18):
    """Same metric end to end from HOST data.

    Headline (``value``): the reference-facing call itself, ``run_pipelined(cfg)``
    (pipeline.py:952) over the log's FBXC files in the page cache, one call per
    step: plan (cached), side + basic views read, CRC-checked and indexed on the
    device, the driver streamed in slices (parallel pread -> pinned ring -> H2D
    -> fused kernel), counters + digest read back.  Every step moves all its
    input bytes H2D inside the timed region.

    Also reported (engine.StreamedRun, the trainer hand-off with the whole CSR
    copied back D2H): a stream of K steps on two alternating engines, the same
    step synchronised on its own, and the device-sink variant."""
    n = corpus.driver.row_count
    api = None
    if cfg is not None:
        reps, times = [], []
        if dist:
            dist.barrier()
        for k in range(K + 1):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            rep = E.run_pipelined(cfg, slice_rows=api_slice_rows)
            dt = time.perf_counter() - t0
            reps.append(rep)
            if k:  # the first call compiles / loads the plan: a warm-up
                times.append(dt)
        tt = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
        if dist:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        rep = reps[-1]
        if len({r.digest for r in reps}) != 1:
            raise SystemExit("e2e parity failure (run_pipelined)")
        api = {"value": round(n * world * K / float(tt[0]), 1), "digest": rep.digest,
               "h2d": rep.bytes_h2d, "ms": round(1e3 * float(tt[0]) / K, 3),
               "stages_ms": {k: round(1e3 * v, 3) for k, v in rep.stage_seconds.items()},
               "launches": rep.launches}
    sr = E.StreamedRun(eng, corpus.driver, slice_rows=slice_rows)
    srs = [E.StreamedRun(e, corpus.driver, slice_rows=stream_slice_rows, taper=False)
           for e in (eng, eng2) if e]
    want = None
    # single synchronised steps
    times = []
    if dist:
        dist.barrier()
    for k in range(K + 1):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        tot = sr.run()
        torch.cuda.synchronize(dev)
        dt = time.perf_counter() - t0
        want = want or tot.digest
        if tot.digest != want:
            raise SystemExit("e2e parity failure (single step)")
        if k:  # first pass is a warm-up
            times.append(dt)
    single = n * world * K / sum(times)
    # pipelined stream of K steps
    for r in srs:  # warm every engine's StreamedRun
        r.run()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    srs[0].start()
    for k in range(K):
        if k + 1 < K:
            srs[(k + 1) % len(srs)].start()
        tot = srs[k % len(srs)].finish()
        if len(srs) == 1 and k + 1 < K:
            srs[0].wait()
        if tot.digest != want:
            raise SystemExit("e2e parity failure (stream)")
    for r in srs:
        r.wait()
    torch.cuda.synchronize(dev)
    dt = time.perf_counter() - t0
    # device sink: the same stream with the CSR left in HBM for a GPU trainer
    dvs = [E.StreamedRun(r.eng, corpus.driver, slice_rows=stream_slice_rows, taper=False,
                         sink="device") for r in srs]
    for r in dvs:
        r.run()
    torch.cuda.synchronize(dev)
    t1 = time.perf_counter()
    dvs[0].start()
    for k in range(K):
        if k + 1 < K:
            dvs[(k + 1) % len(dvs)].start()
        dtot = dvs[k % len(dvs)].finish()
        if len(dvs) == 1 and k + 1 < K:
            dvs[0].wait()
        if dtot.digest != want:
            raise SystemExit("e2e parity failure (device sink)")
    torch.cuda.synchronize(dev)
    ddt = time.perf_counter() - t1
    tt = torch.tensor([dt, sum(times), ddt], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    rate = n * world * K / float(tt[0])
    single = n * world * K / float(tt[1])
    dev_rate = n * world * K / float(tt[2])
    if api is not None and api["digest"] != tot.digest:
        raise SystemExit("e2e parity failure (run_pipelined vs StreamedRun)")
    streamed = {"value": round(rate, 1), "h2d_bytes_per_step": sr.h2d_bytes,
                "d2h_bytes_per_step": sr.d2h_bytes,
                "single_step_value": round(single, 1),
                "device_sink_value": round(dev_rate, 1),
                "device_sink_d2h_bytes_per_step": dvs[0].d2h_bytes,
                "path": f"engine.StreamedRun x{len(srs)} engines alternating over a stream of "
                        f"{K} 1M-record steps from pre-packed pinned slices; "
                        f"{len(srs[0].bounds)} slices per step (<= {srs[0].slice_rows} rows); "
                        "pinned H2D / fused kernel / D2H of the full CSR on three streams per "
                        "engine; wall clock over the whole stream. single_step_value: each "
                        "step synchronised on its own; device_sink_value: CSR left in HBM "
                        "for a GPU trainer"}
    if api is None:
        return {"value": streamed["value"], "unit": "records/s",
                "h2d_bytes_per_step": sr.h2d_bytes, "d2h_bytes_per_step": sr.d2h_bytes,
                "digest": f"0x{tot.digest:016x}", "path": streamed["path"]}
    d2h = 2 * runtime_state_bytes() + 4 * 2  # run + prepare state words, two CRC words
    return {"value": api["value"], "unit": "records/s", "h2d_bytes_per_step": api["h2d"],
            "d2h_bytes_per_step": d2h, "digest": f"0x{api['digest']:016x}",
            "ms_per_step": api["ms"], "stages_ms": api["stages_ms"],
            "launches_per_step": api["launches"],
            "path": "run_pipelined(config) -- the reference-facing drop-in -- over the log's "
                    "FBXC files (page cache), one call per step, wall clock; slices of "
                    f"{api_slice_rows} rows read by parallel pread into a pinned ring, H2D "
                    "overlapped with the fused kernel; the RunReport's counters and digest "
                    "read back",
            "csr_to_host": streamed}


# ---------------------------------------------------------------------------
# the UNMODIFIED reference on the host cores (baseline/_ref: pip-installed from
# /root/reference/pkg; travels to the GPU box).  Falls back to the oracle port
# (oracle/featurebox_oracle.py) only when the installed reference is absent.
# ---------------------------------------------------------------------------

REF_PKG = ROOT / "baseline" / "_ref"


def reference_installed() -> bool:
    return (REF_PKG / "featurebox" / "__init__.py").exists()


def _ref_modules():
    if str(REF_PKG) not in sys.path:
        sys.path.insert(0, str(REF_PKG))
    import featurebox.columnstore as RCS
    import featurebox.corpus as RC
    import featurebox.pipeline as RP
    return RC, RCS, RP


def reference_log(dag: str, rows: int, users: int, seed: int, batch_size: int) -> Path:
    """The benchmark log written by the reference's own (pure-Python) gen_corpus,
    with the Appendix-B DAG's config beside it."""
    from paper_2210_07768_b200.workloads import workload_config, write_lookup_tables
    RC, _, _ = _ref_modules()
    dest = Path(tempfile.mkdtemp(prefix="fbxreflog"))
    RC.gen_corpus(dest, rows=rows, users=users, seed=seed, views=2)
    if dag == "lookup_heavy":
        write_lookup_tables(dest, users)
    (dest / "cfg.json").write_text(json.dumps(workload_config(dag, batch_size=batch_size)))
    return dest


def _ref_sample(args):
    """One process: rows [lo, hi) of the log (driver + the matching basic rows,
    the whole profile view) through the unmodified reference -- its
    run_pipelined end to end, and its _extract_batch alone over the same
    sample's cleaned + joined chunks.  Returns (rows, e2e s, extract s, joined)."""
    log, lo, hi = args
    import shutil
    RC, RCS, RP = _ref_modules()
    sample = Path(tempfile.mkdtemp(prefix="fbxrefsample"))
    for name in ("user_profile.fbxc", "cfg.json", "city_dict.tsv", "token_dict.tsv",
                 "user_dict.tsv", "query_dict.tsv"):
        if (log / name).exists():
            shutil.copy(log / name, sample / name)
    for name in ("user_events.fbxc", "basic.fbxc"):  # gen_corpus: basic row i <-> driver row i
        batch, _ = RCS.read_columns(log / name, rows=(lo, hi))
        RCS.write_view(batch, sample / name)
    cfg = RP.load_config(sample / "cfg.json")
    t0 = time.perf_counter()
    RP.run_pipelined(cfg)
    t_e2e = time.perf_counter() - t0
    # extract-only: the same chunks, cleaned and joined outside the timed part
    prep = RP.prepare(cfg)
    ctx = RP._make_ctx(prep)
    drv = next(v for v in cfg.views if v.name == cfg.driver)
    sides = [v for v in cfg.views if v.name != cfg.driver]
    from featurebox.viewpipe import JoinIndex, JoinSpec, clean_views, join_with_index
    idx = [JoinIndex(clean_views(RCS.read_columns(v.path, v.columns)[0], v.policy),
                     JoinSpec(cfg.join_keys)) for v in sides]
    n = hi - lo
    t_ex, joined = 0.0, 0
    for c0 in range(0, n, cfg.batch_size):
        batch, _ = RCS.read_columns(drv.path, drv.columns, rows=(c0, min(c0 + cfg.batch_size, n)))
        t = clean_views(batch, drv.policy)
        for ix in idx:
            t = join_with_index(t, ix)
        joined += t.schema.row_count
        t1 = time.perf_counter()
        RP._extract_batch(t, prep, ctx)
        t_ex += time.perf_counter() - t1
    shutil.rmtree(sample, ignore_errors=True)
    return n, t_e2e, t_ex, joined


def _cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def reference_cpu(log: Path, sample_rows: int, procs: int | None = None,
                  offset: int = 0, rows: int = 1_000_000) -> dict:
    """All host cores, one process each, on disjoint samples cut from the exact
    log.  Rates = sample rows / slowest process (they run concurrently)."""
    import multiprocessing as mp
    import platform
    procs = procs or os.cpu_count() or 1
    jobs = []
    for k in range(procs):
        lo = (offset + k * sample_rows) % max(1, rows - sample_rows)
        jobs.append((log, lo, lo + sample_rows))
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_ref_sample, jobs)
    wall = time.perf_counter() - t0
    n = sum(r[0] for r in res)
    e2e = n / max(r[1] for r in res)
    ext = sum(r[3] for r in res) / max(r[2] for r in res)
    return {"value": e2e, "unit": "records/s", "cores": procs, "kind": "reference",
            "extract_only_joined_rows_per_s": round(ext, 1),
            "hot_path_records_per_s": round(e2e, 1),
            "sample": f"{procs} processes x {sample_rows} driver rows (+ their basic rows, the whole "
                      f"profile view) cut from the benchmark log, each through the UNMODIFIED "
                      f"reference (baseline/_ref): run_pipelined end to end, and _extract_batch "
                      f"alone over the same cleaned + joined chunks; rate = rows / slowest "
                      f"process (wall {wall:.1f}s)",
            "cpu_model": _cpu_model(), "python": platform.python_version()}


def reference_arm(args, rank, world):
    """The reference's own CPU implementation of the path on the host cores,
    rank 0 only: the unmodified reference package (baseline/_ref) over bounded
    samples of the same log the B200 arm extracts."""
    if rank != 0:
        return
    if not reference_installed():
        print(json.dumps({"impl": "reference", "unavailable": "baseline/_ref missing: pip install "
                          "--no-index --target baseline/_ref /root/reference/pkg"}), flush=True)
        return
    seed = args.seed
    log = reference_log(args.dag, args.rows, args.users, seed, args.batch_size)
    sample = args.ref_sample_rows
    procs = os.cpu_count() or 1
    rates, last = [], None
    for k in range(args.warmup + args.steps):
        last = reference_cpu(log, sample, procs, offset=k * procs * sample, rows=args.rows)
        if k >= args.warmup:
            rates.append(last["value"])
    value = statistics.mean(rates) if rates else 0.0
    out = {"impl": "reference", "metric": "raw log records/sec extracted (device-resident input)",
           "value": round(value, 1), "unit": "records/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(sample * procs / value * 1e3, 3) if value
           else None, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "u64", "data": "synthetic (the reference's own gen_corpus)",
           "config": {"workload": f"{args.dag} DAG (SURVEY Appendix B), samples of the "
                                  f"{args.rows}-record log (users {args.users}, seed {seed}), "
                                  "full emit incl. basic merge",
                      "batch_size": args.batch_size, "parallelism": f"{procs} host processes"},
           "cpu_baseline": {**(last or {}), "value": round(value, 1)},
           "e2e": {"value": round(value, 1), "unit": "records/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
