"""Command-line front end, the reference's (cli.py:1-290) on the B200 engine.

    python -m paper_2210_07768_b200.cli run --config pipeline.json [--mode staged --staging dir]
    torchrun --nproc-per-node G -m paper_2210_07768_b200.cli run --config pipeline.json --sharded
    python -m paper_2210_07768_b200.cli plan --config pipeline.json
    python -m paper_2210_07768_b200.cli gen-corpus --out dir [--instances N ...]
    python -m paper_2210_07768_b200.cli bench-launch [--counts 1,10,100]

Exit codes as the reference: 0 success, 1 runtime failures (bad input data,
stage errors), 2 usage or configuration errors.  ``run`` prints the
reference's report text (its ``[report]`` block parses the same way);
``plan`` the layer plan, placement and the generated kernel's resources;
``bench-launch`` measures this device's per-launch overhead through
``fbx_launch`` (the reference fits its host model, cli.py:101-144).
``bench-alloc`` (the reference's host arena stress) has no counterpart: the
arena is the in-kernel bump pool (``fbx::pool_alloc``), exercised by every run.
"""

from __future__ import annotations

import argparse
import sys
import time
from dataclasses import replace
from pathlib import Path


def _fail(message: str, code: int) -> int:
    print(f"error: {message}", file=sys.stderr)
    return code


def _write_report(args, text: str) -> None:
    print(text)
    if getattr(args, "report", None):
        Path(args.report).write_text(text + "\n", encoding="utf-8")


def cmd_run(args) -> int:
    from .config import ConfigError, load_config
    from .engine import run_pipeline
    try:
        config = load_config(args.config)
        overrides = {}
        if args.mode:
            overrides["mode"] = args.mode
        if args.workers is not None:
            overrides["workers"] = args.workers
        if args.batch_size is not None:
            overrides["batch_size"] = args.batch_size
        if args.staging:
            overrides["staging_dir"] = Path(args.staging)
        if overrides:
            config = replace(config, **overrides)
        if args.sharded:
            report = _run_sharded(config)
            if report is None:  # ranks other than 0 print nothing
                return 0
        else:
            report = run_pipeline(config)
    except ConfigError as exc:
        return _fail(str(exc), 2)
    except Exception as exc:  # noqa: BLE001 -- data or stage failure: runtime, not usage
        return _fail(str(exc), 1)
    _write_report(args, report.to_text())
    return 0


def _run_sharded(config):
    """One log over the torchrun ranks (sharded.run_sharded, NCCL): every rank
    gets the single run's report or failure; rank 0's is printed."""
    import os

    import torch
    import torch.distributed as dist
    from .config import ConfigError
    from .sharded import run_sharded
    if config.mode != "pipelined":
        raise ConfigError("--sharded runs the pipelined mode")
    if not dist.is_initialized():
        if "RANK" not in os.environ:
            raise ConfigError("--sharded: launch under torchrun (RANK / WORLD_SIZE unset)")
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
    try:
        report = run_sharded(config)
    finally:
        rank = dist.get_rank()
        dist.destroy_process_group()
    return report if rank == 0 else None


def cmd_plan(args) -> int:
    from .config import ConfigError, load_config
    from .engine import prepare
    from .opgraph import plan_report
    try:
        config = load_config(args.config)
        prepared = prepare(config)
        text = plan_report(prepared.plan, prepared.dag)
        prog = prepared.program
        text += (f"\nkernel: fbx_pipeline, {prog.threads} threads per chunk CTA, "
                 f"{prog.smem_bytes} B dynamic shared memory, "
                 f"{len(prog.side_kernels)} index kernel(s), cubin {len(prepared.cubin)} B")
    except ConfigError as exc:
        return _fail(str(exc), 2)
    except Exception as exc:  # noqa: BLE001
        return _fail(str(exc), 1)
    _write_report(args, text)
    return 0


def cmd_bench_launch(args) -> int:
    """Per-launch overhead of this device through the engine's own launch path
    (fbx_launch of the run-state snapshot kernel), fitted as the reference fits
    its model: least squares of time over launch count."""
    try:
        counts = [int(c) for c in args.counts.split(",")]
    except ValueError as exc:
        return _fail(str(exc), 2)
    import numpy as np
    import torch
    from . import runtime
    if not torch.cuda.is_available():
        return _fail("bench-launch needs a CUDA device", 1)
    st = torch.zeros(runtime.STATE_BYTES // 8, dtype=torch.int64, device="cuda")
    dst = torch.zeros(runtime.STATE_BYTES // 8, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    points = []
    for count in counts:
        best = float("inf")
        for _ in range(args.repeat):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(count):
                runtime.state_snapshot(st.data_ptr(), dst.data_ptr(), stream)
            torch.cuda.synchronize()
            best = min(best, (time.perf_counter() - t0) * 1e6)
        points.append((count, best))
    x = np.array([c for c, _ in points], float)
    y = np.array([u for _, u in points], float)
    slope = float(np.polyfit(x, y, 1)[0]) if len(points) > 1 else y[0] / max(x[0], 1)
    lines = ["launch overhead calibration (B200, fbx_launch path)"]
    lines += [f"  {c} launches -> {us:.3f} us" for c, us in points]
    lines.append(f"fitted per-launch overhead: {slope:.4f} us (measured)")
    lines += ["", "[report]", f"per_launch_us={slope:.6f}", "source=measured"]
    _write_report(args, "\n".join(lines))
    return 0


def cmd_gen_corpus(args) -> int:
    from .corpus import gen_corpus
    if args.instances < 0 or args.users < 1 or args.batch_size < 1:
        return _fail("instances must be >= 0; users and batch-size >= 1", 2)
    try:
        paths = gen_corpus(args.out, rows=args.instances, users=args.users, seed=args.seed,
                           batch_size=args.batch_size, views=args.views)
    except ValueError as exc:
        return _fail(str(exc), 2)
    except OSError as exc:
        return _fail(str(exc), 1)
    for name in sorted(paths):
        print(f"{name}: {paths[name]}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="featurebox-b200",
        description="Feature-extraction pipeline on the B200: run, plan, and benchmark.")
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("run", help="run a pipeline config end to end")
    p.add_argument("--config", required=True, help="JSON pipeline config path")
    p.add_argument("--mode", choices=("pipelined", "staged"))
    p.add_argument("--workers", type=int, help="host worker thread cap")
    p.add_argument("--batch-size", type=int, dest="batch_size")
    p.add_argument("--staging", help="directory for staged mode files")
    p.add_argument("--report", help="also write the report to this file")
    p.add_argument("--sharded", action="store_true",
                   help="one log over the torchrun ranks (one GPU each), the single run's report")
    p.set_defaults(func=cmd_run)

    p = sub.add_parser("plan", help="print the layer plan and the generated kernel")
    p.add_argument("--config", required=True, help="JSON pipeline config path")
    p.add_argument("--report", help="also write the plan to this file")
    p.set_defaults(func=cmd_plan)

    p = sub.add_parser("bench-launch", help="measure the per-launch overhead")
    p.add_argument("--counts", default="1,10,100,1000,10000",
                   help="launch counts to measure (comma separated)")
    p.add_argument("--repeat", type=int, default=5)
    p.add_argument("--report", help="also write the result to this file")
    p.set_defaults(func=cmd_bench_launch)

    p = sub.add_parser("gen-corpus", help="generate the synthetic corpus")
    p.add_argument("--out", required=True, help="output directory")
    p.add_argument("--instances", type=int, default=20_000)
    p.add_argument("--views", type=int, choices=(1, 2), default=2)
    p.add_argument("--users", type=int, default=2_000)
    p.add_argument("--seed", type=int, default=7)
    p.add_argument("--batch-size", type=int, default=512, dest="batch_size")
    p.set_defaults(func=cmd_gen_corpus)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    return args.func(args)


if __name__ == "__main__":
    sys.exit(main())
