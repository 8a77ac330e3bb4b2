"""The B200 extraction engine: prepare a plan, keep views in HBM, run chunks.

Drop-in boundary (SURVEY.md §8 b): the reference's per-record path between
``read_columns`` of a driver chunk and the training sink --
``clean_views`` -> ``join_with_index`` -> ``_extract_batch`` ->
``check_unique_ids`` + basic merge -> ``_Emitter`` / ``emit_minibatch`` ->
``TrainingSink`` (pipeline.py:952-1094) -- runs as one generated CUDA kernel
per launch (codegen.py) through the C-ABI (include/fbx.h).

* ``prepare(config)`` mirrors the reference's ``prepare`` (pipeline.py:568-694):
  the same validation and errors, then the plan IR, code generation and NVRTC
  compilation (host only: no GPU needed).
* ``Engine`` owns the device state: the compiled program, side-view join
  indexes, the basic-view index, dictionary hash tables, the run-wide
  instance-id set, the bump pool and the output CSR arena.
* ``Engine.run(driver_rows)`` launches the fused kernel over a row range of a
  device-resident driver view and returns a ``CsrBatch`` (device tensors) and
  the counters; ``run_pipelined(config)`` is the whole reference run and
  returns the reference's ``RunReport``.

There is no CPU execution path: without a CUDA device ``Engine`` raises.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import Mapping

import numpy as np

from . import codegen, placement, runtime
from .columns import Kind, ViewImage, open_view, read_view
from .config import (ConfigError, EmitError, BatchInvariantError, CleanConfigError,
                     LayerExecutionError, MergeUniquenessError, PipelineConfig, PoolExhausted,
                     StageError, UnsupportedOnDevice, bind_filter, cleaned_kinds,
                     validate_clean_policy, run_workers)
from .featureops import FeatureConfigError, output_domains, resolve_function
from .opgraph import (DEVICE, OperatorDag, LayerPlan, PlacementBudget, expand_call_graph,
                      layer_schedule, place_operators, reference_node_order,
                      reference_placement)

STAGE_NAMES = {v: k for k, v in codegen.STAGE.items()}
ERR_NAMES = {v: k for k, v in codegen.ERR.items()}


# ---------------------------------------------------------------------------
# prepare (host, once per run)
# ---------------------------------------------------------------------------

@dataclass
class Prepared:
    config: PipelineConfig
    dag: OperatorDag
    plan: LayerPlan
    ir: codegen.PlanIR
    program: codegen.Program
    cubin: bytes
    extract_outputs: tuple[tuple[str, Kind, str], ...]
    node_names: list[str]
    schemas: dict[str, dict[str, Kind]]
    basic_kinds: dict[str, Kind]


def _schema(view: ViewImage | None, path: Path, wanted, where: str) -> dict[str, Kind]:
    if view is not None:
        kinds = {n: view.columns[n].kind for n in view.order}
    else:
        try:
            kinds = dict(open_view(path).schema)
        except OSError as exc:
            raise ConfigError(f"{where}: cannot open: {exc}") from exc
    if wanted is not None:
        missing = set(wanted) - set(kinds)
        if missing:
            raise ConfigError(f"{where}: columns {sorted(missing)} not in file")
        kinds = {n: k for n, k in kinds.items() if n in set(wanted)}
    return kinds


def prepare(config: PipelineConfig, views: Mapping[str, ViewImage] | None = None,
            basic: ViewImage | None = None, stage_strings: bool | None = None,
            compile_program: bool = True) -> Prepared:
    """Validate the config against the schemas and build + compile the plan."""
    import os
    views = views or {}
    if stage_strings is None:
        stage_strings = os.environ.get("FBX_STAGE", "1") != "0"
    cleaned: dict[str, dict[str, Kind]] = {}
    raw: dict[str, dict[str, Kind]] = {}
    for v in config.views:
        kinds = _schema(views.get(v.name), v.path, v.columns, f"view {v.name!r}")
        try:
            validate_clean_policy(kinds, v.policy)
        except (CleanConfigError, KeyError) as exc:
            raise ConfigError(f"view {v.name!r}: {exc}") from exc
        raw[v.name] = kinds
        cleaned[v.name] = cleaned_kinds(kinds, v.policy)
    dk = cleaned[config.driver]
    for col in (config.instance_column, config.label_column):
        if col not in dk:
            raise ConfigError(f"driver view lacks required column {col!r}")
        if dk[col] is not Kind.INT64:
            raise ConfigError(f"column {col!r} must be Int64")
    joined = dict(dk)
    for v in config.views:
        if v.name == config.driver:
            continue
        side = cleaned[v.name]
        for key in config.join_keys:
            if key not in joined or key not in side:
                raise ConfigError(f"join key {key!r} missing from an input view")
            if dk[key] is not side[key]:
                raise ConfigError(f"join key {key!r}: kind mismatch across views")
        for name, kind in side.items():
            if name in config.join_keys:
                continue
            if name in joined:
                raise ConfigError(f"column {name!r} appears in two views; project or rename")
            joined[name] = kind
    try:
        dag = expand_call_graph(config.operators)
        plan = place_operators(layer_schedule(dag), PlacementBudget(config.device_budget_bytes),
                               dag)
        fns = {}
        for name, node in dag.nodes.items():
            fn = resolve_function(node.func.spec, config.tables)
            want = "tuple" if node.role == "body" else "scalar"
            if fn.arity != want:
                raise FeatureConfigError(f"{name}: function {node.func.spec!r} has arity "
                                         f"{fn.arity}, {node.role} node needs {want}")
            fns[name] = fn
    except (FeatureConfigError, ValueError) as exc:
        if isinstance(exc, ConfigError):
            raise
        raise ConfigError(str(exc)) from exc
    missing = set(dag.external_inputs()) - set(joined)
    if missing:
        raise ConfigError(f"operator inputs {sorted(missing)} not present after the join")
    for node in dag.nodes:
        if node in joined:
            raise ConfigError(f"operator node {node!r} collides with a table column name")
    extract_outputs, produced = [], set()
    for spec in config.operators:
        domains = output_domains(spec, config.tables)
        for col in spec.outputs:
            if col in joined:
                raise ConfigError(f"output column {col!r} collides with a table column")
            extract_outputs.append((col, Kind.INT64 if domains[col] == "u64" else Kind.UTF8,
                                    domains[col]))
            produced.add(col)
    bkinds = _schema(basic, config.basic_path, config.basic_columns, "basic features")
    if config.instance_column not in bkinds:
        raise ConfigError(f"basic features lack instance column {config.instance_column!r}")
    overlap = (set(bkinds) - {config.instance_column}) & (set(joined) | produced)
    if overlap:
        raise ConfigError(f"basic columns {sorted(overlap)} collide with pipeline columns")
    merged = set(joined) | produced | set(bkinds)
    doms = {c: d for c, _, d in extract_outputs}
    for col in config.features:
        if col not in merged:
            raise ConfigError(f"feature column {col!r} not in the merged table")
        if col in doms:
            if doms[col] != "u64":
                raise ConfigError(f"feature column {col!r} is not sign-valued")
        else:
            kind = bkinds.get(col, joined.get(col))
            if kind is not Kind.INT64:
                raise ConfigError(f"feature column {col!r} must be Int64")

    # ---- plan IR --------------------------------------------------------------
    def view_ir(name: str) -> codegen.ViewIR:
        v = config.view(name)
        pol = v.policy
        flt = bind_filter(pol.filter, cleaned[name]) if pol.filter is not None else None
        keys = () if name == config.driver else tuple(config.join_keys)
        return codegen.ViewIR(name, dict(raw[name]), dict(pol.fills), list(pol.extractions),
                              flt, keys)

    refplace = reference_placement(dag, config.device_budget_bytes)
    order = reference_node_order(plan, refplace)
    rank = {n: i for i, (_, n) in enumerate(order)}
    specs = {s.name: s for s in config.operators}
    pre_of: dict[str, dict[int, str]] = {}
    nodes = []
    for layer, name in order:
        nd = dag.nodes[name]
        if nd.role == "pre":
            pre_of.setdefault(nd.op, {})[nd.slot] = name
            inputs = nd.reads
        elif nd.role == "body":
            inputs = specs[nd.op].inputs
        else:
            inputs = ()
        ref_pool = (fns[name].op == "token" and nd.role != "body"
                    and refplace[name] == DEVICE)
        nodes.append(codegen.NodeIR(name, nd.role, nd.op, fns[name], layer, rank[name],
                                    tuple(inputs), nd.slot, nd.writes, ref_pool))
    tables = {t: i for i, t in enumerate(sorted(config.tables))}
    ir = codegen.PlanIR(
        driver=view_ir(config.driver),
        sides=[view_ir(v.name) for v in config.views if v.name != config.driver],
        basic=codegen.ViewIR("basic", dict(bkinds), {}, [], None, (config.instance_column,)),
        join_keys=tuple(config.join_keys), nodes=nodes, pre_of=pre_of,
        producer=dict(dag.col_producer), features=dict(config.features),
        instance_column=config.instance_column, label_column=config.label_column,
        chunk=config.batch_size, tables=tables,
        table_defaults={t: config.tables[t].default for t in config.tables},
        extract_outputs=[(c, d) for c, _, d in extract_outputs], stage_strings=stage_strings,
        pool_bytes=config.pool_bytes, lanes_per_group=config.lanes_per_group)
    prog = codegen.generate(ir)
    cubin = runtime.compile_source(prog.source) if compile_program else b""
    return Prepared(config, dag, plan, ir, prog, cubin, tuple(extract_outputs),
                    [n for _, n in order], raw, bkinds)


# ---------------------------------------------------------------------------
# device views
# ---------------------------------------------------------------------------

def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 engine needs a CUDA device (no CPU execution path)")
    return torch


def _pad16(a: np.ndarray) -> np.ndarray:
    raw = np.ascontiguousarray(a).view(np.uint8).reshape(-1)
    out = np.zeros(((raw.size + 31) // 16) * 16, dtype=np.uint8)
    out[: raw.size] = raw
    return out


class DeviceView:
    """FBXC column images resident in HBM (16-byte padded segments)."""

    def __init__(self, view: ViewImage, columns=None, device="cuda"):
        torch = _torch()
        self.n = view.row_count
        self.kinds = {n: view.columns[n].kind for n in view.order}
        self.tensors: dict[str, dict[str, "torch.Tensor"]] = {}
        self.bytes = 0
        for name in view.order:
            if columns is not None and name not in columns:
                continue
            col = view.columns[name]
            parts = {"nulls": col.nulls[: (col.n + 7) // 8], "data": col.data}
            if col.kind.var_length:
                parts["offsets"] = col.offsets
            self.tensors[name] = {}
            for part, arr in parts.items():
                host = torch.from_numpy(_pad16(arr))
                t = host.to(device, non_blocking=False)
                self.tensors[name][part] = t
                self.bytes += arr.nbytes
        self.torch = torch

    def ptr(self, name: str, part: str) -> int:
        t = self.tensors[name].get(part)
        return 0 if t is None else t.data_ptr()

    @classmethod
    def from_fbxc(cls, path, columns=None, device="cuda", verify: bool = True) -> "DeviceView":
        """FBXC ingest with no decode (columnstore.py:499-608): the
        file body goes to HBM in one copy and the columns are views of it.  A full
        read checks the body's CRC-32 on the device (columnstore.py:554-562)."""
        from .columns import ChecksumError, open_view
        torch = _torch()
        vf = open_view(path)
        dev = torch.device(device)
        mm = np.memmap(vf.path, dtype=np.uint8, mode="r")
        body = torch.zeros(vf.body_bytes + 64, dtype=torch.uint8, device=dev)
        host = torch.from_numpy(np.array(mm[vf.body_offset:vf.body_offset + vf.body_bytes]))
        body[:vf.body_bytes].copy_(host)
        del mm
        names = [n for n, _ in vf.schema]
        if verify and (columns is None or set(columns) >= set(names)):
            crc = crc32_device(body[:vf.body_bytes])
            if crc != vf.checksum:
                raise ChecksumError(f"{vf.path}: body CRC {crc:#010x} != footer {vf.checksum:#010x}")
        self = cls.__new__(cls)
        self.n = vf.row_count
        self.kinds = {n: k for n, k in vf.schema}
        self.tensors, self.bytes, self.torch = {}, 0, torch
        # FBXC segments are packed (byte-identical to the reference writer); the
        # kernels want 16-B aligned segments with 16 B of slack: one device-side
        # copy per segment into an aligned arena
        want = [(name, part) for name, _ in vf.schema
                if columns is None or name in columns
                for part in ("nulls", "data", "offsets") if (name, part) in vf.segments]
        place, cur = {}, 0
        for key in want:
            place[key] = cur
            cur += (vf.segments[key][1] + 31) // 16 * 16
        arena = torch.zeros(cur + 16, dtype=torch.uint8, device=dev)
        for (name, part), dst in place.items():
            o, ln = vf.segments[(name, part)]
            a = o - vf.body_offset
            if ln:
                arena[dst:dst + ln].copy_(body[a:a + ln])
            self.tensors.setdefault(name, {})[part] = arena[dst:dst + ln]
            self.bytes += ln
        self._arena = arena
        return self


    @classmethod
    def from_file(cls, path, columns=None, device="cuda", verify: bool = True,
                  defer_crc: bool = False) -> "DeviceView":
        """FBXC ingest through the host reader (fbx_read_spans): the wanted
        segments are read by parallel pread into pinned memory and reach HBM in
        one H2D copy, with no decode, no page faults on a mapping and no pageable
        staging.  A full read (every column) moves the whole body and checks its
        CRC-32 on the device first (columnstore.py:554-562), then lays the
        segments out 16-B aligned by device copies.  ``defer_crc``: the CRC stays
        on the device until ``verify_crc()`` (no host synchronisation here)."""
        from .columns import UnknownColumnError
        torch = _torch()
        vf = open_view(path)
        names = [n for n, _ in vf.schema]
        if columns is not None:
            unknown = set(columns) - set(names)
            if unknown:
                raise UnknownColumnError(sorted(unknown)[0])
        full = columns is None or set(columns) >= set(names)
        dev = torch.device(device)
        want = [(name, part) for name, _ in vf.schema
                if columns is None or name in columns
                for part in ("nulls", "data", "offsets") if (name, part) in vf.segments]
        place, cur = {}, 0
        for key in want:
            place[key] = cur
            cur += (vf.segments[key][1] + 31) // 16 * 16
        self = cls.__new__(cls)
        self._crc = None
        self.n = vf.row_count
        self.kinds = {n: k for n, k in vf.schema if columns is None or n in columns}
        self.tensors, self.bytes, self.torch = {}, 0, torch
        arena = torch.zeros(cur + 16, dtype=torch.uint8, device=dev)
        if full and verify:
            host = torch.empty(vf.body_bytes + 16, dtype=torch.uint8, pin_memory=True)
            runtime.read_spans(vf.path, host.data_ptr(), [vf.body_offset], [vf.body_bytes], [0])
            body = torch.empty(vf.body_bytes + 64, dtype=torch.uint8, device=dev)
            body[:vf.body_bytes].copy_(host[:vf.body_bytes], non_blocking=True)
            self._crc = (crc32_device_async(body[:vf.body_bytes]), vf.checksum, vf.path)
            if not defer_crc:
                self.verify_crc()
            for (name, part), dst in place.items():
                o, ln = vf.segments[(name, part)]
                if ln:
                    a = o - vf.body_offset
                    arena[dst:dst + ln].copy_(body[a:a + ln])
        else:
            host = torch.empty(cur + 16, dtype=torch.uint8, pin_memory=True)
            keys = list(place)
            runtime.read_spans(vf.path, host.data_ptr(), [vf.segments[k][0] for k in keys],
                               [vf.segments[k][1] for k in keys], [place[k] for k in keys])
            arena.copy_(host, non_blocking=True)
        for (name, part), dst in place.items():
            ln = vf.segments[(name, part)][1]
            self.tensors.setdefault(name, {})[part] = arena[dst:dst + ln]
            self.bytes += ln
        self._arena = arena
        self.h2d_bytes = (vf.body_bytes if full and verify else cur)
        return self

    def verify_crc(self):
        """Raise ChecksumError if the body CRC computed on the device (a full
        read) differs from the file's trailer."""
        from .columns import ChecksumError
        if getattr(self, "_crc", None) is None:
            return
        out, want, path = self._crc
        crc = int(out.cpu().numpy().view(np.uint32)[0])
        self._crc = None
        if crc != want:
            raise ChecksumError(f"{path}: body CRC {crc:#010x} != footer {want:#010x}")


def crc32_device_async(t):
    """zlib CRC-32 of a contiguous device tensor's bytes (fbx_crc32), left in a
    one-word device tensor (no host synchronisation)."""
    torch = _torch()
    t = t.contiguous().view(torch.uint8)
    n = t.numel()
    scratch = torch.empty(runtime.crc32_scratch_words(n) + 1, dtype=torch.int32, device=t.device)
    out = torch.zeros(1, dtype=torch.int32, device=t.device)
    stream = torch.cuda.current_stream(t.device).cuda_stream
    runtime.crc32(t.data_ptr() if n else out.data_ptr(), n, scratch.data_ptr(), out.data_ptr(),
                  stream)
    return out


def crc32_device(t) -> int:
    """zlib CRC-32 of a contiguous device tensor's bytes (fbx_crc32)."""
    return int(crc32_device_async(t).cpu().numpy().view(np.uint32)[0])


# ---------------------------------------------------------------------------
# results
# ---------------------------------------------------------------------------

@dataclass
class Counters:
    digest: int = 0
    instances: int = 0
    signs: int = 0
    malformed: int = 0
    filtered: int = 0
    joined: int = 0
    launches: int = 0


@dataclass
class CsrBatch:
    """Emitted instances of one launch, in the reference's emission order:
    per driver chunk of ``batch_size`` rows, ascending u64 instance id."""

    ids: object      # torch uint64-as-int64 [n]
    labels: object   # torch uint8 [n]
    offsets: object  # torch int64 [n + 1]
    slots: object    # torch int16 (u16 bits) [m]
    signs: object    # torch int64 (u64 bits) [m]
    counters: Counters

    def minibatches(self, batch_size: int):
        """The trainer hand-off (TrainingSink.consume, pipeline.py:436-455): mini-batch
        b is instances [b*batch_size, (b+1)*batch_size) of the run -- the _Emitter's
        cut (pipeline.py:765-777) -- as device tensor views (offsets rebased to the
        batch's own sign range).  No host round trip."""
        n = self.counters.instances
        for b0 in range(0, n, batch_size):
            b1 = min(n, b0 + batch_size)
            off = self.offsets[b0:b1 + 1]
            s0, s1 = int(off[0].item()), int(off[-1].item())
            yield DeviceMiniBatch(self.ids[b0:b1], self.labels[b0:b1], off - s0,
                                  self.slots[s0:s1], self.signs[s0:s1])

    def to_numpy(self) -> dict[str, np.ndarray]:
        n, m = self.counters.instances, self.counters.signs
        return {"ids": self.ids[:n].cpu().numpy().view(np.uint64),
                "labels": self.labels[:n].cpu().numpy(),
                "offsets": self.offsets[: n + 1].cpu().numpy().view(np.uint64),
                "slots": self.slots[:m].cpu().numpy().view(np.uint16),
                "signs": self.signs[:m].cpu().numpy().view(np.uint64)}


@dataclass
class DeviceMiniBatch:
    """One emitted mini-batch in HBM (MiniBatch, pipeline.py:357-369): CSR of
    (slot u16, sign u64) per instance, rows in emission order."""

    ids: object      # torch int64 (u64 bits) [b]
    labels: object   # torch uint8 [b]
    offsets: object  # torch int64 [b + 1], offsets[0] == 0
    slots: object    # torch int16 (u16 bits)
    signs: object    # torch int64 (u64 bits)


def _nvtx_push(msg: str):
    """NVTX range around a launch / slice (visible to nsys / ncu --nvtx; a no-op
    without a tool attached)."""
    try:
        import torch
        torch.cuda.nvtx.range_push(msg)
    except Exception:  # noqa: BLE001 -- tracing must never fail a run
        pass


def _nvtx_pop():
    try:
        import torch
        torch.cuda.nvtx.range_pop()
    except Exception:  # noqa: BLE001
        pass


def _next_pow2(n: int) -> int:
    return 1 << max(4, (max(n, 1) - 1).bit_length())


class Engine:
    """Device state of one prepared plan on one GPU."""

    LAUNCH_ROWS_MAX = 1 << 24  # look-back counts are launch-local, 28 bits

    def __init__(self, prepared: Prepared, views: Mapping[str, ViewImage] | None = None,
                 basic: ViewImage | None = None, device: str = "cuda",
                 max_rows_per_launch: int = 1 << 22, pool_bytes_per_row: int = 96,
                 device_views: Mapping[str, "DeviceView"] | None = None,
                 defer_prepare_check: bool = False):
        torch = _torch()
        self.torch = torch
        self.prepared = prepared
        self.device = torch.device(device)
        self.config = cfg = prepared.config
        self.ir = ir = prepared.ir
        self.prog = prepared.program
        self.slots = self.prog.slots
        self.params = np.zeros(runtime.FBX_MAX_PARAM_SLOTS, dtype=np.uint64)
        # launches cover whole chunks; round UP so a run of <= max rows is one launch
        self.max_rows = min(-(-max_rows_per_launch // ir.chunk) * ir.chunk,
                            max(ir.chunk, self.LAUNCH_ROWS_MAX // ir.chunk * ir.chunk))
        self.pool_bytes_per_row = pool_bytes_per_row
        if prepared.program.json_kind:  # canonical JSON can outgrow its source (escapes)
            self.pool_bytes_per_row += 512
        with torch.cuda.device(self.device):
            # one loaded module per plan and device (engines of a plan share it)
            mods = prepared.__dict__.setdefault("_modules", {})
            if self.device not in mods:
                mods[self.device] = runtime.Program(prepared.cubin)
            self.module = mods[self.device]
            self.state = torch.zeros(runtime.STATE_BYTES // 8, dtype=torch.int64,
                                     device=self.device)
            self._set("state", self.state.data_ptr())
            self.prepare_counters = Counters()
            self._keep: list = []
            self._defer_prepare = defer_prepare_check
            self._upload_sides(views or {}, basic, device_views or {})
            self._upload_tables()
            self._idset_cap = 0
            self.idset = None
            self.streams = None
            if self.prog.smem_bytes:
                # static + dynamic > 48 KB needs the opt-in attribute
                self.module.set_dynamic_smem("fbx_pipeline", self.prog.smem_bytes)

    # -- params ----------------------------------------------------------------
    def _set(self, name: str, value: int):
        if name in self.slots:
            self.params[self.slots[name]] = np.uint64(int(value) & ((1 << 64) - 1))

    def _sm_count(self) -> int:
        if getattr(self, "_sms", None) is None:
            self._sms = self.torch.cuda.get_device_properties(self.device).multi_processor_count
        return self._sms

    def _stream(self) -> int:
        return self.torch.cuda.current_stream(self.device).cuda_stream

    # -- prepare-time device work -------------------------------------------------
    def _load_view(self, name: str, path: Path, columns, given: ViewImage | None) -> ViewImage:
        if given is not None:
            return given.project(columns)
        return read_view(path, columns)

    def _upload_sides(self, views: Mapping[str, ViewImage], basic: ViewImage | None,
                      device_views: Mapping[str, "DeviceView"]):
        """Side views and the basic view into HBM (``device_views``: already there,
        keyed by view name / "basic"), their hash indexes built by the prep kernels."""
        torch, cfg, ir = self.torch, self.config, self.ir
        sides = [(k, v) for k, v in enumerate(ir.sides)]
        if ir.basic is not None:
            sides.append((len(ir.sides), ir.basic))
        side_pool_cap = 0
        prepared_views = []
        self.side_tables = {}
        for k, v in sides:
            key = "basic" if v is ir.basic else v.name
            dv = device_views.get(key)
            if dv is None:
                if v is ir.basic:
                    img = self._load_view("basic", cfg.basic_path, cfg.basic_columns, basic)
                else:
                    src = cfg.view(v.name)
                    img = self._load_view(v.name, src.path, src.columns, views.get(v.name))
                dv = DeviceView(img, device=self.device)
            self._keep.append(dv)
            if v is ir.basic:
                self._basic_dv = dv
            n = dv.n
            cap = _next_pow2(2 * n)
            table = torch.zeros(cap * 32, dtype=torch.uint8, device=self.device)
            self._keep.append(table)
            self.side_tables[k] = table
            self._set(f"side{k}.rows", n)
            self._set(f"side{k}.table", table.data_ptr())
            self._set(f"side{k}.mask", cap - 1)
            for c in dv.tensors:
                for part in ("nulls", "data", "offsets"):
                    self._set(f"side{k}.{c}.{part}", dv.ptr(c, part))
            for e in v.extractions:
                if e.kind is Kind.UTF8:
                    ptr = torch.zeros(n + 2, dtype=torch.int64, device=self.device)
                    ln = torch.zeros(n + 4, dtype=torch.int32, device=self.device)
                    self._keep += [ptr, ln]
                    self._set(f"side{k}.ext.{e.output}.ptr", ptr.data_ptr())
                    self._set(f"side{k}.ext.{e.output}.len", ln.data_ptr())
                else:
                    val = torch.zeros(n + 2, dtype=torch.int64, device=self.device)
                    nul = torch.zeros(n + 16, dtype=torch.uint8, device=self.device)
                    self._keep += [val, nul]
                    self._set(f"side{k}.ext.{e.output}.val", val.data_ptr())
                    self._set(f"side{k}.ext.{e.output}.null", nul.data_ptr())
                src_bytes = int(dv.tensors[e.source]["data"].numel())
                grow = 6 if e.kind is Kind.JSON else 1  # ensure_ascii: 1 byte -> "\\uXXXX"
                side_pool_cap += grow * src_bytes + 128 * (n // 256 + 1)
            prepared_views.append((k, v, n))
        pool = torch.zeros(side_pool_cap + 256, dtype=torch.uint8, device=self.device)
        self._keep.append(pool)
        self._set("side_pool", pool.data_ptr())
        self._set("side_pool_cap", side_pool_cap)
        stream = self._stream()
        status = torch.zeros(1, dtype=torch.int64, device=self.device)
        runtime.state_reset(self.state.data_ptr(), status.data_ptr(), 1, stream)
        self._side_views = prepared_views
        self._launch_side_prep(stream)
        if self._defer_prepare:
            # the prepare-time state is kept on the device (stream-ordered copy)
            # and checked by finish_prepare() after the run: no host sync here
            self._prep_state = self.state.clone()
        else:
            self._settle_prepare(self._read_state())
        # basic uniqueness (pipeline.py:975): int-keyed basic indices raise it in the
        # prep kernel itself (basic_dup); other key shapes count repeats in the slots
        if ir.basic is not None and len(ir.sides) not in self.prog.int_keyed:
            self._check_basic_unique(len(ir.sides))

    def _settle_prepare(self, st: dict):
        self.prepare_counters.malformed = st["malformed"]
        self.prepare_counters.filtered = st["filtered"]
        if st["error_key"] != placement.NONE and \
                (st["error_key"] & 0xFF) == codegen.ERR["basic_dup"]:
            self._raise_basic_dup()
        self._raise_if_error(st, prepare=True)

    def _raise_basic_dup(self):
        """The basic view repeats an instance id (the index build saw it): name the
        id check_unique_ids names -- the first row, in row order, whose id occurred
        before (viewpipe.py:562-576, pipeline.py:975-980) -- by sorting the id
        column on the device (fbx_sort_keys + fbx_first_repeat, the staged mode's
        check)."""
        torch = self.torch
        dv = self._basic_dv
        col = self.ir.instance_column
        kind = dv.kinds[col]
        n = dv.n
        stream = self._stream()
        raw = dv.tensors[col]["data"]
        if kind is Kind.FLOAT32:
            bits = raw[:4 * n].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        else:
            bits = raw[:8 * n].view(torch.int64)
        m = max(n, 1)
        isnull = torch.zeros(m + 16, dtype=torch.uint8, device=self.device)
        runtime.call("fbx_unpack_nulls", dv.ptr(col, "nulls"), n, isnull.data_ptr(), stream)
        skey = torch.empty(m, dtype=torch.int64, device=self.device)
        srow = torch.empty(m, dtype=torch.int32, device=self.device)
        cnt = torch.zeros(1, dtype=torch.int64, device=self.device)
        rs = torch.empty(m, dtype=torch.int32, device=self.device)
        ks = torch.empty(m, dtype=torch.int64, device=self.device)
        fs = torch.empty(m, dtype=torch.uint8, device=self.device)
        runtime.call("fbx_sort_keys", bits.data_ptr(), isnull.data_ptr(), n, skey.data_ptr(),
                     srow.data_ptr(), cnt.data_ptr(), rs.data_ptr(), ks.data_ptr(), fs.data_ptr(),
                     stream)
        best = torch.empty(1, dtype=torch.int64, device=self.device)
        runtime.call("fbx_first_repeat", skey.data_ptr(), srow.data_ptr(), int(cnt.item()),
                     best.data_ptr(), stream)
        row = int(best.cpu().numpy().view(np.uint64)[0])
        if row == placement.NONE:
            return  # not a repeat after all: the error word decides
        v = int(bits[row].item())
        if kind is Kind.FLOAT32:
            v = float(np.int32(np.uint32(v)).view(np.float32))
        raise StageError("prepare", None,
                         MergeUniquenessError(f"basic features: duplicate instance id {v}"))

    def finish_prepare(self):
        """A deferred prepare check (``defer_prepare_check``): the side views'
        clean counters and the first prepare-time failure."""
        ps = getattr(self, "_prep_state", None)
        if ps is not None:
            self._prep_state = None
            raw = ps.cpu().numpy().view(np.uint64)
            self._settle_prepare({f: int(raw[i]) for i, f in enumerate(runtime.STATE_FIELDS)})

    def _launch_side_prep(self, stream: int) -> int:
        """Every side view's and the basic view's index build in one launch
        (fbx_side_prep_all: a CTA range per view)."""
        if not self._side_views:
            return 0
        total = 0
        for k, v, n in self._side_views:
            grid = max(1, min((n + 255) // 256, 1184))
            self._set(f"side{k}.grid", grid)
            total += grid
        self.module.launch("fbx_side_prep_all", total, 256, 0, stream, self.params)
        return 1

    def rebuild_indices(self, stream: int | None = None) -> int:
        """Rebuild the side-view and basic-view hash indices from their resident
        images (the per-run prepare phase of pipeline.py:970-980, on the device):
        zero the tables, re-run the prep kernels.  Returns the launch count.
        Prepare-time failures were checked when the engine was built."""
        stream = self._stream() if stream is None else stream
        for t in self.side_tables.values():
            runtime.memset_async(t.data_ptr(), 0, t.numel(), stream)
        return self._launch_side_prep(stream)

    def _check_basic_unique(self, k: int):
        torch = self.torch
        words = 4 if k in self.prog.int_keyed else 8  # 16-B ISlot | 32-B Slot
        aux = self.side_tables[k].view(torch.int32).view(-1, words)[:, 3]
        mx = int(aux.max().item()) if aux.numel() else 0
        if mx > 1:
            self._raise_basic_dup()
            raise StageError("prepare", None,
                             MergeUniquenessError("basic features: duplicate instance id"))

    def _upload_tables(self):
        torch = self.torch
        stream = self._stream()
        for name, ti in self.ir.tables.items():
            if f"dict{ti}.slots" not in self.slots:
                continue
            t = self.config.tables[name]
            # the HBM table is immutable: built once per loaded DictTable and device,
            # shared by every engine of that config (the reference parses the TSV
            # once per load_config too)
            built = t.__dict__.setdefault("_device_tables", {})
            if self.device not in built:
                blob, offs, vals = t.arrays()
                cap = _next_pow2(2 * len(vals))
                slots = torch.empty(cap * 32, dtype=torch.uint8, device=self.device)
                dblob = torch.from_numpy(_pad16(blob)).to(self.device)
                doffs = torch.from_numpy(_pad16(offs)).to(self.device)
                dvals = torch.from_numpy(_pad16(vals)).to(self.device)
                dup = torch.zeros(1, dtype=torch.int64, device=self.device)
                try:
                    runtime.dict_build(slots.data_ptr(), cap, dblob.data_ptr(), doffs.data_ptr(),
                                       dvals.data_ptr(), len(vals), dup.data_ptr(), stream)
                except runtime.FbxError as exc:
                    raise ConfigError(f"table {name!r}: {exc}") from exc
                built[self.device] = (slots, dblob, doffs, dvals, dup, cap)
            slots, dblob, doffs, dvals, dup, cap = built[self.device]
            self._keep += [slots, dblob, doffs, dvals, dup]
            self._set(f"dict{ti}.slots", slots.data_ptr())
            self._set(f"dict{ti}.mask", cap - 1)
            self._set(f"dict{ti}.keys", dblob.data_ptr())

    # -- state ---------------------------------------------------------------------
    def _read_state(self) -> dict[str, int]:
        raw = self.state.cpu().numpy().view(np.uint64)
        return {f: int(raw[i]) for i, f in enumerate(runtime.STATE_FIELDS)}

    def _raise_if_error(self, st: dict, prepare: bool = False):
        """Raise the run's first failure in the reference's pipeline order."""
        if prepare:
            self.raise_key(st["error_key"], st["error_detail"], st)
        else:
            self.raise_key(*self.first_failure(st), st)

    def first_failure(self, st: dict) -> tuple[int, int]:
        """(error key, detail) of the run's first failure in the reference's
        pipeline order (``placement.NONE`` without one).

        ``error_key`` holds the row-level failures at their own chunk.  Two
        kinds surface later in the reference and are placed here (placement.py):
        a repeated instance id fails the merge of the chunk holding its second
        occurrence (``fbx_dup_resolve``), and a null / non-0/1 label fails the
        merge of the chunk whose ``_Emitter.add`` flushes its mini-batch
        (pipeline.py:748-777) -- or the final flush (stage "emit", no batch
        index)."""
        key = st["error_key"]
        detail = st["error_detail"]
        if st.get("dup_seen"):
            dk, did = self._dup_key()
            if dk < key:
                key, detail = dk, did
        lk = st.get("emit_key_resolved") or self._label_key(st)
        if lk is not None and lk[0] < key:
            key, detail = lk
        return key, detail

    def raise_key(self, key: int, detail: int, st: dict | None = None):
        """Raise the StageError an error key names (nothing for ``NONE``)."""
        if key == placement.NONE:
            return
        chunk = key >> 32
        stage = STAGE_NAMES.get((key >> 28) & 0xF, "extract")
        layer = (key >> 20) & 0xFF
        rank = (key >> 8) & 0xFFF
        code = ERR_NAMES.get(key & 0xFF, "value")
        cause = _cause(code, detail, st or {})
        if stage == "extract" and layer:
            node = self.prepared.node_names[rank]
            cause = LayerExecutionError(layer, node, cause)
        raise StageError(stage, None if stage in ("prepare", "emit") else chunk, cause)

    def settle_run(self, st: dict) -> dict:
        """End of a run: note whether the id set saw a repeat (its pair array
        then needs clearing), repeat the run if the device arena ran out
        (ArenaRetry), settle the reference arena's PoolExhausted for flagged
        chunks (fbx_pool_account).  Returns the settled state."""
        self._dup_dirty = bool(st["dup_seen"])
        if st["pool_overflow"]:
            raise ArenaRetry(st["pool_overflow"])
        if st["pool_flagged"] and not getattr(self, "ring", False):  # ring: per launch
            self._pool_account()
            st = dict(st, **{k: v for k, v in self._read_state().items()
                             if k in ("error_key", "error_detail")})
        return st

    def check_run(self, st: dict):
        """``settle_run`` and raise the run's first failure."""
        self._raise_if_error(self.settle_run(st))

    def ring_after_launch(self, stream: int) -> int:
        """Ring runs: the reference arena's demand of the launch just enqueued is
        settled now (fbx_pool_account, stream-ordered), before the next launch
        reuses the planes.  Returns the number of launches enqueued."""
        if not (self.ring and self.prog.ref_pool):
            return 0
        self._pool_account(self._last_launch_tiles, stream)
        return 1

    def _pool_account(self, n_tiles: int | None = None, stream: int | None = None):
        p = self.prog
        runtime.pool_account(self.pool_flag.data_ptr(), self.pool_chunk.data_ptr(),
                             self._run_tiles if n_tiles is None else n_tiles,
                             p.tiles_per_chunk, p.tile_rows,
                             self.pool_keys.data_ptr(), p.pool_kw, self.pool_sizes.data_ptr(),
                             p.pool_ni, self.pool_joined.data_ptr(), self.pool_nodes.data_ptr(),
                             len(p.ref_pool), self.config.lanes_per_group,
                             self.config.pool_bytes, self.pool_rank.data_ptr(),
                             self.pool_gsum.data_ptr(), self.state.data_ptr(),
                             self._stream() if stream is None else stream)

    def grow_arena(self, need: int):
        """Size the device arena for ``need`` bytes per launch (+25 %) and drop the
        run buffers so the next ``reserve`` reallocates them."""
        self._arena_min = max(getattr(self, "_arena_min", 0), int(need * 1.25) + (1 << 20))
        self._arena_key = None

    def _dup_row(self) -> tuple[int, int]:
        """(row, id) of check_unique_ids' failure: the first row, in row order,
        whose id occurred before (some id's second occurrence, minimised over
        ids), ``NONE`` without one; the id as the column's signed Int64 value,
        as the reference's message prints it."""
        out = self.torch.empty(2, dtype=self.torch.int64, device=self.device)
        runtime.dup_resolve(self.idset_w.data_ptr(), self.idset_d.data_ptr(),
                            self._idset_cap + 2, out.data_ptr(), self._stream())
        row, slot = (int(x) for x in out.cpu().numpy().view(np.uint64))
        if row == placement.NONE:
            return row, 0
        # slot cap holds id 0 (the set stores it as 1)
        ident = 0 if slot >= self._idset_cap else int(self.idset[slot].item())
        return row, ident

    def _dup_key(self) -> tuple[int, int]:
        """(error key, id) of check_unique_ids' failure (the merge of the chunk
        holding ``_dup_row``'s row)."""
        row, ident = self._dup_row()
        if row == placement.NONE:
            return row, 0
        return placement.dup_key(row, self.ir.chunk), ident

    def _global_incl(self, t0: int, t1: int) -> np.ndarray:
        """Run-global inclusive instance counts of tiles [t0, t1): the look-back
        status words are launch-local, plus the run total before each launch
        (written by the previous launch's last tile)."""
        words = self.status[t0:t1].cpu().numpy().view(np.uint64)
        incl = ((words >> np.uint64(34)) & np.uint64(0xFFFFFFF)).astype(np.int64)
        lb = self.lbuf.cpu().numpy().view(np.uint64)
        for a, b, k in self._launch_tiles:
            lo, hi = max(a, t0), min(b, t1)
            if lo < hi:
                incl[lo - t0:hi - t0] += np.int64(lb[2 * k])
        return incl

    def _chunk_ends(self, t0: int, t1: int) -> np.ndarray:
        """Run-global inclusive instance counts at the end of every chunk whose
        sub-tiles are [t0, t1) (look-back status words)."""
        spc = self.prog.tiles_per_chunk
        incl = self._global_incl(t0, t1)
        nch = -(-(t1 - t0) // spc)
        return np.array([incl[min((c + 1) * spc, t1 - t0) - 1] for c in range(nch)],
                        dtype=np.int64)

    def _merge_range(self, i0: int, i1: int, s0: int, s1: int, t0: int, t1: int,
                     st: dict, stream=None):
        """batch_size > 1024: the chunks of tiles [t0, t1) hold instances [i0, i1)
        and signs [s0, s1), each chunk emitted as sorted 512-row sub-tiles; re-order
        every chunk's instances by ascending u64 id and rebuild its offsets / slots
        / signs (fbx_merge_subtiles: per-instance rank by binary search in the
        chunk's other sub-tiles, a scan of the new lengths, one scatter)."""
        torch = self.torch
        n, m = i1 - i0, s1 - s0
        if n <= 0:
            return
        incl = self._global_incl(t0, t1)
        starts = np.concatenate([[i0], incl]).astype(np.int64) - i0
        dev = self.device
        d_starts = torch.from_numpy(starts).to(dev, non_blocking=False)
        ids_o = torch.empty(n, dtype=torch.int64, device=dev)
        lab_o = torch.empty(n, dtype=torch.uint8, device=dev)
        off_o = torch.empty(n + 1, dtype=torch.int64, device=dev)
        slot_o = torch.empty(max(m, 1), dtype=torch.int16, device=dev)
        sign_o = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
        scratch = torch.empty(3 * n + 1, dtype=torch.int64, device=dev)
        bad = torch.empty(1, dtype=torch.int32, device=dev)
        s = self._stream() if stream is None else stream
        ins = (self.o_ids[i0:].data_ptr(), self.o_lab[i0:].data_ptr(), self.o_off[i0:].data_ptr(),
               self.o_slot[s0:].data_ptr(), self.o_sign[s0:].data_ptr())
        outs = (ids_o.data_ptr(), lab_o.data_ptr(), off_o.data_ptr(), slot_o.data_ptr(),
                sign_o.data_ptr())
        runtime.merge_subtiles(d_starts.data_ptr(), self.prog.tiles_per_chunk, t1 - t0, n, s0,
                               max(1, len(self.ir.features)), ins, outs, scratch.data_ptr(),
                               bad.data_ptr(), s)
        # a repeated id (the run then fails) can leave the CSR inconsistent: the
        # kernel flags it and writes nothing -- such a CSR is never handed out
        # (the run raises), and _check_merges raises if the run did not fail
        self.o_ids[i0:i1].copy_(ids_o)
        self.o_lab[i0:i1].copy_(lab_o)
        self.o_off[i0:i1 + 1].copy_(off_o)
        if m:
            self.o_slot[s0:s1].copy_(slot_o[:m])
            self.o_sign[s0:s1].copy_(sign_o[:m])
        if not hasattr(self, "_merge_bad"):
            self._merge_bad = []
        self._merge_bad.append((bad, st))

    def _check_merges(self):
        """After a run with chunk merges: an inconsistent CSR is only legal in a
        run that fails (a repeated id)."""
        for bad, st in getattr(self, "_merge_bad", []):
            if int(bad.item()) and not (st["dup_seen"] or st["error_key"] != (1 << 64) - 1):
                raise RuntimeError("inconsistent CSR after a run without failures")
        self._merge_bad = []

    def _resolve_big_label_error(self, st: dict):
        """Place a label failure from the final (merged) order: the kernel marked
        bad labels 0xFE (null) / 0xFF (not 0/1) in the emitted label byte; a
        null anywhere in the first bad label's batch wins (emit_minibatch runs
        before MiniBatch.validate)."""
        if st.get("emit_null_pos", placement.NONE) == placement.NONE and \
                st.get("emit_range_pos", placement.NONE) == placement.NONE:
            return
        n, bs = int(st["instances"]), self.ir.chunk
        bad = self.torch.nonzero(self.o_lab[:n] >= 0xFE)
        if not bad.numel():
            return
        p = int(bad[0, 0].item())
        batch = p // bs
        nulls = self.torch.nonzero(self.o_lab[batch * bs:min(n, (batch + 1) * bs)] == 0xFE)
        lf = (batch, 0, int(nulls[0, 0].item())) if nulls.numel() else (batch, 1, p % bs)
        ends = self._chunk_ends(0, self._run_tiles)
        st["emit_key_resolved"] = (placement.label_key(lf, ends, self._run_chunk0, bs),
                                   st["emit_range_label"] if lf[1] else 0)

    def _merge_big_chunks(self, st: dict):
        self._merge_range(0, int(st["instances"]), 0, int(st["signs"]), 0, self._run_tiles, st)
        self._resolve_big_label_error(st)
        self._check_merges()

    def _label_key(self, st: dict):
        """(error key, label) of the run's first label failure, or None: the
        kernel keeps the first null and the first non-0/1 label by emission
        position; the batch is mapped to the chunk whose merge flushes it
        (look-back status words: inclusive instance counts per chunk)."""
        bs = self.ir.chunk
        lf = placement.label_failure(st.get("emit_null_pos", placement.NONE),
                                     st.get("emit_range_pos", placement.NONE), bs)
        if lf is None:
            return None
        ends = self._global_incl(0, self._run_tiles)
        return (placement.label_key(lf, ends, self._chunk_minus_tile, bs),
                st["emit_range_label"] if lf[1] else 0)

    def begin_run(self, rows_hint: int) -> int:
        """Start a run: clear the run-wide instance-id set (check_unique_ids'
        `seen`), the counters / error word, and -- for a reserved run -- the
        look-back status of every tile.  Returns the number of libfbx kernels
        it launched."""
        torch = self.torch
        nk = 0
        cap = _next_pow2(2 * max(rows_hint, 1))
        if self.idset is None or self._idset_cap < cap:
            # + 2: the id-0 slot; + 1024: the dummy words of rows that do not insert
            self.idset = torch.zeros(cap + 2 + 1024, dtype=torch.int64, device=self.device)
            # winner chunk per slot (no reset: read only for claimed slots) and the
            # later-occurrence chunk pairs (only written when an id repeats)
            self.idset_w = torch.empty(cap + 2, dtype=torch.int64, device=self.device)
            self.idset_d = torch.zeros(2 * (cap + 2), dtype=torch.int64, device=self.device)
            self._idset_cap = cap
        else:
            # one launch: the id set, and the pairs only if the previous run's state
            # (still in place: cleared just below) recorded a repeated id
            runtime.idset_clear(self.idset.data_ptr(), self.idset.numel(),
                                self.idset_d.data_ptr(), self.idset_d.numel(),
                                self.state.data_ptr(), self._stream())
            nk += 1
        if getattr(self, "status", None) is not None:
            # the launch run-total words and every tile's look-back status
            runtime.state_reset(self.state.data_ptr(), self.status_all.data_ptr(),
                                self.status_all.numel(), self._stream())
            nk += 1
        self._launch_k = 0
        self._launch_tiles = []
        self._dup_dirty = False
        self._set("idset", self.idset.data_ptr())
        self._set("idset_mask", self._idset_cap - 1)
        self._set("idset_w", self.idset_w.data_ptr())
        self._set("idset_d", self.idset_d.data_ptr())
        self._run_tiles = 0
        return nk

    def reserve(self, rows: int, launch_rows: int | None = None, ring: bool = False):
        """Run-wide buffers: look-back status for every tile of the run (the
        look-back continues across launches), the CSR for every row, and a
        bump pool sized for the largest launch.  ``ring``: the CSR and the
        reference-arena planes hold ONE launch (each launch writes its CSR at
        the start, offsets launch-local) -- bounded memory for file streams."""
        torch = self.torch
        # no launch of this run covers more than its rows: size the pool for that
        launch_rows = rows if launch_rows is None else max(1, min(launch_rows, rows))
        tiles = self.tiles_for(rows)
        k = max(1, len(self.ir.features))
        self.ring = ring
        crows = launch_rows if ring else rows
        ptiles = self.tiles_for(launch_rows) if ring else tiles
        need = (tiles, rows, k, launch_rows, getattr(self, "_arena_min", 0), ring)
        if getattr(self, "_arena_key", None) != need:
            dev = self.device
            # [run totals before launch k: 2 words per launch (<= one launch per
            #  tile) | look-back status per tile], cleared together by state_reset
            self.status_all = torch.zeros(3 * (tiles + 1), dtype=torch.int64, device=dev)
            self.lbuf = self.status_all[: 2 * (tiles + 1)]
            self.status = self.status_all[2 * (tiles + 1):]
            self.o_ids = torch.empty(crows + 1, dtype=torch.int64, device=dev)
            self.o_lab = torch.empty(crows + 16, dtype=torch.uint8, device=dev)
            self.o_off = torch.empty(crows + 2, dtype=torch.int64, device=dev)
            self.o_slot = torch.empty(crows * k + 8, dtype=torch.int16, device=dev)
            self.o_sign = torch.empty(crows * k + 1, dtype=torch.int64, device=dev)
            pool_cap = 0
            if codegen_pool_sites(self.prog):
                lt = self.tiles_for(launch_rows)  # grants round up per tile and site
                pool_cap = (self.pool_bytes_per_row * launch_rows
                            + lt * self.prog.pool_slack_per_tile + (1 << 20))
                pool_cap = max(pool_cap, getattr(self, "_arena_min", 0))
            self.pool = torch.empty(pool_cap + 256, dtype=torch.uint8, device=dev)
            self.pool_cap = pool_cap
            if self.prog.ref_pool:  # rows of flagged tiles for fbx_pool_account
                p = self.prog
                plane = ptiles * p.tile_rows
                self.pool_flag = torch.zeros(ptiles + 1, dtype=torch.uint8, device=dev)
                self.pool_chunk = torch.zeros(ptiles + 1, dtype=torch.int64, device=dev)
                self.pool_keys = torch.zeros(max(1, p.pool_kw) * plane + 1, dtype=torch.int64,
                                             device=dev)
                self.pool_sizes = torch.zeros(p.pool_ni * plane + 1, dtype=torch.int32, device=dev)
                self.pool_joined = torch.zeros(plane + 1, dtype=torch.uint8, device=dev)
                self.pool_rank = torch.zeros(plane + 1, dtype=torch.int32, device=dev)
                self.pool_gsum = torch.zeros(plane + 1, dtype=torch.int64, device=dev)
                # the node table is per plan: built once (a pageable H2D would
                # synchronise the host with every queued upload and index build)
                nodes = self.prepared.__dict__.setdefault("_pool_nodes", {})
                if dev not in nodes:
                    nodes[dev] = torch.tensor([[l, r, i, 0] for l, r, i in p.ref_pool],
                                              dtype=torch.int32, device=dev)
                self.pool_nodes = nodes[dev]
                self._set("pool_flag", self.pool_flag.data_ptr())
                self._set("pool_chunk", self.pool_chunk.data_ptr())
                self._set("pool_keys", self.pool_keys.data_ptr())
                self._set("pool_sizes", self.pool_sizes.data_ptr())
                self._set("pool_joined", self.pool_joined.data_ptr())
                self._set("pool_plane", plane)
            self._arena_key = need
        self._set("tile_status", self.status.data_ptr())
        self._set("out.ids", self.o_ids.data_ptr())
        self._set("out.labels", self.o_lab.data_ptr())
        self._set("out.offsets", self.o_off.data_ptr())
        self._set("out.slots", self.o_slot.data_ptr())
        self._set("out.signs", self.o_sign.data_ptr())
        self._set("pool", self.pool.data_ptr())
        self._set("pool_cap", self.pool_cap)
        return tiles

    def _arena(self, rows: int):
        self.reserve(rows)
        return self.tiles_for(rows)

    def tiles_for(self, rows: int) -> int:
        """Look-back tiles of `rows` driver rows (chunks x sub-tiles per chunk)."""
        return -(-rows // self.ir.chunk) * self.prog.tiles_per_chunk

    def tile_of_row(self, row: int) -> int:
        """Run-global tile id of the chunk that starts at driver row `row`."""
        return (row // self.ir.chunk) * self.prog.tiles_per_chunk

    def bind_driver(self, dview: DeviceView):
        for c in dview.tensors:
            for part in ("nulls", "data", "offsets"):
                self._set(f"drv.{c}.{part}", dview.ptr(c, part))
        self.dview = dview

    def launch(self, row_lo: int, row_hi: int, stream: int | None = None,
               tile_base: int | None = None) -> int:
        """Enqueue one fused launch over driver rows [row_lo, row_hi) (no sync).

        ``row_lo`` must be a multiple of ``batch_size`` (chunk boundaries are
        the reference's read boundaries, pipeline.py:994).  Without
        ``tile_base`` the launch is a run of its own (status + CSR from 0);
        with it the launch continues a reserved run: its tiles are
        ``tile_base + i`` of the run-wide look-back and its CSR lands at the
        run-global positions."""
        if row_lo % self.ir.chunk:
            raise ValueError("row_lo must start a driver chunk")
        rows = row_hi - row_lo
        stream = self._stream() if stream is None else stream
        if rows > self.LAUNCH_ROWS_MAX:
            raise ValueError(f"a launch covers at most {self.LAUNCH_ROWS_MAX} rows "
                             "(28-bit look-back counts)")
        if tile_base is None:
            tiles = self._arena(rows)
            runtime.state_reset(self.state.data_ptr(), self.status_all.data_ptr(),
                                2 * (self.status.numel()) + tiles + 1, stream)
            tile_base = 0
            self._launch_k = 0
            self._launch_tiles = []
        else:
            # continuation of a reserved run: counters / digest / error word keep
            # accumulating across launches; only the bump pool is reset
            tiles = self.tiles_for(rows)
            if tile_base > 0:  # the run's first launch follows begin_run's full reset
                runtime.pool_reset(self.state.data_ptr(), stream)
        self._set("row_lo", row_lo)
        self._set("row_hi", row_hi)
        self._set("chunk0", row_lo // self.ir.chunk)
        self._set("tile_base", tile_base)
        k = self._launch_k
        lb = self.lbuf.data_ptr()
        self._set("launch_base", lb + 16 * k)
        self._set("launch_next", lb + 16 * (k + 1))
        self._set("csr_ring", 1 if self.ring else 0)
        self._set("pool_tile0", tile_base if self.ring else 0)
        self._launch_tiles.append((tile_base, tile_base + tiles, k))
        self._last_launch_tiles = tiles
        self._launch_k = k + 1
        self._chunk_minus_tile = row_lo // self.ir.chunk - tile_base
        self._run_chunk0 = row_lo // self.ir.chunk - tile_base // self.prog.tiles_per_chunk
        self._run_tiles = tile_base + tiles
        _nvtx_push(f"fbx_pipeline rows {row_lo}-{row_hi} tiles {tile_base}+{tiles}")
        try:
            self.module.launch("fbx_pipeline", tiles, self.prog.threads, self.prog.smem_bytes,
                               stream, self.params)
        finally:
            _nvtx_pop()
        return tiles

    def finish(self) -> CsrBatch:
        """Synchronise, read counters, raise the first error in pipeline order."""
        st = self._read_state()
        if self.prog.tiles_per_chunk > 1:
            self._merge_big_chunks(st)
        self.check_run(st)
        c = Counters(st["digest"], st["instances"], st["signs"], st["malformed"],
                     st["filtered"], st["joined"], 1)
        return CsrBatch(self.o_ids, self.o_lab, self.o_off, self.o_slot, self.o_sign, c)

    def run(self, row_lo: int, row_hi: int) -> CsrBatch:
        self.launch(row_lo, row_hi)
        return self.finish()

    def capture_run(self, n_rows: int):
        """A whole device-resident run -- the run-state reset, the id-set clear
        and every launch over rows [0, n_rows) of the bound driver -- captured
        into one CUDA graph (the serving loop replays it; the stage chain of
        run_pipelined, pipeline.py:901-1094, becomes one graph launch).
        Replay with ``g.replay()``, then ``finish()``."""
        torch = self.torch
        self.reserve(n_rows, self.max_rows)
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            self.begin_run(n_rows)
            for lo in range(0, n_rows, self.max_rows):
                self.launch(lo, min(lo + self.max_rows, n_rows),
                            stream=side.cuda_stream, tile_base=self.tile_of_row(lo))
        torch.cuda.current_stream(self.device).wait_stream(side)
        return g


class StreamedRun:
    """End-to-end run from pinned host column images (the e2e path).

    The driver is cut into slices of whole chunks.  Slice k's column spans
    are copied H2D on a copy stream into one of two device buffer sets, the
    fused kernel runs on the compute stream, and the emitted CSR range of
    slice k-1 is copied D2H on a second copy stream -- so PCIe traffic in both
    directions overlaps the kernels.  The look-back continues across the
    launches (run-global tile ids), so the CSR is written at its final
    positions and slices need no host-side fix-up.
    """

    PARTS = ("nulls", "data", "offsets")

    def __init__(self, eng: "Engine", host_view: ViewImage, slice_rows: int = 1 << 17,
                 zero_copy: bool = False, taper: bool = True, sink: str = "host"):
        torch = eng.torch
        self.eng, self.torch = eng, torch
        chunk = eng.ir.chunk
        self.slice_rows = max(chunk, slice_rows - slice_rows % chunk)
        self.n = n = host_view.row_count
        # taper: short first and last slices, so the D2H stream (the bound) starts
        # early and the tail after the last kernel is short (for a run on its own;
        # back-to-back runs overlap their fill and drain instead)
        div = 4 if taper else 1
        S = self.slice_rows
        q = max(chunk, (S // div) // chunk * chunk) if div > 1 else S
        cuts = [0]
        if n > q:
            cuts.append(q)
        while n - cuts[-1] > S + q:
            cuts.append(cuts[-1] + S)
        r = n - cuts[-1]
        if div > 1 and r > 2 * q:
            cuts.append(cuts[-1] + (r - q) // chunk * chunk)
        if cuts[-1] < n:
            cuts.append(n)
        self.bounds = [(a, b) for a, b in zip(cuts, cuts[1:])]
        used = [c for c in host_view.order if any(f"drv.{c}.{p}" in eng.slots for p in self.PARTS)]
        # Each slice's column spans packed into ONE pinned region (16-B aligned
        # pieces) -- the layout a chunk reader produces -- so a slice is one H2D.
        self.packs, self.layout = [], []
        self.h2d_bytes = 0
        cols = {c: host_view.columns[c] for c in used}
        for lo, hi in self.bounds:
            pieces, off = [], 0
            for c, col in cols.items():
                sp = {"nulls": (lo // 8, (hi + 7) // 8)}
                if col.kind.var_length:
                    sp["data"] = (int(col.offsets[lo]) & ~15, (int(col.offsets[hi]) + 15) & ~15)
                    sp["offsets"] = (lo * 4, (hi + 1) * 4)
                else:
                    w = col.kind.fixed_width
                    sp["data"] = (lo * w, hi * w)
                for p, (a, b) in sp.items():
                    pieces.append((c, p, a, b, off))
                    off += (b - a + 15) & ~15
            buf = np.zeros(off + 16, dtype=np.uint8)
            for c, p, a, b, o in pieces:
                src = getattr(cols[c], p)
                raw = np.ascontiguousarray(src).view(np.uint8).reshape(-1)
                seg = raw[a:b]
                buf[o:o + seg.size] = seg
            self.packs.append(torch.from_numpy(buf).pin_memory())
            self.layout.append(pieces)
            self.h2d_bytes += off
        cap = max(p.numel() for p in self.packs)
        # three input buffer sets: the H2D of slice k+1 waits only for kernel k-2
        self.dev = [torch.empty(cap + 32, dtype=torch.uint8, device=eng.device) for _ in range(3)]
        self.s_h2d = torch.cuda.Stream(eng.device)
        self.s_comp = torch.cuda.Stream(eng.device)
        self.s_d2h = torch.cuda.Stream(eng.device)
        k = max(1, len(eng.ir.features))
        self.out = {"ids": torch.empty(n + 1, dtype=torch.int64, pin_memory=True),
                    "labels": torch.empty(n + 16, dtype=torch.uint8, pin_memory=True),
                    "offsets": torch.empty(n + 2, dtype=torch.int64, pin_memory=True),
                    "slots": torch.empty(n * k + 8, dtype=torch.int16, pin_memory=True),
                    "signs": torch.empty(n * k + 1, dtype=torch.int64, pin_memory=True)}
        self.states = torch.empty((len(self.bounds), runtime.STATE_BYTES // 8),
                                  dtype=torch.int64, pin_memory=True)
        # zero-copy: the fused kernels write the CSR straight into these pinned
        # (UVA-mapped) host buffers over PCIe -- no D2H copies, no per-slice sync.
        # Correct, but measured slower than DMA copies on B200/PCIe5 (246 vs 278
        # M rec/s, round 1), so off by default.
        self.zero_copy = zero_copy
        self.trace = None  # set to [] to record a per-slice event timeline (ms)
        # sink "device": the CSR stays in HBM (the engine's torch tensors, for a GPU
        # trainer -- the paper's FeatureBox hand-off); only the per-slice run-state
        # snapshots (mapped pinned memory) come back to the host
        if sink not in ("host", "device"):
            raise ValueError("sink must be 'host' or 'device'")
        self.sink = sink
        if zero_copy and eng.prog.tiles_per_chunk > 1:
            raise UnsupportedOnDevice("zero-copy streamed runs need batch_size <= 1024 (larger "
                                      "chunks are merged on the device before their D2H)")

    def run(self) -> Counters:
        while True:
            try:
                if self.zero_copy:
                    return self._run_zero_copy()
                self.start()
                tot = self.finish()
                self.wait()
                return tot
            except ArenaRetry as exc:  # the device arena was too small: grow, repeat
                self.wait()
                self.eng.grow_arena(exc.need)

    def start(self):
        """Enqueue every slice's H2D and fused kernel (no host synchronisation).

        A StreamedRun may be restarted while the previous run's CSR is still
        draining: the new kernels wait (on the device) for that D2H.  The host
        output buffers of a run stay valid until the next ``start``."""
        torch, eng = self.torch, self.eng
        eng.reserve(self.n, self.slice_rows)
        eng.begin_run(self.n)
        cur = torch.cuda.current_stream(eng.device)
        self.s_comp.wait_stream(cur)
        self.s_h2d.wait_stream(cur)
        if getattr(self, "_last_d2h", None) is not None:
            self.s_comp.wait_event(self._last_d2h)   # the CSR arena is still draining
        self.comp_done = comp_done = [torch.cuda.Event() for _ in self.bounds]
        h2d_done = [torch.cuda.Event() for _ in self.bounds]
        self._trace = trace = [] if self.trace is not None else None
        tiles_before = 0
        self._slice_tiles = []

        def mark(name, k, stream):
            if trace is not None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(stream)
                trace.append((name, k, ev, time.perf_counter()))
        self._mark = mark
        nb = len(self.dev)
        # buffer reuse is ordered by events on the copy stream; the host drains
        # slice by slice in finish(): slice j's D2H is enqueued as soon as its
        # kernel's state snapshot lands in mapped memory.
        for k, (lo, hi) in enumerate(self.bounds):
            buf = k % nb
            with torch.cuda.stream(self.s_h2d):
                if k >= nb:
                    self.s_h2d.wait_event(comp_done[k - nb])  # buffer set reuse
                pk = self.packs[k]
                mark("h2d0", k, self.s_h2d)
                self.dev[buf][: pk.numel()].copy_(pk, non_blocking=True)
                h2d_done[k].record(self.s_h2d)
                mark("h2d1", k, self.s_h2d)
            base = self.dev[buf].data_ptr()
            for c, p, a, b, o in self.layout[k]:
                eng._set(f"drv.{c}.{p}", base + o - a)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(h2d_done[k])
                mark("k0", k, self.s_comp)
                eng.launch(lo, hi, self.s_comp.cuda_stream, tile_base=tiles_before)
                runtime.state_snapshot(eng.state.data_ptr(), self.states[k].data_ptr(),
                                       self.s_comp.cuda_stream)
                comp_done[k].record(self.s_comp)
                mark("k1", k, self.s_comp)
            self._slice_tiles.append((tiles_before, tiles_before + eng.tiles_for(hi - lo)))
            tiles_before += eng.tiles_for(hi - lo)

    def finish(self) -> Counters:
        """Drain the run started by ``start``: per slice, wait for its kernel,
        then enqueue the D2H of its CSR range; check the run's failures."""
        torch, eng = self.torch, self.eng
        comp_done, mark, trace = self.comp_done, self._mark, self._trace
        tot = Counters()
        inst_base, sign_base = 0, 0
        last = None
        for j in range(len(self.bounds)):
            comp_done[j].synchronize()
            st = self.states[j].numpy().view(np.uint64)
            stt = {f: int(st[i]) for i, f in enumerate(runtime.STATE_FIELDS)}
            # failures are resolved once at the end of the run: a label error's
            # flush chunk and a repeated id's second chunk may lie in later slices.
            # Counters accumulate over the run's launches: this slice's share.
            ni, ms = stt["instances"] - inst_base, stt["signs"] - sign_base
            merged = None
            if eng.prog.tiles_per_chunk > 1:  # batch_size > 1024: merge this slice's chunks
                t0, t1 = self._slice_tiles[j]
                with torch.cuda.stream(self.s_comp):
                    eng._merge_range(inst_base, inst_base + ni, sign_base, sign_base + ms,
                                     t0, t1, stt)
                    merged = torch.cuda.Event()
                    merged.record(self.s_comp)
            if self.sink == "device":
                inst_base += ni
                sign_base += ms
                last = stt
                continue
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(merged if merged is not None else comp_done[j])
                mark("d2h0", j, self.s_d2h)
                o = self.out
                a, b = inst_base, inst_base + ni
                o["ids"][a:b].copy_(eng.o_ids[a:b], non_blocking=True)
                o["labels"][a:b].copy_(eng.o_lab[a:b], non_blocking=True)
                o["offsets"][a:b + 1].copy_(eng.o_off[a:b + 1], non_blocking=True)
                o["slots"][sign_base:sign_base + ms].copy_(eng.o_slot[sign_base:sign_base + ms],
                                                           non_blocking=True)
                o["signs"][sign_base:sign_base + ms].copy_(eng.o_sign[sign_base:sign_base + ms],
                                                           non_blocking=True)
                mark("d2h1", j, self.s_d2h)
            inst_base += ni
            sign_base += ms
            last = stt
        tot.digest = last["digest"]
        tot.instances, tot.signs = last["instances"], last["signs"]
        tot.malformed, tot.filtered = last["malformed"], last["filtered"]
        tot.joined = last["joined"]
        tot.launches = len(self.bounds)
        ev = torch.cuda.Event()
        ev.record(self.s_d2h if self.sink == "host" else self.s_comp)
        self._last_d2h = ev
        # the last snapshot is the run's final state (no extra D2H read)
        if eng.prog.tiles_per_chunk > 1:
            self.s_comp.synchronize()
            eng._resolve_big_label_error(last)
            eng._check_merges()
        eng.check_run(last)
        self.d2h_bytes = (tot.instances * 17 + 8 + tot.signs * 10 if self.sink == "host"
                          else runtime.STATE_BYTES * len(self.bounds))
        if trace:
            t0e, t0h = trace[0][2], trace[0][3]
            self.trace = [(nm, k, t0e.elapsed_time(ev), (th - t0h) * 1e3) for nm, k, ev, th in trace]
        return tot

    def wait(self):
        """Block until the last finished run's CSR is in host memory."""
        if getattr(self, "_last_d2h", None) is not None:
            self._last_d2h.synchronize()

    def _run_zero_copy(self) -> Counters:
        torch, eng = self.torch, self.eng
        eng.reserve(self.n, self.slice_rows)
        o = self.out
        for name, t in (("out.ids", o["ids"]), ("out.labels", o["labels"]),
                        ("out.offsets", o["offsets"]), ("out.slots", o["slots"]),
                        ("out.signs", o["signs"])):
            eng._set(name, t.data_ptr())
        cur = torch.cuda.current_stream(eng.device)
        self.s_comp.wait_stream(cur)
        self.s_h2d.wait_stream(cur)
        with torch.cuda.stream(self.s_comp):
            eng.begin_run(self.n)
        comp_done = [torch.cuda.Event() for _ in self.bounds]
        h2d_done = [torch.cuda.Event() for _ in self.bounds]
        tiles_before = 0
        for k, (lo, hi) in enumerate(self.bounds):
            buf = k & 1
            with torch.cuda.stream(self.s_h2d):
                if k >= 2:
                    self.s_h2d.wait_event(comp_done[k - 2])  # buffer set reuse
                pk = self.packs[k]
                self.dev[buf][: pk.numel()].copy_(pk, non_blocking=True)
                h2d_done[k].record(self.s_h2d)
            base = self.dev[buf].data_ptr()
            for c, p, a, b, off in self.layout[k]:
                eng._set(f"drv.{c}.{p}", base + off - a)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(h2d_done[k])
                eng.launch(lo, hi, self.s_comp.cuda_stream, tile_base=tiles_before)
                comp_done[k].record(self.s_comp)
            tiles_before += eng.tiles_for(hi - lo)
        self.s_comp.synchronize()
        st = eng._read_state()
        eng.check_run(st)
        # restore the device CSR for later device-resident launches
        eng._arena_key = None
        tot = Counters(st["digest"], st["instances"], st["signs"], st["malformed"],
                       st["filtered"], st["joined"], len(self.bounds))
        self.d2h_bytes = tot.instances * 17 + 8 + tot.signs * 10
        return tot

    def csr(self, c: Counters) -> dict[str, np.ndarray]:
        n, m = c.instances, c.signs
        o = self.out
        return {"ids": o["ids"][:n].numpy().view(np.uint64),
                "labels": o["labels"][:n].numpy(),
                "offsets": o["offsets"][:n + 1].numpy().view(np.uint64),
                "slots": o["slots"][:m].numpy().view(np.uint16),
                "signs": o["signs"][:m].numpy().view(np.uint64)}


class ArenaRetry(Exception):
    """The engine's own device arena was too small for a run (``need`` bytes per
    launch): not a reference failure -- the caller grows the arena and repeats
    the run (``Engine.grow_arena``)."""

    def __init__(self, need: int):
        super().__init__(f"device arena needs {need} bytes")
        self.need = need


def codegen_pool_sites(prog: codegen.Program) -> bool:
    return "fbx::pool_alloc<NT>" in prog.source.split("// ===== generated plan =====", 1)[-1]


def _cause(code: str, detail: int, st: dict) -> BaseException:
    if code == "type":
        return TypeError("unsupported operand type for mix/fold")
    if code == "encode":
        return UnicodeEncodeError("utf-8", "", 0, 1, "surrogates not allowed")
    if code == "pool":  # fbx_pool_account: (requested << 32) | remaining
        return PoolExhausted(detail >> 32, detail & 0xFFFFFFFF)
    if code == "pool_key":
        return UnsupportedOnDevice("reference arena accounting over Utf8 join keys")
    if code == "null_label":
        return EmitError("null label at emission")
    if code == "label_range":
        return BatchInvariantError(f"label {detail - (1 << 64) if detail >> 63 else detail!r} not 0/1")
    if code == "basic_dup":  # detail: the repeated Int64 id (two's complement)
        sid = detail - (1 << 64) if detail >> 63 else detail
        return MergeUniquenessError(f"basic features: duplicate instance id {sid}")
    if code == "dup_id":
        return MergeUniquenessError(f"extracted features: duplicate instance id {detail}")
    if code == "multi_match":
        return MergeUniquenessError("extracted features: duplicate instance id (side view "
                                    "key matched more than one row)")
    if code == "json_bigint":
        return ValueError("Exceeds the limit (4300 digits) for integer string conversion")
    if code == "float_overflow":
        return OverflowError("float too large to pack with f format")
    if code in ("json_deep", "unicode_lower", "float_slow"):
        return UnsupportedOnDevice(f"row needs an unimplemented device path: {code}")
    return ValueError(f"value error ({code})")


# ---------------------------------------------------------------------------
# run reports (pipeline.py:461-540)
# ---------------------------------------------------------------------------

@dataclass
class RunReport:
    mode: str
    digest: int
    batches: int
    instances: int
    signs: int
    launches: int
    overhead_us: float
    bytes_h2d: int
    transfer_seconds: float
    intermediate_bytes_written: int
    intermediate_files: tuple[str, ...]
    rows_dropped: int
    rows_filtered: int
    batch_size: int
    workers: int
    wall_seconds: float
    stage_seconds: dict[str, float] = field(default_factory=dict)

    def to_text(self) -> str:
        lines = [
            f"== run report ({self.mode}) ==",
            f"batches emitted: {self.batches} x batch_size {self.batch_size}",
            f"instances: {self.instances} ({self.rows_dropped} dropped malformed, "
            f"{self.rows_filtered} filtered)",
            f"feature signs: {self.signs}",
            f"device launches: {self.launches} (measured overhead {self.overhead_us:.3f} us)",
            f"h2d transfers: {self.bytes_h2d} bytes ({self.transfer_seconds:.9f} s measured)",
            f"intermediate bytes written: {self.intermediate_bytes_written}",
        ]
        for stage in sorted(self.stage_seconds):
            lines.append(f"stage {stage}: {self.stage_seconds[stage]:.3f} s")
        lines.append(f"wall: {self.wall_seconds:.3f} s on {self.workers} worker(s)")
        lines.append(f"batch digest: 0x{self.digest:016x}")
        lines += ["", "[report]"]
        kv = {"mode": self.mode, "digest": f"0x{self.digest:016x}", "batches": self.batches,
              "instances": self.instances, "signs": self.signs, "launches": self.launches,
              "overhead_us": f"{self.overhead_us:.3f}", "bytes_h2d": self.bytes_h2d,
              "transfer_seconds": f"{self.transfer_seconds:.9f}",
              "intermediate_bytes": self.intermediate_bytes_written,
              "rows_dropped": self.rows_dropped, "rows_filtered": self.rows_filtered,
              "batch_size": self.batch_size, "workers": self.workers,
              "wall_seconds": f"{self.wall_seconds:.3f}"}
        for stage in sorted(self.stage_seconds):
            kv[f"stage_{stage}_s"] = f"{self.stage_seconds[stage]:.3f}"
        lines.extend(f"{k}={v}" for k, v in kv.items())
        return "\n".join(lines)


def parse_report_block(text: str) -> dict[str, str]:
    out, seen = {}, False
    for line in text.splitlines():
        if line.strip() == "[report]":
            seen = True
            continue
        if seen and "=" in line:
            k, _, v = line.partition("=")
            out[k.strip()] = v.strip()
    return out


@dataclass
class RunResult:
    report: RunReport
    csr: dict[str, np.ndarray] | None


def run_views(config: PipelineConfig, views: Mapping[str, ViewImage], basic: ViewImage,
              collect: bool = False, device: str = "cuda", prepared: Prepared | None = None,
              max_rows_per_launch: int = 1 << 22) -> RunResult:
    """The pipelined run over in-memory views (H2D once, device-resident)."""
    t0 = time.perf_counter()
    stage: dict[str, float] = {}
    prep = prepared or prepare(config, views, basic)
    workers = run_workers(config)  # the reference's ExecContext checks (pipeline.py:697-711)
    stage["prepare"] = time.perf_counter() - t0
    eng = Engine(prep, views, basic, device=device, max_rows_per_launch=max_rows_per_launch)
    torch = eng.torch
    drv = views[config.driver].project(config.view(config.driver).columns)
    t1 = time.perf_counter()
    dv = DeviceView(drv, device=eng.device)
    torch.cuda.synchronize(eng.device)
    stage["read"] = time.perf_counter() - t1
    eng.bind_driver(dv)
    n = drv.row_count
    # one reserved run: the look-back, the CSR positions and the id set span
    # every launch, so emission order and error placement are run-global
    step = eng.max_rows
    t2 = time.perf_counter()
    while True:
        eng.reserve(n, min(step, max(n, 1)))
        eng.begin_run(n)
        tiles = 0
        launches = 0
        for lo in range(0, n, step):
            hi = min(lo + step, n)
            tiles += eng.launch(lo, hi, tile_base=tiles)
            launches += 1
        try:
            b = eng.finish()
            break
        except ArenaRetry as exc:  # the device arena was too small: grow, repeat the run
            eng.grow_arena(exc.need)
    total = b.counters
    total.launches = launches
    stage["extract"] = time.perf_counter() - t2
    _fused_stages(stage)
    csr = b.to_numpy() if collect else None
    bs = config.batch_size
    rep = RunReport(
        mode="pipelined", digest=total.digest, batches=math.ceil(total.instances / bs),
        instances=total.instances, signs=total.signs, launches=total.launches + len(eng.ir.sides)
        + 1, overhead_us=0.0, bytes_h2d=dv.bytes, transfer_seconds=stage["read"],
        intermediate_bytes_written=0, intermediate_files=(),
        rows_dropped=total.malformed + eng.prepare_counters.malformed,
        rows_filtered=total.filtered + eng.prepare_counters.filtered,
        batch_size=bs, workers=workers, wall_seconds=time.perf_counter() - t0,
        stage_seconds=stage)
    return RunResult(rep, csr)


_PREPARED: dict[str, Prepared] = {}


def _config_key(config: PipelineConfig) -> str:
    """What the generated plan depends on: every config field, with each
    dictionary table reduced to (default, size, entry count) -- its contents
    only reach the device tables, which the engine builds from the config of
    the call -- and the input files' schemas (an edited file re-plans)."""
    import dataclasses
    import hashlib
    parts = []
    for f in dataclasses.fields(config):
        v = getattr(config, f.name)
        if f.name == "tables":
            v = sorted((n, t.default, t.size_bytes, len(t.entries)) for n, t in v.items())
        elif f.name == "views":  # file paths do not shape the plan; schemas do (below)
            v = [(x.name, x.columns, x.policy) for x in v]
        elif f.name in ("basic_path", "staging_dir"):
            continue
        parts.append((f.name, repr(v)))
    for v in config.views:
        parts.append(repr(open_view(v.path).schema))
    parts.append(repr(open_view(config.basic_path).schema))
    return hashlib.sha256(repr(parts).encode()).hexdigest()


def _fused_stages(stage: dict) -> None:
    """The reference's pipelined stage keys (pipeline.py:984-1094: prepare, read,
    clean, join, extract, merge, emit).  Clean, join, merge and emit run inside the
    fused kernel, so their time is in "extract"; their keys read 0.0."""
    for k in ("prepare", "read", "clean", "join", "extract", "merge", "emit"):
        stage.setdefault(k, 0.0)


def _prepared(config: PipelineConfig) -> Prepared:
    """prepare() once per plan key (_config_key): the plan cache.  The returned
    Prepared carries the CALL's config (its dictionary tables)."""
    import dataclasses
    try:
        key = _config_key(config)
    except Exception:  # noqa: BLE001 -- an unreadable file: prepare raises the reference's error
        return prepare(config)
    prep = _PREPARED.get(key)
    if prep is None:
        prep = prepare(config)
        _PREPARED.clear()  # one plan at a time (the engines hold its module)
        _PREPARED[key] = prep
    if prep.config is not config:
        mods = prep.__dict__.get("_modules")
        prep = dataclasses.replace(prep, config=config)
        if mods is not None:
            prep.__dict__["_modules"] = mods
    return prep


def run_pipelined(config: PipelineConfig, collect: bool = False,
                  slice_rows: int = 1 << 19) -> RunReport:
    """Reference-compatible ``run_pipelined`` (pipeline.py:952-1114) on the B200.

    prepare (plan cached per config + schemas) -> side views and basic features
    read by the host reader into HBM, CRC-checked on the device, indexed by
    the prep kernels (pipeline.py:970-980) -> the driver streamed from its file
    in slices of whole chunks (stream.FileRun: parallel pread into a pinned
    ring, H2D on a copy stream, the fused kernel on a compute stream, CSR in a
    one-slice ring; bounded host and device memory) -> the run's counters and
    digest, failures raised in the reference's pipeline order.  ``collect``:
    the device-resident run over in-memory views (the whole CSR returned in
    ``run_views``' result; tests)."""
    if collect:
        views = {}
        for v in config.views:
            try:
                views[v.name] = read_view(v.path, v.columns)
            except Exception as exc:  # noqa: BLE001
                raise StageError("prepare", None, exc) from exc
        try:
            basic = read_view(config.basic_path, config.basic_columns)
        except Exception as exc:  # noqa: BLE001
            raise StageError("prepare", None, exc) from exc
        return run_views(config, views, basic, collect=collect).report
    return _stream_pipelined(config, slice_rows).report()


@dataclass
class _StreamedRun:
    """A run_pipelined over a driver file (or a record shard of it), its
    failures not yet raised (sharded.py folds them across ranks)."""
    config: PipelineConfig
    engine: "Engine"
    state: dict
    counters: Counters
    launches: int
    launch_s: float
    bytes_h2d: int
    transfer_s: float
    stage: dict
    t0: float
    read_failure: "StageError | None" = None
    workers: int = 1

    def first_failure(self) -> tuple[int, int]:
        """(error key, detail) of the run's first failure; a read failure is
        key (chunk, "read") with detail -1."""
        key, detail = placement.NONE, 0
        if self.state is not None:
            key, detail = self.engine.first_failure(self.state)
        if self.read_failure is not None:
            rk = placement.key_of(self.read_failure.batch_index, "read", 0)
            if rk < key:
                key, detail = rk, -1
        return key, detail

    def report(self) -> RunReport:
        """Raise the run's first failure (single run), else its RunReport."""
        key, detail = self.first_failure()
        if self.read_failure is not None and key == placement.key_of(
                self.read_failure.batch_index, "read", 0):
            raise self.read_failure
        self.engine.raise_key(key, detail, self.state)
        return self.to_report()

    def to_report(self, counters: Counters | None = None, launches: int | None = None,
                  bytes_h2d: int | None = None) -> RunReport:
        c = counters or self.counters
        bs = self.config.batch_size
        n_launch = self.launches if launches is None else launches
        pc = self.engine.prepare_counters
        return RunReport(
            mode="pipelined", digest=c.digest, batches=math.ceil(c.instances / bs),
            instances=c.instances, signs=c.signs, launches=n_launch,
            overhead_us=1e6 * self.launch_s / max(1, n_launch),
            bytes_h2d=self.bytes_h2d if bytes_h2d is None else bytes_h2d,
            transfer_seconds=self.transfer_s, intermediate_bytes_written=0,
            intermediate_files=(), rows_dropped=c.malformed + pc.malformed,
            rows_filtered=c.filtered + pc.filtered, batch_size=bs, workers=self.workers,
            wall_seconds=time.perf_counter() - self.t0, stage_seconds=self.stage)


def driver_streams(config: PipelineConfig) -> bool:
    """Whether run_pipelined streams the driver file in slices: chunks of at
    most one CTA (batch_size <= 1024) and more than one chunk -- else (one
    chunk: the reference reads, and CRC-checks, the whole body) the run is
    device-resident."""
    prep = _prepared(config)
    drv_cfg = config.view(config.driver)
    try:
        dfile = open_view(drv_cfg.path)
    except Exception as exc:  # noqa: BLE001
        raise StageError("prepare", None, exc) from exc
    names = [c for c, _ in dfile.schema]
    full_read = drv_cfg.columns is None or set(drv_cfg.columns) >= set(names)
    return not (prep.program.tiles_per_chunk > 1 or
                (full_read and dfile.row_count <= config.batch_size))


def _stream_pipelined(config: PipelineConfig, slice_rows: int = 1 << 19,
                      rows: tuple[int, int] | None = None) -> _StreamedRun:
    """run_pipelined's body: prepare, then stream the driver (or its record
    shard ``rows``, whole chunks) through the engine; failures of the prepare
    stage raise here, the run's own are left in the result's state."""
    from .stream import FileRun, _ReadFailure
    t0 = time.perf_counter()
    stage: dict[str, float] = {}
    prep = _prepared(config)
    workers = run_workers(config)  # the reference's ExecContext (pipeline.py:697-701)
    drv_cfg = config.view(config.driver)
    torch = _torch()
    try:
        dfile = open_view(drv_cfg.path)
    except Exception as exc:  # noqa: BLE001
        raise StageError("prepare", None, exc) from exc
    n = dfile.row_count
    bs = config.batch_size
    names = [c for c, _ in dfile.schema]
    full_read = drv_cfg.columns is None or set(drv_cfg.columns) >= set(names)
    streamed = not (prep.program.tiles_per_chunk > 1 or (full_read and n <= bs))
    if rows is not None and not streamed:
        raise ValueError("a record shard streams its rows: batch_size <= 1024, more than one chunk")
    fr = None
    if streamed:
        # the driver's first slices are read while the side views are prepared
        # (measured: faster than reading the side / basic files first)
        fr = FileRun(prep, drv_cfg.path, drv_cfg.columns, slice_rows=slice_rows, rows=rows)
        fr.start()
    try:
        dvs = {v.name: DeviceView.from_file(v.path, v.columns, defer_crc=streamed)
               for v in config.views if v.name != config.driver}
        dvs["basic"] = DeviceView.from_file(config.basic_path, config.basic_columns,
                                            defer_crc=streamed)
    except Exception as exc:  # noqa: BLE001
        if fr is not None:
            fr.stop()
        raise StageError("prepare", None, exc) from exc

    def settle_prepare():
        """Deferred prepare checks, in the reference's order: each side view's
        and the basic view's body CRC, then the index builds' failures."""
        try:
            for dv in dvs.values():
                dv.verify_crc()
        except Exception as exc:  # noqa: BLE001
            raise StageError("prepare", None, exc) from exc
        eng.finish_prepare()
    bytes_h2d = sum(d.h2d_bytes for d in dvs.values())
    try:
        eng = Engine(prep, device_views=dvs, defer_prepare_check=streamed)
    except BaseException:
        if fr is not None:
            fr.stop()
        raise
    launches = 1 + len(eng._side_views)  # the prepare-time state reset + index builds
    stage["prepare"] = time.perf_counter() - t0
    t1 = time.perf_counter()
    launch_s = 0.0
    if not streamed:
        # one chunk reads the whole body (the reference then checks its CRC), or
        # chunks larger than a CTA (merged on the device): device-resident run
        try:
            dv = DeviceView.from_file(drv_cfg.path, drv_cfg.columns)
        except Exception as exc:  # noqa: BLE001
            raise StageError("read", 0, exc) from exc
        bytes_h2d += dv.h2d_bytes
        stage["read"] = time.perf_counter() - t1
        eng.bind_driver(dv)
        t2 = time.perf_counter()
        step = eng.max_rows
        while True:
            eng.reserve(n, min(step, max(n, 1)))
            launches += eng.begin_run(n)
            tiles = 0
            for lo in range(0, n, step):
                tiles += eng.launch(lo, min(lo + step, n), tile_base=tiles)
                launches += 1
            try:
                b = eng.finish()
                break
            except ArenaRetry as exc:
                eng.grow_arena(exc.need)
        launch_s = time.perf_counter() - t2
        stage["extract"] = time.perf_counter() - t2
        transfer_s = stage["read"]
        c = b.counters
        st = None  # finish() raised the run's failures
        read_failure = None
    else:
        while True:
            if fr is None:  # a repeat after the device arena grew
                fr = FileRun(prep, drv_cfg.path, drv_cfg.columns, slice_rows=slice_rows,
                             rows=rows)
            eng.reserve(fr.n, fr.slice_rows, ring=True)
            launches += eng.begin_run(fr.n)
            read_failure = None
            try:
                t = fr.run(eng)
            except _ReadFailure as exc:
                settle_prepare()
                read_failure = StageError("read", fr.bounds[exc.index][0] // bs, exc.cause)
                read_failure.__cause__ = exc.cause
                t = exc.timings
            launches += t["launches"]
            launch_s += t["launch_s"]
            if read_failure is None:
                settle_prepare()
            try:
                st = eng.settle_run(eng._read_state())
                break
            except ArenaRetry as exc:
                eng.grow_arena(exc.need)
                fr = None
        stage["read"] = t["read_s"]
        stage["transfer"] = t["h2d_s"]
        stage["extract"] = t["kernel_s"]
        transfer_s = t["h2d_s"]
        bytes_h2d += t["h2d_bytes"]
        c = Counters(st["digest"], st["instances"], st["signs"], st["malformed"],
                     st["filtered"], st["joined"], t["slices"])
    stage["stream"] = time.perf_counter() - t1
    _fused_stages(stage)
    return _StreamedRun(config, eng, st, c, launches, launch_s, bytes_h2d, transfer_s, stage, t0,
                        read_failure, workers)


def run_pipeline(config: PipelineConfig, mode: str | None = None) -> RunReport:
    """Dispatch to the configured (or overridden) mode (pipeline.py:1117-1124)."""
    effective = mode or config.mode
    if effective == "staged":
        from .staged import run_staged
        return run_staged(config)
    if effective == "pipelined":
        return run_pipelined(config)
    raise ConfigError(f"unknown mode {effective!r}")


# ---------------------------------------------------------------------------
# _extract_batch drop-in (pipeline.py:718-737): row-aligned output columns
# ---------------------------------------------------------------------------

def prepare_extract(config: PipelineConfig, table_kinds: Mapping[str, Kind]) -> Prepared:
    """Plan the operator DAG over an already cleaned + joined table."""
    kinds = dict(table_kinds)
    try:
        dag = expand_call_graph(config.operators)
        plan = place_operators(layer_schedule(dag), PlacementBudget(config.device_budget_bytes),
                               dag)
        fns = {}
        for name, node in dag.nodes.items():
            fn = resolve_function(node.func.spec, config.tables)
            want = "tuple" if node.role == "body" else "scalar"
            if fn.arity != want:
                raise FeatureConfigError(f"{name}: function {node.func.spec!r} has arity "
                                         f"{fn.arity}, {node.role} node needs {want}")
            fns[name] = fn
    except (FeatureConfigError, ValueError) as exc:
        if isinstance(exc, ConfigError):
            raise
        raise ConfigError(str(exc)) from exc
    missing = set(dag.external_inputs()) - set(kinds)
    if missing:
        raise ConfigError(f"operator inputs {sorted(missing)} not present in the table")
    extract_outputs = []
    for spec in config.operators:
        domains = output_domains(spec, config.tables)
        for col in spec.outputs:
            if col in kinds:
                raise ConfigError(f"output column {col!r} collides with a table column")
            extract_outputs.append((col, Kind.INT64 if domains[col] == "u64" else Kind.UTF8,
                                    domains[col]))
    refplace = reference_placement(dag, config.device_budget_bytes)
    order = reference_node_order(plan, refplace)
    rank = {n: i for i, (_, n) in enumerate(order)}
    specs = {s.name: s for s in config.operators}
    pre_of: dict[str, dict[int, str]] = {}
    nodes = []
    for layer, name in order:
        nd = dag.nodes[name]
        if nd.role == "pre":
            pre_of.setdefault(nd.op, {})[nd.slot] = name
            inputs = nd.reads
        elif nd.role == "body":
            inputs = specs[nd.op].inputs
        else:
            inputs = ()
        ref_pool = (fns[name].op == "token" and nd.role != "body"
                    and refplace[name] == DEVICE)
        nodes.append(codegen.NodeIR(name, nd.role, nd.op, fns[name], layer, rank[name],
                                    tuple(inputs), nd.slot, nd.writes, ref_pool))
    ir = codegen.PlanIR(
        driver=codegen.ViewIR("table", kinds, {}, [], None), sides=[], basic=None,
        join_keys=(), nodes=nodes, pre_of=pre_of, producer=dict(dag.col_producer),
        features={}, instance_column=config.instance_column, label_column=config.label_column,
        chunk=256, tables={t: i for i, t in enumerate(sorted(config.tables))},
        table_defaults={t: config.tables[t].default for t in config.tables},
        extract_outputs=[(c, d) for c, _, d in extract_outputs], stage_strings=False,
        mode="extract", pool_bytes=config.pool_bytes, lanes_per_group=config.lanes_per_group)
    prog = codegen.generate(ir)
    return Prepared(config, dag, plan, ir, prog, runtime.compile_source(prog.source),
                    tuple(extract_outputs), [n for _, n in order], {"table": kinds}, {})


class ExtractEngine:
    """``_extract_batch`` on the device through the C-ABI engine object
    (``fbx_create`` / ``fbx_extract`` / ``fbx_output_*``, include/fbx.h): staging,
    launch, the reference arena, error decoding and string compaction all happen
    in libfbx.so; see capi.CEngine."""

    def __init__(self, prepared: Prepared, device: str = "cuda"):
        torch = _torch()
        dev = torch.device(device)
        idx = dev.index if dev.index is not None else torch.cuda.current_device()
        from .capi import CEngine
        self.c = CEngine(prepared, idx)
        self.prepared = prepared

    def extract(self, table: ViewImage) -> ViewImage:
        return self.c.extract(table)


def prepare_clean_ir(config: PipelineConfig, view_cfg, kinds: Mapping[str, Kind]) -> codegen.PlanIR:
    """The plan of one view's ``clean_views`` kernel (staged mode, codegen mode
    "clean"): the view's fills, JSON extractions and bound filter."""
    pol = view_cfg.policy
    try:
        validate_clean_policy(dict(kinds), pol)
    except (CleanConfigError, KeyError) as exc:
        raise ConfigError(f"view {view_cfg.name!r}: {exc}") from exc
    cleaned = cleaned_kinds(dict(kinds), pol)
    flt = bind_filter(pol.filter, cleaned) if pol.filter is not None else None
    drv = codegen.ViewIR(view_cfg.name, dict(kinds), dict(pol.fills), list(pol.extractions), flt,
                         ())
    return codegen.PlanIR(
        driver=drv, sides=[], basic=None, join_keys=(), nodes=[], pre_of={}, producer={},
        features={}, instance_column=config.instance_column, label_column=config.label_column,
        chunk=256, tables={}, table_defaults={}, extract_outputs=[], stage_strings=False,
        mode="clean", pool_bytes=config.pool_bytes, lanes_per_group=config.lanes_per_group)


def extract_batch(table: ViewImage, config: PipelineConfig, device: str = "cuda") -> ViewImage:
    """One-call ``_extract_batch`` equivalent (plans, compiles, runs)."""
    kinds = {c: table.columns[c].kind for c in table.order}
    return ExtractEngine(prepare_extract(config, kinds), device=device).extract(table)
