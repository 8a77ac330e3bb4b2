"""Staged mode on the B200: ``run_staged`` (pipeline.py:783-895).

The reference runs every stage to completion over whole tables and writes each
boundary to an FBXC file in ``staging_dir``:

  clean    cleaned_<view>.fbxc   clean_views of every view (viewpipe.py:334-431)
  join     joined.fbxc           join_views of the cleaned driver with each side
                                 (inner; rows in (key image, left, right) order)
  extract  extracted.fbxc        _extract_batch over the joined table
  merge    merged.fbxc           check_unique_ids on both sides, then join_views
                                 with the basic features on the instance id
  emit                           emit_minibatch over batch_size slices -> digest

Every stage's table work runs on the device: the clean stage is a generated
kernel per view (codegen mode "clean": the fused kernel's own clean_view code,
row-aligned outputs) compacted by ``fbx_select_rows`` / ``fbx_take``; joins sort
the right side's key images (``fbx_sort_keys``, CUB radix sort) and match by
binary search (``fbx_join_count`` / ``fbx_join_fill``); the uniqueness checks
are ``fbx_first_repeat`` over sorted ids; extraction is the C-ABI engine object
(``fbx_extract``) and the emission its ``fbx_emit_csr``.  The host moves bytes
(file reads, H2D, D2H, the FBXC writes) -- the materialisation the mode exists
for.  Join keys: one Int64 or Float32 column (Utf8 / multi-column keys raise
UnsupportedOnDevice at the join stage).
"""

from __future__ import annotations

import math
import time
from pathlib import Path

import numpy as np

from . import codegen, runtime
from .columns import ColumnImage, Kind, ViewImage, read_view, write_view
from .config import (ConfigError, EmitError, MergeUniquenessError, PipelineConfig, StageError,
                     UnsupportedOnDevice)


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 staged mode needs a CUDA device (no CPU execution path)")
    return torch


class DTable:
    """A table resident in HBM, row-aligned: per column a null byte per row and
    the value (Int64 bits / Float32 bits) or the string's (pointer, length)."""

    def __init__(self, n: int, order: list[str], kinds: dict[str, Kind], keys=()):
        self.n, self.order, self.kinds, self.keys = n, order, kinds, tuple(keys)
        self.cols: dict[str, dict] = {}
        self.keep: list = []

    # -- host image <-> device ------------------------------------------------
    @classmethod
    def upload(cls, view: ViewImage, stream: int) -> "DTable":
        torch = _torch()
        t = cls(view.row_count, list(view.order), {c: view.columns[c].kind for c in view.order},
                view.key_columns)
        n = t.n
        for c in view.order:
            img = view.columns[c]
            col = {"null": torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")}
            bm = torch.from_numpy(np.array(img.nulls, np.uint8)).cuda() if n else None
            if n:
                runtime.call("fbx_unpack_nulls", bm.data_ptr(), n, col["null"].data_ptr(), stream)
            if img.kind.var_length:
                data = torch.from_numpy(np.concatenate([np.asarray(img.data, np.uint8),
                                                        np.zeros(16, np.uint8)])).cuda()
                offs = torch.from_numpy(np.array(img.offsets, np.uint32).view(np.int32)).cuda()
                col["ptr"] = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
                col["len"] = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
                runtime.call("fbx_spans", offs.data_ptr(), data.data_ptr(), n,
                             col["ptr"].data_ptr(), col["len"].data_ptr(), stream)
                t.keep += [data, offs]
            else:
                dt = np.int64 if img.kind is Kind.INT64 else np.int32
                col["val"] = torch.from_numpy(np.asarray(img.data).view(dt).copy()).cuda()
            t.keep.append(bm)
            t.cols[c] = col
        return t

    def download(self, stream: int) -> ViewImage:
        """The FBXC image of the table (null bitmaps packed, strings gathered on
        the device, then one D2H per segment)."""
        torch = _torch()
        n = self.n
        cols = {}
        for c in self.order:
            kind, col = self.kinds[c], self.cols[c]
            bm = torch.zeros((n + 7) // 8 + 1, dtype=torch.uint8, device="cuda")
            if n:
                runtime.call("fbx_pack_nulls", col["null"].data_ptr(), 0, n, bm.data_ptr(), stream)
            nulls = bm[: (n + 7) // 8].cpu().numpy()
            if kind.var_length:
                offs = torch.empty(n + 1, dtype=torch.int64, device="cuda")
                runtime.exclusive_scan_u32(col["len"].data_ptr(), offs.data_ptr(), n, stream)
                o = offs.cpu().numpy().view(np.uint64)
                total = int(o[-1])
                if total > 0xFFFFFFFF:
                    raise ConfigError(f"column {c!r}: payload exceeds the u32 offset range")
                out = torch.empty(max(total, 1), dtype=torch.uint8, device="cuda")
                if n:
                    runtime.gather_strings(col["ptr"].data_ptr(), col["len"].data_ptr(),
                                           offs.data_ptr(), n, out.data_ptr(), stream)
                data = out[:total].cpu().numpy()
                cols[c] = ColumnImage(kind, n, nulls, data, o.astype(np.uint32))
            else:
                v = col["val"][:n].cpu().numpy()
                data = v if kind is Kind.INT64 else v.view(np.float32)
                cols[c] = ColumnImage(kind, n, nulls, np.ascontiguousarray(data))
        return ViewImage(cols, tuple(self.keys), tuple(self.order))

    def take(self, rows, m: int, stream: int, names=None) -> "DTable":
        """Rows ``rows[:m]`` (a device int32 tensor) of the named columns."""
        torch = _torch()
        names = list(self.order) if names is None else list(names)
        out = DTable(m, names, {c: self.kinds[c] for c in names}, ())
        for c in names:
            src, col = self.cols[c], {}
            for part, (dt, w) in {"null": (torch.uint8, 1), "val": (None, 0), "ptr": (torch.int64, 8),
                                  "len": (torch.int32, 4)}.items():
                if part not in src:
                    continue
                if part == "val":
                    dt = src["val"].dtype
                    w = src["val"].element_size()
                col[part] = torch.empty(max(m, 1), dtype=dt, device="cuda")
                if m:
                    runtime.call("fbx_take", src[part].data_ptr(), w, rows.data_ptr(), m,
                                 col[part].data_ptr(), stream)
            out.cols[c] = col
        out.keep = list(self.keep)  # string pointers reference the source buffers
        return out


def _key(t: DTable, keys, where: str):
    if len(keys) != 1:
        raise UnsupportedOnDevice(f"{where}: staged joins on the device take one key column")
    k = keys[0]
    kind = t.kinds[k]
    if kind not in (Kind.INT64, Kind.FLOAT32):
        raise UnsupportedOnDevice(f"{where}: staged join on a {kind.name} key")
    torch = _torch()
    v = t.cols[k]["val"]
    if kind is Kind.FLOAT32:  # the IEEE bits, zero-extended: big-endian byte order
        v = (v.to(torch.int64) & 0xFFFFFFFF)
    return v, t.cols[k]["null"]


def _sorted_keys(t: DTable, keys, stream: int, where: str):
    torch = _torch()
    key, nul = _key(t, keys, where)
    n = max(t.n, 1)
    skey = torch.empty(n, dtype=torch.int64, device="cuda")
    srow = torch.empty(n, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    rs = torch.empty(n, dtype=torch.int32, device="cuda")
    ks = torch.empty(n, dtype=torch.int64, device="cuda")
    fs = torch.empty(n, dtype=torch.uint8, device="cuda")
    runtime.call("fbx_sort_keys", key.data_ptr(), nul.data_ptr(), t.n, skey.data_ptr(),
                 srow.data_ptr(), cnt.data_ptr(), rs.data_ptr(), ks.data_ptr(), fs.data_ptr(),
                 stream)
    return skey, srow, int(cnt.item())


def join_tables(left: DTable, right: DTable, keys, stream: int, where: str) -> DTable:
    """join_views (viewpipe.py:550-559): inner equi-join, the left columns then
    the right non-key columns, rows in (key image, left row, right row) order."""
    torch = _torch()
    for k in keys:
        if k not in left.kinds or k not in right.kinds:
            raise StageError(where, None, ConfigError(f"join key {k!r} missing from an input"))
        if left.kinds[k] is not right.kinds[k]:
            raise StageError(where, None, ConfigError(
                f"join key {k!r}: kind {left.kinds[k].name} vs {right.kinds[k].name}"))
    rcols = [c for c in right.order if c not in keys]
    clash = set(rcols) & set(left.order)
    if clash:
        raise StageError(where, None, ConfigError(
            f"join would duplicate columns {sorted(clash)}; rename before joining"))
    skey, srow, nr = _sorted_keys(right, keys, stream, where)
    lkey, lnul = _key(left, keys, where)
    nl = left.n
    first = torch.empty(max(nl, 1), dtype=torch.int64, device="cuda")
    cnt = torch.empty(max(nl, 1), dtype=torch.int32, device="cuda")
    runtime.call("fbx_join_count", lkey.data_ptr(), lnul.data_ptr(), nl, skey.data_ptr(), nr,
                 first.data_ptr(), cnt.data_ptr(), stream)
    off = torch.empty(nl + 1, dtype=torch.int64, device="cuda")
    runtime.exclusive_scan_u32(cnt.data_ptr(), off.data_ptr(), nl, stream)
    m = int(off[nl].item())
    lrows = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
    rrows = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
    runtime.call("fbx_join_fill", lkey.data_ptr(), nl, first.data_ptr(), cnt.data_ptr(),
                 off.data_ptr(), srow.data_ptr(), m, lrows.data_ptr(), rrows.data_ptr(), stream)
    out = left.take(lrows, m, stream)
    r = right.take(rrows, m, stream, rcols)
    for c in rcols:
        out.order.append(c)
        out.kinds[c] = right.kinds[c]
        out.cols[c] = r.cols[c]
    out.keep += r.keep
    out.keys = tuple(keys)
    return out


def first_repeat(t: DTable, column: str, side: str, stream: int):
    """check_unique_ids (viewpipe.py:562-576) on the device: raises the
    reference's MergeUniquenessError at the first row, in row order, whose id
    occurred before."""
    torch = _torch()
    if column not in t.kinds:
        raise ConfigError(f"{side}: missing id column {column!r}")
    skey, srow, nv = _sorted_keys(t, (column,), stream, "merge")
    best = torch.empty(1, dtype=torch.int64, device="cuda")
    runtime.call("fbx_first_repeat", skey.data_ptr(), srow.data_ptr(), nv, best.data_ptr(), stream)
    row = int(best.cpu().numpy().view(np.uint64)[0])
    if row != (1 << 64) - 1:
        v = int(t.cols[column]["val"][row].item())
        if t.kinds[column] is Kind.FLOAT32:
            v = float(np.int32(v).view(np.float32))
        raise MergeUniquenessError(f"{side}: duplicate instance id {v}")


class _CleanKernel:
    """The generated clean_views kernel of one view (codegen mode "clean")."""

    def __init__(self, config: PipelineConfig, view_cfg, kinds: dict[str, Kind]):
        from .engine import prepare_clean_ir
        self.ir = prepare_clean_ir(config, view_cfg, kinds)
        self.prog = codegen.generate(self.ir)
        self.mod = runtime.Program(runtime.compile_source(self.prog.source))
        self.ckinds = self.ir.driver.cleaned_kinds()

    def run(self, t: DTable, state, stream: int) -> tuple[DTable, object]:
        torch = _torch()
        n = t.n
        params = np.zeros(runtime.FBX_MAX_PARAM_SLOTS, dtype=np.uint64)
        slots = self.prog.slots

        def put(name, value):
            if name in slots:
                params[slots[name]] = np.uint64(int(value) & ((1 << 64) - 1))
        put("state", state.data_ptr())
        put("side0.rows", n)
        keep = torch.zeros(max(n, 1), dtype=torch.uint8, device="cuda")
        put("clean.keep", keep.data_ptr())
        # the input view as FBXC segments on the device (the side loader reads them)
        src = {}
        for c in t.order:
            col = t.cols[c]
            bm = torch.zeros((n + 7) // 8 + 16, dtype=torch.uint8, device="cuda")
            if n:
                runtime.call("fbx_pack_nulls", col["null"].data_ptr(), 0, n, bm.data_ptr(), stream)
            put(f"side0.{c}.nulls", bm.data_ptr())
            src[c] = [bm]
            if "val" in col:
                put(f"side0.{c}.data", col["val"].data_ptr())
        # strings: the loader reads offsets + bytes; rebuild a packed image
        for c in t.order:
            if "ptr" in t.cols[c]:
                offs = torch.empty(n + 2, dtype=torch.int64, device="cuda")
                runtime.exclusive_scan_u32(t.cols[c]["len"].data_ptr(), offs.data_ptr(), n, stream)
                total = int(offs[n].item()) if n else 0
                data = torch.zeros(total + 32, dtype=torch.uint8, device="cuda")
                if n:
                    runtime.gather_strings(t.cols[c]["ptr"].data_ptr(), t.cols[c]["len"].data_ptr(),
                                           offs.data_ptr(), n, data.data_ptr(), stream)
                o32 = offs[: n + 1].to(torch.int32)
                put(f"side0.{c}.offsets", o32.data_ptr())
                put(f"side0.{c}.data", data.data_ptr())
                src[c] += [offs, data, o32]
        out = DTable(n, list(self.ckinds), dict(self.ckinds), t.keys)
        pool_cap = 0
        for c, kind in self.ckinds.items():
            col = {"null": torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")}
            put(f"clean.{c}.null", col["null"].data_ptr())
            if kind.var_length:
                col["ptr"] = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
                col["len"] = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
                put(f"clean.{c}.ptr", col["ptr"].data_ptr())
                put(f"clean.{c}.len", col["len"].data_ptr())
            else:
                col["val"] = torch.empty(max(n, 1), dtype=torch.int64 if kind is Kind.INT64
                                         else torch.int32, device="cuda")
                put(f"clean.{c}.val", col["val"].data_ptr())
            out.cols[c] = col
        for e in self.ir.driver.extractions:  # unescaped / canonical JSON strings
            src_bytes = int(src[e.source][2].numel()) if len(src.get(e.source, [])) > 2 else 0
            grow = 6 if e.kind is Kind.JSON else 1  # ensure_ascii: 1 byte -> "\\uXXXX"
            pool_cap += grow * src_bytes + 128 * (n // 256 + 1)
        pool = torch.zeros(pool_cap + 256, dtype=torch.uint8, device="cuda")
        put("side_pool", pool.data_ptr())
        put("side_pool_cap", pool_cap)
        grid = max(1, min((n + 255) // 256, 1184))
        self.mod.launch("fbx_clean_rows", grid, 256, 0, stream, params)
        out.keep = [src, pool] + list(t.keep)
        return out, keep


def _stage_error(st: dict, stage: str) -> BaseException | None:
    from .engine import ERR_NAMES, _cause
    key = st["error_key"]
    if key == (1 << 64) - 1:
        return None
    code = ERR_NAMES.get(key & 0xFF, "value")
    return StageError(stage, None, _cause(code, st["error_detail"], st))


def run_staged(config: PipelineConfig):
    """Reference-compatible ``run_staged`` (pipeline.py:783-895) on the B200."""
    from .engine import ExtractEngine, RunReport, prepare, prepare_extract
    torch = _torch()
    prepare(config, compile_program=False)  # the reference's validation (ConfigError)
    if config.staging_dir is None:
        raise ConfigError("staged mode requires staging_dir")
    from .config import run_workers
    workers = run_workers(config)  # the reference's ExecContext (pipeline.py:697-701)
    staging = Path(config.staging_dir)
    staging.mkdir(parents=True, exist_ok=True)
    stream = torch.cuda.current_stream().cuda_stream
    stage_seconds: dict[str, float] = {}
    files: list[Path] = []
    counters = {"malformed": 0, "filtered": 0}
    io = {"h2d": 0, "launches": 0, "transfer": 0.0}
    wall0 = time.perf_counter()
    state = torch.zeros(runtime.STATE_BYTES // 8, dtype=torch.int64, device="cuda")

    def timed(stage: str, fn):
        t0 = time.perf_counter()
        try:
            return fn()
        except (ConfigError, StageError):
            raise
        except Exception as exc:  # noqa: BLE001 -- the reference's timed() wrapper
            raise StageError(stage, None, exc) from exc
        finally:
            stage_seconds[stage] = stage_seconds.get(stage, 0.0) + time.perf_counter() - t0

    def read_state() -> dict:
        raw = state.cpu().numpy().view(np.uint64)
        return {f: int(raw[i]) for i, f in enumerate(runtime.STATE_FIELDS)}

    def upload(view: ViewImage) -> DTable:
        t0 = time.perf_counter()
        t = DTable.upload(view, stream)
        torch.cuda.synchronize()
        io["transfer"] += time.perf_counter() - t0
        io["h2d"] += sum(view.columns[c].nbytes() for c in view.order)
        return t

    def write(t: DTable | ViewImage, name: str) -> Path:
        img = t.download(stream) if isinstance(t, DTable) else t
        dest = staging / name
        write_view(img, dest)
        files.append(dest)
        return dest

    sides = [v for v in config.views if v.name != config.driver]

    def stage_clean() -> dict:
        out = {}
        for view in config.views:
            img = read_view(view.path, view.columns)
            t = upload(img)
            runtime.state_reset(state.data_ptr(), state.data_ptr(), 0, stream)
            kern = _CleanKernel(config, view, {c: img.columns[c].kind for c in img.order})
            ct, keep = kern.run(t, state, stream)
            io["launches"] += 2
            st = read_state()
            err = _stage_error(st, "clean")
            if err is not None:
                raise err
            counters["malformed"] += st["malformed"]
            counters["filtered"] += st["filtered"]
            rows = torch.empty(max(t.n, 1), dtype=torch.int32, device="cuda")
            cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
            runtime.call("fbx_select_rows", keep.data_ptr(), t.n, rows.data_ptr(), cnt.data_ptr(),
                         stream)
            m = int(cnt.item())
            kept = ct.take(rows, m, stream)
            kept.keys = t.keys
            write(kept, f"cleaned_{view.name}.fbxc")
            out[view.name] = kept
        return out

    cleaned = timed("clean", stage_clean)

    def stage_join() -> DTable:
        acc = cleaned[config.driver]
        for side in sides:
            acc = join_tables(acc, cleaned[side.name], tuple(config.join_keys), stream, "join")
        write(acc, "joined.fbxc")
        return acc

    table = timed("join", stage_join) if sides else cleaned[config.driver]

    def stage_extract() -> ViewImage:
        img = table.download(stream)
        kinds = {c: img.columns[c].kind for c in img.order}
        eng = ExtractEngine(prepare_extract(config, kinds))
        extracted = eng.extract(img)
        io["launches"] += 1
        io["h2d"] += sum(img.columns[c].nbytes() for c in img.order)
        write(extracted, "extracted.fbxc")
        return extracted, eng

    extracted, eng = timed("extract", stage_extract)

    def stage_merge() -> DTable:
        ex = upload(extracted)
        basic = upload(read_view(config.basic_path, config.basic_columns))
        first_repeat(ex, config.instance_column, "extracted features", stream)
        first_repeat(basic, config.instance_column, "basic features", stream)
        merged = join_tables(ex, basic, (config.instance_column,), stream, "merge")
        write(merged, "merged.fbxc")
        return merged

    merged = timed("merge", stage_merge)

    def stage_emit() -> dict:
        img = merged.download(stream)
        feats = [(img.columns[c], slot) for c, slot in config.features.items()]
        for c, what in ((config.label_column, "label"), (config.instance_column, "instance")):
            if c not in img.columns:
                raise EmitError(f"{what} column {c!r} missing")
        for c in config.features:
            if c not in img.columns:
                raise EmitError(f"feature column {c!r} missing")
        io["launches"] += 2
        return eng.c.emit_csr(img.columns[config.instance_column],
                              img.columns[config.label_column], feats)

    out = timed("emit", stage_emit)
    n = int(merged.n)
    intermediate = sum(f.stat().st_size for f in files)
    return RunReport(
        mode="staged", digest=int(out["digest"]), batches=math.ceil(n / config.batch_size),
        instances=n, signs=int(len(out["signs"])), launches=io["launches"], overhead_us=0.0,
        bytes_h2d=io["h2d"], transfer_seconds=io["transfer"],
        intermediate_bytes_written=intermediate,
        intermediate_files=tuple(sorted(f.name for f in files)),
        rows_dropped=counters["malformed"], rows_filtered=counters["filtered"],
        batch_size=config.batch_size, workers=workers, wall_seconds=time.perf_counter() - wall0,
        stage_seconds=stage_seconds)


__all__ = ["run_staged", "DTable", "join_tables", "first_repeat"]
