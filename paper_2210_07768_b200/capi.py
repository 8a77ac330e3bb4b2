"""ctypes binding of libfbx.so's engine object (include/fbx.h, "The engine object").

This is the reference-facing boundary of SURVEY.md §8(b): ``fbx_create`` binds a
compiled plan once (NodeEvaluator.__init__, device.py:263-293), ``fbx_extract``
is ``pipeline._extract_batch`` (pipeline.py:718-737), ``fbx_emit_csr`` is
``emit_minibatch`` + ``MiniBatch.validate`` + the batch digest (pipeline.py:
357-433) and ``fbx_last_error`` locates a failure like ``LayerExecutionError``
(device.py:34-41).  Everything below the C-ABI (staging, launches, the arena,
error decoding, string compaction) is C++/CUDA; this module only marshals
FBXC column images and maps a status back to the reference's exception.
"""

from __future__ import annotations

import ctypes
from typing import Mapping, Sequence

import numpy as np

from . import runtime
from .columns import ColumnImage, Kind, ViewImage
from .config import (BatchInvariantError, EmitError, LayerExecutionError, PoolExhausted,
                     UnsupportedOnDevice)

c_u, c_ull, c_int, vp = ctypes.c_uint, ctypes.c_ulonglong, ctypes.c_int, ctypes.c_void_p

S_OK, S_CONFIG, S_POOL, S_TYPE, S_VALUE, S_ENCODE, S_CUDA, S_OVERFLOW, S_UNSUPPORTED, \
    S_EMIT, S_INVARIANT, S_INTERNAL = range(12)


class Column(ctypes.Structure):
    _fields_ = [("kind", c_u), ("nulls", vp), ("data", vp), ("offsets", vp),
                ("data_bytes", c_ull)]


class PoolNode(ctypes.Structure):
    _fields_ = [("layer", c_u), ("rank", c_u), ("input", c_u), ("pad", c_u)]


class Plan(ctypes.Structure):
    _fields_ = [("cubin", vp), ("cubin_bytes", ctypes.c_size_t), ("kernel", ctypes.c_char_p),
                ("slot_state", c_int), ("slot_rows", c_int), ("slot_pool", c_int),
                ("slot_pool_cap", c_int), ("slot_pool_sizes", c_int),
                ("n_inputs", c_u), ("input_kinds", vp), ("input_slots", vp),
                ("n_outputs", c_u), ("output_kinds", vp), ("output_slots", vp),
                ("n_tables", c_u), ("table_slots", vp),
                ("n_pool_nodes", c_u), ("pool_nodes", vp), ("pool_planes", c_u),
                ("pool_bytes", c_ull), ("lanes_per_group", c_ull),
                ("n_nodes", c_u), ("node_names", vp), ("arena_bytes_per_row", c_ull)]


class Table(ctypes.Structure):
    _fields_ = [("keys", vp), ("key_offsets", vp), ("values", vp), ("n", c_ull)]


class Counters(ctypes.Structure):
    _fields_ = [("launches", c_ull), ("rows", c_ull), ("bytes_h2d", c_ull),
                ("device_ms", ctypes.c_double)]


class Csr(ctypes.Structure):
    _fields_ = [("ids", vp), ("labels", vp), ("offsets", vp), ("slots", vp), ("signs", vp),
                ("capacity", c_ull), ("n_signs", c_ull), ("digest", c_ull)]


def _bind():
    L = runtime.lib()
    if getattr(L, "_fbx_engine_bound", False):
        return L
    L.fbx_create.argtypes = [ctypes.POINTER(Plan), ctypes.POINTER(Table), c_int,
                             ctypes.POINTER(vp)]
    L.fbx_destroy.argtypes = [vp]
    L.fbx_extract.argtypes = [vp, ctypes.POINTER(Column), c_u, c_ull,
                              ctypes.POINTER(Counters), vp]
    L.fbx_output_info.argtypes = [vp, c_u, ctypes.POINTER(c_u), ctypes.POINTER(c_ull),
                                  ctypes.POINTER(c_ull)]
    L.fbx_output_copy.argtypes = [vp, c_u, vp, vp, vp, vp]
    L.fbx_emit_csr.argtypes = [vp, ctypes.POINTER(Column), ctypes.POINTER(Column),
                               ctypes.POINTER(Column), vp, c_u, c_ull, ctypes.POINTER(Csr), vp]
    L.fbx_last_error.argtypes = [vp, ctypes.POINTER(c_int), ctypes.POINTER(ctypes.c_char_p),
                                 ctypes.POINTER(c_ull)]
    L.fbx_error_message.argtypes = [vp]
    L.fbx_error_message.restype = ctypes.c_char_p
    for name in ("fbx_create", "fbx_destroy", "fbx_extract", "fbx_output_info",
                 "fbx_output_copy", "fbx_emit_csr", "fbx_last_error"):
        getattr(L, name).restype = c_int
    L._fbx_engine_bound = True
    return L


def column_struct(img: ColumnImage, keep: list) -> Column:
    """An FBXC image as an fbx_column (host pointers; the arrays stay in `keep`)."""
    nulls = np.ascontiguousarray(img.nulls)
    data = np.ascontiguousarray(img.data)
    keep += [nulls, data]
    c = Column(int(img.kind), nulls.ctypes.data, data.ctypes.data, None, 0)
    if img.kind.var_length:
        offs = np.ascontiguousarray(img.offsets, dtype=np.uint32)
        base = int(offs[0]) if img.n else 0
        if base:  # a slice of a bigger image: re-base its offsets
            offs = (offs - np.uint32(base)).astype(np.uint32)
            data = np.ascontiguousarray(img.data[base:base + int(offs[-1])])
            keep.append(data)
            c.data = data.ctypes.data
        keep.append(offs)
        c.offsets = offs.ctypes.data
        c.data_bytes = int(offs[-1]) if img.n else 0
    return c


def _slot(slots: Mapping[str, int], name: str) -> int:
    return slots.get(name, -1)


class CEngine:
    """One fbx_engine for an extraction plan (``engine.prepare_extract``)."""

    def __init__(self, prepared, device: int = 0):
        self.L = L = _bind()
        self.prepared = prepared
        prog, ir, cfg = prepared.program, prepared.ir, prepared.config
        s = prog.slots
        self.inputs = list(ir.driver.kinds)
        self.outputs = list(prepared.extract_outputs)
        keep: list = []
        in_kinds = np.array([int(ir.driver.kinds[c]) for c in self.inputs] or [0], np.uint32)
        in_slots = np.array([[_slot(s, f"drv.{c}.{p}") for p in ("nulls", "data", "offsets")]
                             for c in self.inputs] or [[-1] * 3], np.int32)
        out_kinds = np.array([int(k) for _, k, _ in self.outputs] or [0], np.uint32)
        out_slots = np.array([[_slot(s, f"out{j}.{p}") for p in ("nulls", "data", "ptr", "len")]
                              for j in range(len(self.outputs))] or [[-1] * 4], np.int32)
        tnames = sorted(ir.tables, key=ir.tables.get)
        t_slots = np.array([[_slot(s, f"dict{ir.tables[t]}.{p}") for p in ("slots", "mask", "keys")]
                            for t in tnames] or [[-1] * 3], np.int32)
        tables = (Table * max(1, len(tnames)))()
        for i, t in enumerate(tnames):
            blob, offs, vals = cfg.tables[t].arrays()
            blob = np.ascontiguousarray(blob) if blob.size else np.zeros(1, np.uint8)
            keep += [blob, offs, vals]
            tables[i] = Table(blob.ctypes.data, offs.ctypes.data, vals.ctypes.data, len(vals))
        pnodes = (PoolNode * max(1, len(prog.ref_pool)))(
            *[PoolNode(lay, rank, inp, 0) for lay, rank, inp in prog.ref_pool])
        names = [n.encode() for n in prepared.node_names]
        c_names = (ctypes.c_char_p * max(1, len(names)))(*names)
        cubin = ctypes.create_string_buffer(prepared.cubin, len(prepared.cubin))
        keep += [in_kinds, in_slots, out_kinds, out_slots, t_slots, tables, pnodes, c_names, cubin]
        plan = Plan(ctypes.cast(cubin, vp), len(prepared.cubin), b"fbx_extract_rows",
                    _slot(s, "state"), _slot(s, "rows"), _slot(s, "pool"), _slot(s, "pool_cap"),
                    _slot(s, "pool_sizes"), len(self.inputs), in_kinds.ctypes.data,
                    in_slots.ctypes.data, len(self.outputs), out_kinds.ctypes.data,
                    out_slots.ctypes.data, len(tnames), t_slots.ctypes.data,
                    len(prog.ref_pool), ctypes.addressof(pnodes), prog.pool_ni,
                    cfg.pool_bytes, cfg.lanes_per_group, len(names),
                    ctypes.addressof(c_names), 64 + (512 if prog.json_kind else 0))
        h = vp()
        rc = L.fbx_create(ctypes.byref(plan), tables, int(device), ctypes.byref(h))
        if rc:
            raise runtime.FbxError(f"fbx_create: {L.fbx_error_message(None).decode()}")
        self.h = h
        self.counters = Counters()

    def close(self):
        if getattr(self, "h", None):
            self.L.fbx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    # -- errors ------------------------------------------------------------------
    def error(self, status: int) -> BaseException:
        """The reference exception for a failed call (LayerExecutionError around
        an operator's cause)."""
        layer, node, detail = c_int(), ctypes.c_char_p(), c_ull()
        self.L.fbx_last_error(self.h, ctypes.byref(layer), ctypes.byref(node),
                              ctypes.byref(detail))
        msg = self.L.fbx_error_message(self.h).decode(errors="replace")
        d = detail.value
        cause: BaseException
        if status == S_POOL:
            cause = PoolExhausted(d >> 32, d & 0xFFFFFFFF)
        elif status == S_TYPE:
            cause = TypeError("unsupported operand type for mix/fold")
        elif status == S_ENCODE:
            cause = UnicodeEncodeError("utf-8", "", 0, 1, "surrogates not allowed")
        elif status == S_OVERFLOW:
            cause = OverflowError("float too large to pack with f format")
        elif status == S_UNSUPPORTED:
            cause = UnsupportedOnDevice(msg)
        elif status == S_EMIT:
            cause = EmitError(msg.split(": ", 1)[-1])
        elif status == S_INVARIANT:
            cause = BatchInvariantError(msg.split(": ", 1)[-1])
        elif status == S_VALUE:
            cause = ValueError(msg)
        else:
            return RuntimeError(f"fbx status {status}: {msg}")
        if layer.value:
            return LayerExecutionError(layer.value, node.value.decode(), cause)
        return cause

    # -- _extract_batch ------------------------------------------------------------
    def extract(self, table: ViewImage, stream: int = 0) -> ViewImage:
        n = table.row_count
        keep: list = []
        cols = (Column * max(1, len(self.inputs)))(
            *[column_struct(table.columns[c], keep) for c in self.inputs])
        st = self.L.fbx_extract(self.h, cols, len(self.inputs), n, ctypes.byref(self.counters),
                                vp(stream))
        if st < 0:
            raise runtime.FbxError(f"fbx_extract: {self.L.fbx_error_message(None).decode()}")
        if st:
            raise self.error(st)
        out = {c: table.columns[c] for c in table.order}
        for j, (col, kind, _dom) in enumerate(self.outputs):
            k, rows, nbytes = c_u(), c_ull(), c_ull()
            self.L.fbx_output_info(self.h, j, ctypes.byref(k), ctypes.byref(rows),
                                   ctypes.byref(nbytes))
            nulls = np.zeros((n + 7) // 8, np.uint8)
            if k.value == Kind.INT64:
                data = np.zeros(n, np.int64)
                self.L.fbx_output_copy(self.h, j, nulls.ctypes.data, data.ctypes.data, None,
                                       vp(stream))
                out[col] = ColumnImage(Kind.INT64, n, nulls, data)
            else:
                data = np.zeros(max(1, nbytes.value), np.uint8)
                offs = np.zeros(n + 1, np.uint32)
                self.L.fbx_output_copy(self.h, j, nulls.ctypes.data, data.ctypes.data,
                                       offs.ctypes.data, vp(stream))
                out[col] = ColumnImage(Kind.UTF8, n, nulls, data[:nbytes.value], offs)
        return ViewImage(out, table.key_columns, tuple(table.order) + tuple(
            c for c, *_ in self.outputs))

    # -- emit_minibatch --------------------------------------------------------------
    def emit_csr(self, ids: ColumnImage, labels: ColumnImage,
                 features: Sequence[tuple[ColumnImage, int]], stream: int = 0) -> dict:
        """emit_minibatch + validate over one batch: CSR (ids, labels, offsets,
        slots, signs) and the batch digest; raises the reference's EmitError /
        BatchInvariantError."""
        n = ids.n
        keep: list = []
        cid, clab = column_struct(ids, keep), column_struct(labels, keep)
        feats = (Column * max(1, len(features)))(*[column_struct(c, keep) for c, _ in features])
        slots = np.array([s for _, s in features] or [0], np.uint32)
        csr = Csr()
        st = self.L.fbx_emit_csr(self.h, ctypes.byref(cid), ctypes.byref(clab), feats,
                                 slots.ctypes.data, len(features), n, ctypes.byref(csr), vp(stream))
        if st < 0:
            raise runtime.FbxError(f"fbx_emit_csr: {self.L.fbx_error_message(None).decode()}")
        if st:
            raise self.error(st)
        m = csr.n_signs
        out = {"ids": np.zeros(n, np.uint64), "labels": np.zeros(n, np.uint8),
               "offsets": np.zeros(n + 1, np.uint64), "slots": np.zeros(max(1, m), np.uint16),
               "signs": np.zeros(max(1, m), np.uint64)}
        csr = Csr(out["ids"].ctypes.data, out["labels"].ctypes.data, out["offsets"].ctypes.data,
                  out["slots"].ctypes.data, out["signs"].ctypes.data, max(1, m), 0, 0)
        st = self.L.fbx_emit_csr(self.h, ctypes.byref(cid), ctypes.byref(clab), feats,
                                 slots.ctypes.data, len(features), n, ctypes.byref(csr), vp(stream))
        if st:
            raise self.error(st) if st > 0 else runtime.FbxError(
                self.L.fbx_error_message(None).decode())
        out["slots"], out["signs"] = out["slots"][:m], out["signs"][:m]
        out["digest"] = csr.digest
        return out
