"""Reference-side binding: run the UNMODIFIED reference pipeline with the B200
engine in the seat of ``featurebox.pipeline._extract_batch`` (pipeline.py:718-737).

    import featurebox.pipeline as P
    from paper_2210_07768_b200 import refshim
    refshim.install(P)                     # patches P._extract_batch
    report = P.run_pipelined(P.load_config("pipeline.json"))
    refshim.uninstall(P)

The shim is the maintainer-side glue INTEGRATION.md describes: it converts the
reference's ``ColumnBatch`` (Python value lists + null bytearrays) into FBXC
column images, plans the reference's operator DAG once per ``_Prepared`` with
this package's planner (NVRTC-compiled ``fbx_extract_rows``), runs it through the
C-ABI engine object (``fbx_create`` / ``fbx_extract``, include/fbx.h), and
rebuilds the appended output columns with the reference's own ``Column.build``.
A failure comes back as the reference's ``LayerExecutionError(layer, node,
cause)``, so the reference's stage wrapping (``StageError``) is unchanged.
Nothing here imports the reference: its classes are taken from the patched module.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from . import config as C
from . import featureops as F
from .columns import ColumnImage, Kind, ViewImage

_STATE: dict = {}


def _our_ref(r) -> F.FunctionRef:
    return F.FunctionRef(r.spec, r.arg, r.footprint_bytes, r.kind)


def _our_config(ref_cfg) -> C.PipelineConfig:
    """The planner-relevant part of the reference's PipelineConfig as this
    package's (the schemas are field-for-field the same)."""
    ops = tuple(F.OperatorSpec(o.name, tuple(o.inputs), tuple(o.outputs), _our_ref(o.body),
                               tuple(_our_ref(p) for p in o.pre_calls),
                               tuple(_our_ref(p) for p in o.post_calls), o.footprint_bytes,
                               o.kind) for o in ref_cfg.operators)
    tables = {n: F.DictTable(dict(t.entries), t.default, t.size_bytes)
              for n, t in ref_cfg.tables.items()}
    view = C.ViewSource("table", Path("."), None, C.CleanPolicy())
    return C.PipelineConfig(
        views=(view,), driver="table", basic_path=Path("."), operators=ops, tables=tables,
        features={}, device_budget_bytes=ref_cfg.device_budget_bytes,
        pool_bytes=ref_cfg.pool_bytes, lanes_per_group=ref_cfg.lanes_per_group,
        instance_column=ref_cfg.instance_column, label_column=ref_cfg.label_column)


def batch_to_view(table) -> ViewImage:
    """A reference ColumnBatch as FBXC column images (no per-value Python work
    beyond the list -> array conversion)."""
    cols = {}
    order = []
    for name, kind in table.schema.columns:
        col = table.columns[name]
        k = Kind(kind.value)
        n = len(col.values)
        nulls = np.frombuffer(bytes(col.nulls), dtype=np.uint8).copy()
        if nulls.size < (n + 7) // 8:
            nulls = np.concatenate([nulls, np.zeros((n + 7) // 8 - nulls.size, np.uint8)])
        if k is Kind.INT64:
            img = ColumnImage(k, n, nulls, np.array(col.values, dtype=np.int64))
        elif k is Kind.FLOAT32:
            img = ColumnImage(k, n, nulls, np.array(col.values, dtype=np.float32))
        else:
            blobs = [v.encode("utf-8", "surrogatepass") for v in col.values]
            offs = np.zeros(n + 1, dtype=np.uint64)
            np.cumsum([len(b) for b in blobs], out=offs[1:])
            data = np.frombuffer(b"".join(blobs), dtype=np.uint8).copy()
            img = ColumnImage(k, n, nulls, data, offs.astype(np.uint32))
        cols[name] = img
        order.append(name)
    return ViewImage(cols, tuple(table.schema.key_columns), tuple(order))


def _engine_for(prepared, table_kinds, device):
    key = (id(prepared), tuple(table_kinds.items()))
    ent = _STATE.get("engines", {}).get(key)
    if ent is None or ent[0] is not prepared:
        from .capi import CEngine
        from .engine import prepare_extract
        ours = prepare_extract(_our_config(prepared.config), table_kinds)
        ent = (prepared, CEngine(ours, device))
        _STATE.setdefault("engines", {})[key] = ent
    return ent[1]


def install(pipeline_module, device: int = 0) -> None:
    """Patch ``pipeline_module._extract_batch`` (the reference's
    featurebox.pipeline) to run on the B200 engine."""
    P = pipeline_module
    if "orig" not in _STATE:
        _STATE["orig"] = P._extract_batch
    import importlib
    pkg = P.__name__.rsplit(".", 1)[0]
    Column, ColumnBatch, ViewSchema = P.Column, P.ColumnBatch, P.ViewSchema
    LayerExecutionError = importlib.import_module(pkg + ".device").LayerExecutionError
    PoolExhausted = importlib.import_module(pkg + ".mempool").PoolExhausted

    def b200_extract_batch(table, prepared, ctx):
        kinds = {n: Kind(k.value) for n, k in table.schema.columns}
        eng = _engine_for(prepared, kinds, device)
        try:
            out = eng.extract(batch_to_view(table))
        except C.LayerExecutionError as exc:  # -> the reference's exception types
            cause = exc.__cause__
            if isinstance(cause, C.PoolExhausted):
                cause = PoolExhausted(cause.requested, cause.remaining)
            err = LayerExecutionError(exc.layer_index, exc.node, cause)  # sets __cause__
        else:
            err = None
        if err is not None:
            raise err
        ctx.count_launches(1)  # one fused kernel per batch (device.py:382 counts per layer)
        spec = list(table.schema.columns)
        columns = dict(table.columns)
        for col, kind, _domain in prepared.extract_outputs:
            spec.append((col, kind))
            columns[col] = Column.build(kind, _values(out.columns[col]))
        schema = ViewSchema(tuple(spec), table.schema.key_columns, table.schema.row_count)
        return ColumnBatch(schema, columns)

    P._extract_batch = b200_extract_batch


def uninstall(pipeline_module) -> None:
    if "orig" in _STATE:
        pipeline_module._extract_batch = _STATE.pop("orig")
    for _, eng in _STATE.pop("engines", {}).values():
        eng.close()


def _values(img: ColumnImage) -> list:
    """An output image as the Python values Column.build takes (None = null;
    strings decoded with lone surrogates kept, like the reference's str)."""
    null = img.null_mask()
    if img.kind is Kind.INT64:
        return [None if z else v for z, v in zip(null.tolist(), img.data.tolist())]
    raw = img.data.tobytes()
    offs = img.offsets.tolist()
    return [None if null[i] else raw[offs[i]:offs[i + 1]].decode("utf-8", "surrogatepass")
            for i in range(img.n)]
