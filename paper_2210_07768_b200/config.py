"""Pipeline configuration: the reference's JSON schema, names and errors.

Mirrors ``pkg/src/featurebox/pipeline.py:91-343`` (``ConfigError``,
``StageError``, ``ViewSource``, ``PipelineConfig``, ``load_config``) and the
clean-policy / filter part of ``viewpipe.py:31-331`` (``CleanPolicy``,
``JsonExtraction``, ``parse_filter``, ``bind_filter``).  Parsing and binding
run on the host once per run; the bound filter is compiled into the fused
kernel by ``codegen.py``.
"""

from __future__ import annotations

import os

import json
import re
import struct
from dataclasses import dataclass, field
from pathlib import Path
from typing import Mapping

from .columns import Kind
from .featureops import (SLOT_MAX, DictTable, FeatureConfigError, FunctionRef, OperatorSpec,
                         load_dict_table, register_operator)

PIPELINED = "pipelined"
STAGED = "staged"
DEFAULT_BATCH_SIZE = 512
DEFAULT_QUEUE_DEPTH = 4
DEFAULT_POOL_BYTES = 8 << 20
DEFAULT_BUDGET_BYTES = 64 << 10
DEFAULT_BANDWIDTH = 1e9
DEFAULT_LAUNCH_OVERHEAD_US = 3.45


class ConfigError(ValueError):
    """The pipeline configuration is malformed (pipeline.py:91)."""


class CleanConfigError(ValueError):
    """A clean policy references missing columns or mismatched kinds."""


class JoinConfigError(ValueError):
    pass


class MergeUniquenessError(ValueError):
    """A merge side holds the same instance id more than once."""


class EmitError(ValueError):
    pass


class BatchInvariantError(ValueError):
    pass


class UnsupportedOnDevice(ConfigError):
    """A construct the B200 engine does not implement bit-exactly yet.

    Raised at plan time (never a silent divergence and never a CPU fallback).
    """


class StageError(RuntimeError):
    """A pipeline stage failed; carries the stage name and batch index."""

    def __init__(self, stage: str, batch_index: int | None, cause: BaseException):
        where = f"batch {batch_index}" if batch_index is not None else "whole input"
        super().__init__(f"stage {stage!r} failed at {where}: {cause}")
        self.stage = stage
        self.batch_index = batch_index
        self.__cause__ = cause


class LayerExecutionError(RuntimeError):
    """An operator failed; identifies the layer and node (device.py:34-41)."""

    def __init__(self, layer_index: int, node: str, cause: BaseException):
        super().__init__(f"layer {layer_index}: operator {node!r} failed: {cause}")
        self.layer_index = layer_index
        self.node = node
        self.__cause__ = cause


class PoolExhausted(MemoryError):
    def __init__(self, requested: int, remaining: int):
        super().__init__(f"arena pool exhausted: requested {requested} bytes, "
                         f"{remaining} remaining")
        self.requested = requested
        self.remaining = remaining


# -- filter expressions (viewpipe.py:54-215) ------------------------------------

_TOKEN_RE = re.compile(
    r"\s*(?:(?P<num>-?\d+\.\d+|-?\d+)|(?P<ident>[A-Za-z_][A-Za-z0-9_]*)"
    r"|(?P<str>'[^']*'|\"[^\"]*\")|(?P<op>==|!=|<=|>=|<|>|&&|\|\||[()]))")
_COMPARE_OPS = ("==", "!=", "<", "<=", ">", ">=")


@dataclass(frozen=True)
class Comparison:
    column: str
    op: str
    literal: int | float | str


@dataclass(frozen=True)
class BoolExpr:
    kind: str  # "and" | "or"
    parts: tuple


def _lex(text: str) -> list[tuple[str, object]]:
    out, pos = [], 0
    while pos < len(text):
        m = _TOKEN_RE.match(text, pos)
        if not m or m.end() == pos:
            rest = text[pos:].strip()
            if not rest:
                break
            raise CleanConfigError(f"filter: cannot tokenize at {rest[:20]!r}")
        pos = m.end()
        if m["num"] is not None:
            out.append(("num", m["num"]))
        elif m["ident"] is not None:
            w = m["ident"]
            out.append(("bool", w) if w in ("and", "or") else ("ident", w))
        elif m["str"] is not None:
            out.append(("str", m["str"][1:-1]))
        else:
            o = m["op"]
            out.append(("bool", "and") if o == "&&" else ("bool", "or") if o == "||" else ("op", o))
    return out


def parse_filter(text: str):
    """Comparisons joined by and/or with parentheses; `and` binds tighter."""
    toks = _lex(text)
    pos = 0

    def peek():
        return toks[pos] if pos < len(toks) else None

    def take():
        nonlocal pos
        if pos >= len(toks):
            raise CleanConfigError("filter: unexpected end of expression")
        pos += 1
        return toks[pos - 1]

    def disj():
        parts = [conj()]
        while peek() == ("bool", "or"):
            take()
            parts.append(conj())
        return parts[0] if len(parts) == 1 else BoolExpr("or", tuple(parts))

    def conj():
        parts = [atom()]
        while peek() == ("bool", "and"):
            take()
            parts.append(atom())
        return parts[0] if len(parts) == 1 else BoolExpr("and", tuple(parts))

    def atom():
        tok = take()
        if tok == ("op", "("):
            inner = disj()
            if take() != ("op", ")"):
                raise CleanConfigError("filter: expected ')'")
            return inner
        if tok[0] != "ident":
            raise CleanConfigError(f"filter: expected column name, got {tok[1]!r}")
        op = take()
        if op[0] != "op" or op[1] not in _COMPARE_OPS:
            raise CleanConfigError(f"filter: expected comparison after {tok[1]!r}")
        lit = take()
        if lit[0] == "num":
            value = float(lit[1]) if "." in lit[1] else int(lit[1])
        elif lit[0] == "str":
            value = lit[1]
        else:
            raise CleanConfigError(f"filter: expected literal, got {lit[1]!r}")
        return Comparison(tok[1], op[1], value)

    expr = disj()
    if peek() is not None:
        raise CleanConfigError(f"filter: trailing tokens at {peek()[1]!r}")
    return expr


def canon_f32(value: float) -> float:
    return struct.unpack("<f", struct.pack("<f", value))[0]


def bind_filter(expr, kinds: Mapping[str, Kind]):
    """Check columns / literal kinds; canonicalise Float32 literals."""
    if isinstance(expr, BoolExpr):
        return BoolExpr(expr.kind, tuple(bind_filter(p, kinds) for p in expr.parts))
    if expr.column not in kinds:
        raise KeyError(expr.column)
    kind = kinds[expr.column]
    lit = expr.literal
    if kind in (Kind.UTF8, Kind.JSON):
        if not isinstance(lit, str):
            raise CleanConfigError(f"filter: column {expr.column!r} is text, literal {lit!r} is not")
    else:
        if isinstance(lit, str):
            raise CleanConfigError(f"filter: column {expr.column!r} is numeric, literal is text")
        if kind is Kind.FLOAT32:
            lit = canon_f32(float(lit))
    return Comparison(expr.column, expr.op, lit)


# -- clean policy (viewpipe.py:218-331) --------------------------------------------

@dataclass(frozen=True)
class JsonExtraction:
    source: str
    path: str
    output: str
    kind: Kind

    def __post_init__(self):
        if not self.path or any(not p for p in self.path.split(".")):
            raise CleanConfigError(f"bad extraction path {self.path!r}")
        if not self.output:
            raise CleanConfigError("extraction output name must be non-empty")


@dataclass(frozen=True)
class CleanPolicy:
    fills: Mapping[str, object] = field(default_factory=dict)
    extractions: tuple[JsonExtraction, ...] = ()
    filter: object | None = None

    def __post_init__(self):
        outs = [e.output for e in self.extractions]
        if len(set(outs)) != len(outs):
            raise CleanConfigError("duplicate extraction output names")


def _check_fill(column: str, kind: Kind, value) -> None:
    if isinstance(value, bool):
        raise CleanConfigError(f"fill for {column!r}: bool is not a column value")
    if kind is Kind.INT64 and isinstance(value, int):
        return
    if kind is Kind.FLOAT32 and isinstance(value, (int, float)):
        return
    if kind in (Kind.UTF8, Kind.JSON) and isinstance(value, str):
        return
    raise CleanConfigError(f"fill for {column!r}: {value!r} does not match kind {kind.name}")


def cleaned_kinds(kinds: Mapping[str, Kind], policy: CleanPolicy) -> dict[str, Kind]:
    out = dict(kinds)
    for e in policy.extractions:
        out.setdefault(e.output, e.kind)
    return out


def validate_clean_policy(kinds: Mapping[str, Kind], policy: CleanPolicy) -> None:
    """Static checks of a policy against a schema (viewpipe.py:297-318)."""
    for column, value in policy.fills.items():
        if column not in kinds:
            raise CleanConfigError(f"fill references unknown column {column!r}")
        _check_fill(column, kinds[column], value)
    for ext in policy.extractions:
        if ext.source not in kinds:
            raise CleanConfigError(f"extraction source {ext.source!r} unknown")
        if kinds[ext.source] is not Kind.JSON:
            raise CleanConfigError(f"extraction source {ext.source!r} is not Json")
        if ext.output in kinds and kinds[ext.output] is not ext.kind:
            raise CleanConfigError(
                f"extraction output {ext.output!r} collides with an existing column "
                f"of a different kind")
    if policy.filter is not None:
        bind_filter(policy.filter, cleaned_kinds(kinds, policy))


# -- pipeline config (pipeline.py:115-343) -------------------------------------------

@dataclass(frozen=True)
class ViewSource:
    name: str
    path: Path
    columns: tuple[str, ...] | None
    policy: CleanPolicy


def host_worker_count(requested: int | None = None) -> int:
    """Effective host workers (device.py:81-96): the requested count (else the CPU
    count), capped by FEATUREBOX_THREADS when it is set; a bad cap is a ValueError
    (a ConfigError once a run starts, pipeline.py:697-701)."""
    base = requested if requested is not None else (os.cpu_count() or 1)
    cap_text = os.environ.get("FEATUREBOX_THREADS")
    if cap_text:
        try:
            cap = int(cap_text)
        except ValueError:
            raise ValueError(f"FEATUREBOX_THREADS={cap_text!r} is not an integer") from None
        if cap < 1:
            raise ValueError("FEATUREBOX_THREADS must be >= 1")
        base = min(base, cap)
    return max(1, base)


def run_workers(config: "PipelineConfig") -> int:
    """The run-start checks of the reference's ExecContext (pipeline.py:697-711,
    device.py:116-125): host_worker_count (a bad FEATUREBOX_THREADS is a
    ConfigError), then the device shape, fusion mode and bandwidth (ValueError,
    raised as the reference raises it).  Returns the effective host workers."""
    try:
        workers = host_worker_count(config.workers)
    except ValueError as exc:
        raise ConfigError(str(exc)) from exc
    if config.fusion not in ("fused", "unfused"):
        raise ValueError("fusion must be 'fused' or 'unfused'")
    if config.lanes_per_group < 1 or config.work_groups < 1:
        raise ValueError("device shape must be at least 1x1")
    if not config.bandwidth_bytes_per_s > 0:
        raise ValueError("bandwidth must be positive")
    return workers


@dataclass(frozen=True)
class PipelineConfig:
    views: tuple[ViewSource, ...]
    driver: str
    basic_path: Path
    operators: tuple[OperatorSpec, ...]
    tables: Mapping[str, DictTable]
    features: Mapping[str, int]
    join_keys: tuple[str, ...] = ()
    basic_columns: tuple[str, ...] | None = None
    batch_size: int = DEFAULT_BATCH_SIZE
    mode: str = PIPELINED
    staging_dir: Path | None = None
    workers: int | None = None
    queue_depth: int = DEFAULT_QUEUE_DEPTH
    device_budget_bytes: int | float = DEFAULT_BUDGET_BYTES
    pool_bytes: int = DEFAULT_POOL_BYTES
    lanes_per_group: int = 256
    work_groups: int = 8
    bandwidth_bytes_per_s: float = DEFAULT_BANDWIDTH
    per_launch_overhead_us: float = DEFAULT_LAUNCH_OVERHEAD_US
    fusion: str = "fused"
    instance_column: str = "instance_id"
    label_column: str = "label"

    def __post_init__(self):
        if not self.views:
            raise ConfigError("at least one view is required")
        names = [v.name for v in self.views]
        if len(set(names)) != len(names):
            raise ConfigError("view names must be unique")
        if self.driver not in names:
            raise ConfigError(f"driver view {self.driver!r} not among views")
        if len(self.views) > 1 and not self.join_keys:
            raise ConfigError("multiple views require join keys")
        if self.batch_size < 1:
            raise ConfigError("batch_size must be >= 1")
        if self.mode not in (PIPELINED, STAGED):
            raise ConfigError(f"mode must be {PIPELINED!r} or {STAGED!r}")
        if self.queue_depth < 1:
            raise ConfigError("queue_depth must be >= 1")
        if self.workers is not None and self.workers < 1:
            raise ConfigError("workers must be >= 1")
        if self.pool_bytes <= 0 or self.pool_bytes % 128 != 0:
            raise ConfigError("pool_bytes must be a positive multiple of 128")
        for col, slot in self.features.items():
            if not 0 <= slot <= SLOT_MAX:
                raise ConfigError(f"feature {col!r}: slot {slot} outside u16")

    def view(self, name: str) -> ViewSource:
        return next(v for v in self.views if v.name == name)


def _req(obj: Mapping, key: str, where: str):
    if key not in obj:
        raise ConfigError(f"{where}: missing required key {key!r}")
    return obj[key]


def _resolve(base: Path, p: str) -> Path:
    path = Path(p)
    return path if path.is_absolute() else base / path


def _function_ref(raw: Mapping, where: str, tables: Mapping[str, DictTable]) -> FunctionRef:
    spec = _req(raw, "fn", where)
    footprint = raw.get("footprint_bytes")
    if footprint is None and isinstance(spec, str) and spec.startswith("lookup:"):
        t = spec.partition(":")[2]
        if t in tables:
            footprint = tables[t].size_bytes
    try:
        return FunctionRef(spec=spec, arg=raw.get("arg"),
                           footprint_bytes=64 if footprint is None else int(footprint),
                           kind=raw.get("kind", "compute-bound"))
    except FeatureConfigError as exc:
        raise ConfigError(f"{where}: {exc}") from exc


def config_from_dict(raw: Mapping, base: str | Path = ".",
                     tables: Mapping[str, DictTable] | None = None) -> PipelineConfig:
    """Build a PipelineConfig from the parsed JSON form (load_config's body)."""
    if not isinstance(raw, dict):
        raise ConfigError("config root must be an object")
    base = Path(base)
    if tables is None:
        tables = {}
        for name, t in raw.get("tables", {}).items():
            try:
                tables[name] = load_dict_table(_resolve(base, _req(t, "path", f"table {name!r}")),
                                               default=t.get("default", 0),
                                               size_bytes=t.get("size_bytes"))
            except (OSError, ValueError) as exc:
                if isinstance(exc, ConfigError):
                    raise
                raise ConfigError(f"table {name!r}: {exc}") from exc
    views = []
    for v in _req(raw, "views", "config"):
        name = _req(v, "name", "view")
        where = f"view {name!r}"
        clean = v.get("clean", {})
        exts = []
        for e in clean.get("extract", ()):
            try:
                exts.append(JsonExtraction(source=_req(e, "source", where),
                                           path=_req(e, "path", where),
                                           output=_req(e, "output", where),
                                           kind=Kind.from_name(_req(e, "kind", where))))
            except (ValueError, CleanConfigError) as exc:
                if isinstance(exc, ConfigError):
                    raise
                raise ConfigError(f"{where}: {exc}") from exc
        filt = clean.get("filter")
        try:
            policy = CleanPolicy(fills=dict(clean.get("fills", {})), extractions=tuple(exts),
                                 filter=parse_filter(filt) if filt else None)
        except CleanConfigError as exc:
            raise ConfigError(f"{where}: {exc}") from exc
        cols = v.get("columns")
        views.append(ViewSource(name, _resolve(base, _req(v, "path", where)),
                                tuple(cols) if cols is not None else None, policy))
    operators, registry = [], {}
    for o in raw.get("operators", ()):
        name = _req(o, "name", "operator")
        where = f"operator {name!r}"
        try:
            spec = OperatorSpec(
                name=name,
                inputs=tuple(_req(o, "inputs", where)),
                outputs=tuple(_req(o, "outputs", where)),
                body=_function_ref(_req(o, "body", where), where, tables),
                pre_calls=tuple(_function_ref(p, where, tables) for p in o.get("pre", ())),
                post_calls=tuple(_function_ref(p, where, tables) for p in o.get("post", ())),
                footprint_bytes=int(o.get("footprint_bytes", 64)),
                kind=o.get("kind", "compute-bound"))
            register_operator(spec, registry)
        except FeatureConfigError as exc:
            raise ConfigError(f"{where}: {exc}") from exc
        operators.append(spec)
    features = {str(c): int(s) for c, s in raw.get("emit", {}).get("features", {}).items()}
    basic = _req(raw, "basic", "config")
    device = raw.get("device", {})
    staging = raw.get("staging_dir")
    try:
        return PipelineConfig(
            views=tuple(views),
            driver=_req(raw, "driver", "config"),
            basic_path=_resolve(base, _req(basic, "path", "basic")),
            basic_columns=tuple(basic["columns"]) if basic.get("columns") is not None else None,
            join_keys=tuple(raw.get("join", {}).get("keys", ())),
            operators=tuple(operators),
            tables=tables,
            features=features,
            batch_size=int(raw.get("batch_size", DEFAULT_BATCH_SIZE)),
            mode=raw.get("mode", PIPELINED),
            staging_dir=_resolve(base, staging) if staging else None,
            workers=int(raw["workers"]) if raw.get("workers") is not None else None,
            queue_depth=int(raw.get("queue_depth", DEFAULT_QUEUE_DEPTH)),
            device_budget_bytes=device.get("budget_bytes", DEFAULT_BUDGET_BYTES),
            pool_bytes=int(device.get("pool_bytes", DEFAULT_POOL_BYTES)),
            lanes_per_group=int(device.get("lanes_per_group", 256)),
            work_groups=int(device.get("work_groups", 8)),
            bandwidth_bytes_per_s=float(device.get("bandwidth_bytes_per_s", DEFAULT_BANDWIDTH)),
            per_launch_overhead_us=float(device.get("per_launch_overhead_us",
                                                    DEFAULT_LAUNCH_OVERHEAD_US)),
            fusion=device.get("fusion", "fused"),
            instance_column=raw.get("instance_column", "instance_id"),
            label_column=raw.get("label_column", "label"),
        )
    except (TypeError, ValueError) as exc:
        if isinstance(exc, ConfigError):
            raise
        raise ConfigError(f"config: {exc}") from exc


def load_config(path: str | Path) -> PipelineConfig:
    """Parse a JSON pipeline config; paths resolve relative to the file."""
    path = Path(path)
    try:
        raw = json.loads(path.read_text(encoding="utf-8"))
    except OSError as exc:
        raise ConfigError(f"cannot read config {path}: {exc}") from exc
    except json.JSONDecodeError as exc:
        raise ConfigError(f"config {path} is not valid JSON: {exc}") from exc
    return config_from_dict(raw, path.parent)
