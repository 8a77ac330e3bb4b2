"""Plan -> CUDA: the runtime-compiled fused meta-kernel of a whole plan.

The reference runs each layer of the operator DAG as one "meta-kernel" over
a chunk (device.py:341-410, runtime compilation :207).
Every operator is row-local, so on the B200 the whole per-record path of a
driver chunk -- clean (viewpipe.py:334-431), side-view join probe
(viewpipe.py:537-547), the layered DAG (device.py:434-444), the uniqueness
check + basic merge (pipeline.py:1055-1075) and emission (pipeline.py:
375-433) -- is generated as ONE kernel: one CTA per chunk of ``batch_size``
rows, one thread per row, the layer order as program order.  The chunk's
instances are then sorted by instance id in shared memory (the reference's
merge order, viewpipe.py:521), the CSR offsets are placed with a decoupled
look-back across chunks, and counters/digest are reduced once per CTA.

Static typing of values lets the generator specialise every node:
  i64 (Int64 column) | u64 (sign / lookup result) | f32 (Float32 column) | str.
A string is a view ``fbx::Str`` into the staged record bytes, an input
column, the HBM pool or a per-thread decimal buffer; only ``lower`` (when a
byte changes), multi-part ``concat`` and escaped JSON strings allocate, via
the block-level bump allocator (mempool.py:114-134).

Constructs without a bit-exact device implementation raise
``UnsupportedOnDevice`` at plan time (never a silent divergence).
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass, field
from fractions import Fraction
from pathlib import Path
from typing import Mapping, Sequence

from .columns import Kind
from .config import BoolExpr, Comparison, UnsupportedOnDevice
from .featureops import FunctionDef, fnv1a64

CSRC = Path(__file__).resolve().parent / "csrc"
INCLUDE = Path(__file__).resolve().parent.parent / "include"

INT64_MIN, INT64_MAX = -(1 << 63), (1 << 63) - 1
SPAN_BUDGET = 40 * 1024  # bytes of dynamic shared memory for staged record spans
OUT_BUDGET = 96 * 1024   # cap for staging a tile's CSR before the coalesced write-out
STATIC_SMEM_EST = 6 * 1024
MASK64 = (1 << 64) - 1

STAGE = {"prepare": 0, "read": 1, "clean": 2, "join": 3, "extract": 4, "merge": 5, "emit": 6}
ERR = {"type": 1, "value": 2, "encode": 3, "pool": 4, "null_label": 5, "label_range": 6,
       "dup_id": 7, "multi_match": 8, "json_bigint": 9, "json_deep": 10,
       "unicode_lower": 11, "float_overflow": 12, "float_slow": 13, "internal": 14,
       "pool_key": 15, "basic_dup": 16}


def library_source() -> str:
    """fbx_abi.h + fbx_core.cuh, flattened for NVRTC (no include paths)."""
    abi = (INCLUDE / "fbx_abi.h").read_text()
    core = (CSRC / "device" / "fbx_core.cuh").read_text()
    uni = (CSRC / "device" / "fbx_unicode.cuh").read_text()
    p10 = (CSRC / "device" / "fbx_pow10.cuh").read_text()
    return abi + "\n" + core.replace('#include "fbx_abi.h"', "").replace(
        '#include "fbx_unicode.cuh"', uni).replace('#include "fbx_pow10.cuh"', p10)


# ---------------------------------------------------------------------------
# plan IR consumed by the generator (built by engine.prepare)
# ---------------------------------------------------------------------------

@dataclass
class ViewIR:
    name: str
    kinds: dict[str, Kind]          # input columns (after projection), ordered
    fills: dict[str, object]
    extractions: list               # config.JsonExtraction
    filter: object | None           # bound filter expression
    keys: tuple[str, ...] = ()      # join key columns (side views / basic)

    def cleaned_kinds(self) -> dict[str, Kind]:
        out = dict(self.kinds)
        for e in self.extractions:
            out.setdefault(e.output, e.kind)
        return out


@dataclass
class NodeIR:
    name: str
    role: str                       # pre | body | post
    op: str                         # operator name
    fn: FunctionDef
    layer: int
    rank: int                       # (layer, name) rank: error priority
    inputs: tuple[str, ...] = ()    # body: operator inputs; pre: (column,)
    slot: int | None = None
    writes: tuple[str, ...] = ()
    ref_pool: bool = False          # the reference runs it on the device from its arena pool


@dataclass
class PlanIR:
    driver: ViewIR
    sides: list[ViewIR]
    basic: ViewIR | None
    join_keys: tuple[str, ...]
    nodes: list[NodeIR]             # in (layer, name) order
    pre_of: dict[str, dict[int, str]]
    producer: dict[str, str]        # column -> node producing it
    features: dict[str, int]
    instance_column: str
    label_column: str
    chunk: int
    tables: dict[str, int]          # dictionary name -> table index
    table_defaults: dict[str, int]
    extract_outputs: list[tuple[str, str]] = field(default_factory=list)  # (col, domain)
    stage_strings: bool = True
    mode: str = "pipeline"          # "pipeline" | "extract" (row-aligned _extract_batch)
    #                                 | "clean" (clean_views of `driver`, row-aligned: staged mode)
    pool_bytes: int = 8 << 20       # the reference arena's capacity (config device.pool_bytes)
    lanes_per_group: int = 256      # its group size (config device.lanes_per_group)


@dataclass
class Program:
    source: str
    slots: dict[str, int]           # param slot name -> index
    threads: int
    smem_bytes: int
    kernels: list[str]
    side_kernels: list[str]
    notes: list[str]
    int_keyed: tuple[int, ...] = ()   # tables with 16-B fbx::ISlot slots
    json_kind: bool = False           # Json-kind extraction: canonical JSON into the pool
    tiles_per_chunk: int = 1          # > 1: chunk cut into 512-row sub-tiles (merged after)
    # the reference arena's accounting (fbx_pool_account): device token nodes as
    # (layer, rank, input plane) in the reference's order, key words per row
    # (~0: rows in table order), lane-size planes, rows per tile
    ref_pool: tuple = ()
    pool_kw: int = 0
    pool_ni: int = 0
    tile_rows: int = 512
    # bump-pool rounding per tile, summed over the plan's pool sites: a CTA grant
    # rounds to 128 B, a warp grant to 16 B per warp (the engine's arena slack)
    pool_slack_per_tile: int = 0


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------

@dataclass
class V:
    """A value in generated code: C var `c` (+ `c_n` null flag, `c_l` lone)."""

    t: str                # i64 | u64 | f32 | str
    c: str
    nullable: bool = True
    lone: bool = False
    lower: bool = False   # str view whose (ASCII) bytes are lowercased on read

    @property
    def n(self) -> str:
        return f"{self.c}_n" if self.nullable else "false"

    @property
    def l(self) -> str:  # noqa: E743
        return f"{self.c}_l" if self.lone else "false"


def _c_bytes(b: bytes) -> str:
    return "{" + ",".join(str(x) for x in b) + ("}" if b else "0}")


def _u64(v: int) -> str:
    return f"0x{v & MASK64:016X}ull"


def _i64(v: int) -> str:
    return f"((i64){_u64(v)})"


def _f32_bits(x: float) -> int:
    b = struct.unpack("<I", struct.pack("<f", x))[0]
    if (b & 0x7F800000) == 0x7F800000 and (b & 0x007FFFFF):
        b |= 0x00400000
    return b


class Gen:
    """Line emitter with slot + constant pools."""

    def __init__(self):
        self.lines: list[str] = []
        self.ind = 0
        self.slots: dict[str, int] = {}
        self.consts: list[bytes] = []
        self.const_off: dict[bytes, int] = {}
        self.const_size = 0
        self.tmp = 0

    def __call__(self, line: str = ""):
        lead = len(line) - len(line.lstrip("}"))
        self.ind -= lead
        self.lines.append("  " * self.ind + line if line else "")
        self.ind += line.count("{") - line.count("}") + lead

    def slot(self, name: str) -> int:
        if name not in self.slots:
            self.slots[name] = len(self.slots)
        return self.slots[name]

    def p(self, name: str, ctype: str = "u64") -> str:
        return f"(({ctype})P.v[{self.slot(name)}])"

    def const(self, data: bytes) -> str:
        """Offset expression of a byte constant in the K_STR blob."""
        if data not in self.const_off:
            self.const_off[data] = self.const_size
            self.consts.append(data)
            self.const_size += len(data)
        return f"(K_STR + {self.const_off[data]})"

    def fresh(self, base: str) -> str:
        self.tmp += 1
        return f"{base}{self.tmp}"


# ---------------------------------------------------------------------------
# the generator
# ---------------------------------------------------------------------------

class PlanCodegen:
    def __init__(self, ir: PlanIR):
        self.ir = ir
        self.g = Gen()
        self.notes: list[str] = []
        # A chunk (batch_size rows) is one CTA up to 1024 rows.  Larger chunks are cut
        # into sub-tiles of 512 rows (tiles_per_chunk of them, the last ones possibly
        # empty); each sub-tile emits its rows sorted by id and the engine merges the
        # sub-tiles of every chunk afterwards (Engine._merge_big_chunks).
        self.tile_rows = ir.chunk if ir.chunk <= 1024 else 512
        self.spc = -(-ir.chunk // self.tile_rows)  # sub-tiles per chunk
        self.nt = 1 << (max(32, self.tile_rows) - 1).bit_length()  # power of two
        self.nsort = self.nt
        if len(ir.features) > 64:
            raise UnsupportedOnDevice("more than 64 emitted features")
        import os
        # CTAs per SM (sets the register budget): 1024 threads per SM at 64 registers
        # (2 x 512 for the reference's batch_size 512).
        # 3 (<= 40 registers) spills 160-340 B/thread and measured 2-4 % slower on
        # every Appendix-B DAG (round 1), so it is only reachable via the knob.
        default_mb = max(1, min(32, 1024 // self.nt))  # 1024 threads / SM at 64 registers
        self.min_blocks = int(os.environ.get("FBX_MIN_BLOCKS") or default_mb)
        self.pool_sites = 0
        self.json_kind = False
        self._ids_tail: list[str] = []
        # the reference arena (mempool.py): device token nodes in the reference's
        # order; nodes on the same input share one plane of per-row lane sizes
        self.pool_nodes = [nd for nd in ir.nodes if nd.ref_pool]
        planes: dict[tuple, int] = {}
        self.pool_plane_of: dict[str, int] = {}
        for nd in self.pool_nodes:
            key = ("col", nd.inputs[0]) if nd.role == "pre" else ("post", nd.op)
            self.pool_plane_of[nd.name] = planes.setdefault(key, len(planes))
        self.pool_ni = len(planes)
        self.pool_stored: set[int] = set()
        self.pool_kw = 0
        self.pool_kw_bad = False
        self.pf_slot: dict[int, int] = {}
        self.prefetched: dict[tuple, str] = {}
        self.defer_gathers = os.environ.get("FBX_DEFER_GATHERS", "1") != "0"
        # work-balanced warps (rows sorted by string bytes): measured 1-3 % faster on
        # sign_heavy / default / fig4 / cross_heavy, 10 % slower on lookup_heavy
        # (latency-bound dictionary probes, scattered rows) -> off for lookup plans
        has_lookup = any(nd.fn.op == "lookup" for nd in ir.nodes)
        # row sort: on for every plan (end of r1: lookup_heavy 0.330 -> 0.325 ms with it)
        self.sort_rows = os.environ.get("FBX_SORT_ROWS", "1") != "0"
        # warp-aggregated pool grants (no CTA barrier): cross_heavy 0.306 -> 0.296 ms,
        # sign_heavy / default -0.5 %; lookup plans +4 % -> off there
        self.pool_warp = os.environ.get("FBX_POOL_WARP_GRANTS", "0" if has_lookup else "1") != "0"
        self.dict_prefetch = os.environ.get("FBX_DICT_PREFETCH", "1") != "0"
        self.dict_pf: dict[str, tuple] = {}
        # profiling aid: per-phase SM cycles (lane 0 of every warp), printed by the last CTA
        self.phase_timers = os.environ.get("FBX_PHASE_TIMERS", "0") != "0"

    # -- value helpers ---------------------------------------------------------
    def kind_t(self, kind: Kind) -> str:
        return {Kind.INT64: "i64", Kind.FLOAT32: "f32", Kind.UTF8: "str", Kind.JSON: "str"}[kind]

    def decl(self, v: V, init_null: bool = True):
        g = self.g
        ctype = {"i64": "u64", "u64": "u64", "f32": "u32", "str": "fbx::Str"}[v.t]
        init = "fbx::Str{nullptr, 0u}" if v.t == "str" else "0"
        g(f"{ctype} {v.c} = {init};")
        if v.nullable:
            g(f"bool {v.c}_n = {'true' if init_null else 'false'};")
        if v.lone:
            g(f"bool {v.c}_l = false;")

    def row_error(self, stage: str, code: str, layer: int = 0, rank: int = 0,
                  detail: str = "0ull"):
        self.g(f"fbx::raise_err(ST, fbx::err_key(chunk, {STAGE[stage]}u, {layer}u, {rank}u, "
               f"{ERR[code]}u), {detail}); alive = false;")

    # stringify a value for lower/trim/token/concat/lookup (Python str(v))
    def as_str(self, v: V, what: str) -> V:
        if v.t == "str":
            return v
        g = self.g
        s = V("str", g.fresh("dec"), v.nullable)
        buf = s.c + "_buf"
        g(f"__align__(16) u8 {buf}[24];")
        self.decl(s)
        cond = f"alive && !{v.n}" if v.nullable else "alive"
        g(f"if ({cond}) {{")
        if v.t == "f32":  # repr(float) of the widened value
            g(f"u32 L = fbx::f32_repr({buf}, {v.c});")
        else:
            signed = "true" if v.t == "i64" else "false"
            g(f"u32 L = fbx::int_dec_len({v.c}, {signed}); "
              f"fbx::int_dec({buf}, {v.c}, {signed}, L);")
        g(f"{s.c} = fbx::Str{{{buf}, L}};")
        if s.nullable:
            g(f"{s.c}_n = false;")
        g("}")
        return s

    def materialize(self, v: V) -> V:
        """Copy a lazily-lowered view into the pool (consumers that compare
        or store bytes)."""
        if v.t != "str" or not v.lower:
            return v
        g = self.g
        out = V("str", g.fresh("mz"), v.nullable, v.lone)
        self.decl(out)
        cond = f"alive && !{v.n}" if v.nullable else "alive"
        ptr = self.pool_alloc(f"({cond}) ? {v.c}.n : 0u")
        g(f"if (({cond}) && ({ptr} || {v.c}.n == 0u)) {{ if ({v.c}.n) fbx::str_copy_lower({ptr}, {v.c});"
          f" {out.c} = fbx::Str{{{ptr} ? {ptr} : {v.c}.p, {v.c}.n}};"
          + (f" {out.c}_n = false;" if out.nullable else "")
          + (f" {out.c}_l = {v.l};" if out.lone else "") + " }")
        return out

    def pool_alloc(self, size_expr: str) -> str:
        """CTA-uniform pool allocation; returns the pointer var."""
        g = self.g
        self.pool_sites += 1
        ptr = g.fresh("pa")
        g(f"u8* {ptr};")
        g("{")
        g("bool exh = false;")
        g(f"{ptr} = fbx::pool_alloc<NT>(sm.scan, &sm.pool_base, ST, POOL, POOL_CAP, "
          f"(u32)({size_expr}), &exh);")
        g("(void)exh;  // device arena too small: state.pool_overflow, the engine grows it + re-runs")
        g("}")
        return ptr

    # -- staging of the chunk's string spans ------------------------------------------
    def span_decls(self):
        ns_ = len(self.staged)
        g = self.g
        g("// TMA bulk-copy each var-length column's contiguous chunk span into shared")
        g("// memory (first fit in column order; a span that does not fit stays in HBM)")
        g(f"__shared__ const u8* sm_span_buf[{ns_}];")
        g(f"__shared__ u64 sm_span_lo[{ns_}];")
        g(f"__shared__ bool sm_span_ok[{ns_}];")

    def span_tma(self, bounds):
        """One thread: place the spans, arm the mbarrier, issue the bulk copies.
        bounds(i, offsets_ptr) -> (lo, hi) C expressions of span i."""
        g = self.g
        g("u32 used = 0;")
        g("fbx::mbar_init(&sm.bar, 1u);")
        for i, c in enumerate(self.staged):
            offs = g.p(f"drv.{c}.offsets", "const u32*")
            lo, hi = bounds(i, offs)
            g("{")
            g(f"u64 lo = {lo}, hi = {hi};")
            g("u64 alo = lo & ~15ull, ahi = (hi + 15ull) & ~15ull;")
            g("bool ok = used + (ahi - alo) <= SPAN_BUDGET;")
            g(f"sm_span_lo[{i}] = alo; sm_span_ok[{i}] = ok; sm_span_buf[{i}] = dyn_smem + used;")
            g(f"sm.span_lo[{i}] = alo; sm.span_len[{i}] = ok ? (u32)(ahi - alo) : 0u;")
            g("if (ok) used += (u32)(ahi - alo);")
            g("}")
        g("fbx::mbar_expect_tx(&sm.bar, used);")
        for i, c in enumerate(self.staged):
            data = g.p(f"drv.{c}.data", "const u8*")
            g(f"if (sm.span_len[{i}]) fbx::bulk_g2s((void*)sm_span_buf[{i}], "
              f"{data} + sm.span_lo[{i}], sm.span_len[{i}], &sm.bar);")

    # -- the reference arena's demand (fbx_pool_account) -----------------------------
    def pool_decls(self):
        """Shared state of the tile's reference-arena bound (pipeline kernel)."""
        g = self.g
        ni, kw = max(1, self.pool_ni), max(1, len(self.ir.join_keys) if self.ir.sides else 0)
        g("// the reference ArenaPool's demand (mempool.py:114-134): per-input CTA sums of the")
        g("// lane sizes, joined-row count, and per-row key words / sizes / joined flags for")
        g("// fbx_pool_account when the tile's conservative bound exceeds pool_bytes")
        g(f"__shared__ unsigned long long fbx_psum[{ni}]; __shared__ u32 fbx_pjoin;")
        g(f"__shared__ u64 fbx_pkey[{kw}][NT]; __shared__ u32 fbx_psz[{ni}][NT]; __shared__ u8 fbx_pjf[NT];")
        g(f"if (threadIdx.x < {ni}u) fbx_psum[threadIdx.x] = 0ull;")
        g("if (threadIdx.x == 0) fbx_pjoin = 0u;")
        if not self.staged_plan:  # else the row sort / span staging barriers publish them
            g("__syncthreads();")

    def pool_join_site(self, keys: list[V]):
        """Key words of the joined table's order (viewpipe.py:451-534: key image,
        then driver row) and the joined flag of this row."""
        g = self.g
        g("// ---- the reference arena's group order: join-key image, then row ----")
        g("fbx_pjf[RT] = (u8)joined;")
        self.pool_kw = len(keys)
        for j, k in enumerate(keys):
            if k.t in ("i64", "u64", "f32"):  # BE image order == unsigned order of the bits
                g(f"fbx_pkey[{j}][RT] = (u64){k.c};")
            else:
                self.pool_kw_bad = True  # Utf8 keys: the exact accounting fails loudly
        g("{ const u32 pb = __ballot_sync(0xFFFFFFFFu, joined != 0u);")
        g("if ((threadIdx.x & 31u) == 0u && pb) atomicAdd(&fbx_pjoin, (u32)__popc(pb)); }")

    def pool_lane(self, nd: NodeIR, a: V):
        """A device token node's lane size, len(str(v).encode()) or 0 (device.py:
        328-338, featureops.py:325-326), once per input plane."""
        if not nd.ref_pool:
            return
        plane = self.pool_plane_of[nd.name]
        if plane in self.pool_stored:
            return
        self.pool_stored.add(plane)
        g = self.g
        nul = f" && !{a.n}" if a.nullable else ""
        if self.ir.mode == "extract":
            g(f"if (inrange) {g.p('pool_sizes', 'u32*')}[{plane}ull * N + row] = "
              f"(alive{nul}) ? {a.c}.n : 0u;")
            return
        g(f"{{ const u32 psz = (joined{nul}) ? {a.c}.n : 0u; fbx_psz[{plane}][RT] = psz;")
        g("const u32 pws = __reduce_add_sync(0xFFFFFFFFu, psz);")
        g(f"if ((threadIdx.x & 31u) == 0u && pws) atomicAdd(&fbx_psum[{plane}], "
          "(unsigned long long)pws); }")

    def pool_tile_check(self):
        """Thread 0, after the tile's last barrier: the reference demand per layer is
        at most sum(lane sizes) + 127 per group; a tile whose bound may exceed its
        share of pool_bytes leaves its rows for fbx_pool_account."""
        g, ir = self.g, self.ir
        lpg, cap, spc, tr = ir.lanes_per_group, ir.pool_bytes, self.spc, self.tile_rows
        g("{")
        g(f"const u64 PG = ((u64)fbx_pjoin + {lpg - 1}ull) / {lpg}ull;")
        g("bool pneed = false;")
        layers: dict[int, list[int]] = {}
        for nd in self.pool_nodes:
            layers.setdefault(nd.layer, []).append(self.pool_plane_of[nd.name])
        for layer, planes in sorted(layers.items()):
            terms = " + ".join(f"(fbx_psum[{p}] ? fbx_psum[{p}] + 127ull * PG : 0ull)"
                               for p in planes)
            g(f"if (({terms}) * {spc}ull > {cap}ull) pneed = true;  // layer {layer}")
        g(f"const u32 ptile = tile - (u32){g.p('pool_tile0')};  // plane index (ring: launch-local)")
        g(f"{g.p('pool_flag', 'u8*')}[ptile] = (u8)pneed;")
        g("if (pneed) {")
        if self.pool_kw_bad:
            g(f"fbx::raise_err(ST, fbx::err_key(chunk, 4u, 0u, 0u, {ERR['pool_key']}u), 0ull);  // Utf8 join keys")
        g(f"{g.p('pool_chunk', 'u64*')}[ptile] = chunk;")
        g("atomicAdd((unsigned long long*)&ST->pool_flagged, 1ull);")
        g(f"const u64 PL = {g.p('pool_plane')}, PB = (u64)ptile * {tr}ull;")
        g(f"for (u32 r = 0; r < {tr}u; ++r) {{")
        g(f"{g.p('pool_joined', 'u8*')}[PB + r] = fbx_pjf[r];")
        for j in range(self.pool_kw):
            g(f"{g.p('pool_keys', 'u64*')}[{j}ull * PL + PB + r] = fbx_pkey[{j}][r];")
        for p in range(self.pool_ni):
            g(f"{g.p('pool_sizes', 'u32*')}[{p}ull * PL + PB + r] = fbx_psz[{p}][r];")
        g("}")
        g("}")
        g("}")

    # -- column access --------------------------------------------------------------
    def load_driver_column(self, name: str, kind: Kind) -> V:
        g = self.g
        t = self.kind_t(kind)
        v = V(t, f"d_{name}", True)
        nul = g.p(f"drv.{name}.nulls", "const u8*")
        self.decl(v)
        g(f"if (inrange) {{")
        g(f"{v.c}_n = fbx::null_bit({nul}, row);")
        if kind is Kind.INT64:
            g(f"{v.c} = fbx::ldg_u64({g.p(f'drv.{name}.data', 'const u64*')} + row);")
        elif kind is Kind.FLOAT32:
            g(f"{v.c} = fbx::f32_canon_bits(fbx::ldg_u32({g.p(f'drv.{name}.data', 'const u32*')}"
              f" + row));")
        else:
            offs = g.p(f"drv.{name}.offsets", "const u32*")
            data = g.p(f"drv.{name}.data", "const u8*")
            g(f"u32 o0 = fbx::ldg_u32({offs} + row), o1 = fbx::ldg_u32({offs} + row + 1);")
            if self.ir.stage_strings and name in self.staged:
                idx = self.staged.index(name)
                g(f"const u8* base = sm_span_ok[{idx}] ? (sm_span_buf[{idx}] - sm_span_lo[{idx}])"
                  f" : {data};")
                g(f"{v.c} = fbx::Str{{base + o0, o1 - o0}};")
            else:
                g(f"{v.c} = fbx::Str{{{data} + o0, o1 - o0}};")
        g("}")
        return v

    # -- JSON extraction ---------------------------------------------------------
    def json_source(self, view: ViewIR, src: V, exts: list, prefix: str, stage: str,
                    on_malformed: str) -> dict[str, V]:
        """Parse one JSON source; returns output column -> V."""
        g = self.g
        np_ = len(exts)
        if np_ > 8:
            raise UnsupportedOnDevice("more than 8 extractions from one JSON source")
        segs, offs, lens, nseg = b"", [], [], []
        for e in exts:
            parts = [p.encode("utf-8") for p in e.path.split(".")]
            if len(parts) > 8:
                raise UnsupportedOnDevice("JSON path deeper than 8 segments")
            o, ln = [], []
            for p in parts:
                o.append(len(segs))
                ln.append(len(p))
                segs += p
            offs += o + [0] * (8 - len(o))
            lens += ln + [0] * (8 - len(ln))
            nseg.append(len(parts))
            if e.kind is Kind.JSON:
                self.json_kind = True
        tag = g.fresh("jp")
        self.globals.append(f"__device__ const u8 {tag}_seg[] = {_c_bytes(segs)};")
        self.globals.append(f"__device__ const u16 {tag}_off[] = "
                            "{" + ",".join(map(str, offs)) + "};")
        self.globals.append(f"__device__ const u8 {tag}_len[] = "
                            "{" + ",".join(map(str, lens)) + "};")
        self.globals.append(f"__device__ const u8 {tag}_ns[] = "
                            "{" + ",".join(map(str, nseg)) + "};")
        km = f"{tag}_KM"
        cases = []
        for pi, e in enumerate(exts):
            for si, seg in enumerate(e.path.split(".")):
                b = seg.encode("utf-8")
                pre = int.from_bytes(b[:8].ljust(8, b"\0"), "little")
                cases.append(f"    case {pi * 8 + si}: return len == {len(b)}u && pre == "
                             f"0x{pre:016X}ull;")
        nsegs = ", ".join(str(len(e.path.split("."))) for e in exts)
        self.globals.append(
            f"struct {km} {{\n"
            f"  static FBX_DI u32 nseg(int p) {{ const u32 t[{np_}] = {{{nsegs}}}; return t[p]; }}\n"
            f"  static FBX_DI bool eq(int p, u32 sidx, u64 pre, u32 len) {{\n"
            f"    switch (p * 8 + (int)sidx) {{\n" + "\n".join(cases) +
            "\n    default: return false;\n    }\n  }\n};")
        leaf = g.fresh("leaf")
        g(f"fbx::JLeaf {leaf}[{np_}];")
        g(f"bool {leaf}_ok = false;")
        g(f"if (alive && !{src.n}) {{")
        g(f"u32 js = fbx::json_extract<{np_}, {km}>({src.c}, fbx::JPathSet{{{tag}_seg, {tag}_off, "
          f"{tag}_len, {tag}_ns}}, {leaf});")
        g(f"if (js == fbx::JS_OK) {{ {leaf}_ok = true; }}")
        g(f"else if (js == fbx::JS_MALFORMED) {{ {on_malformed} }}")
        g("else if (js == fbx::JS_BIGINT) {")
        self.row_error(stage, "json_bigint")
        g("} else {")
        self.row_error(stage, "json_deep")
        g("}")
        g("}")
        out = {}
        for pi, e in enumerate(exts):
            lf = f"{leaf}[{pi}]"
            if e.kind is Kind.UTF8:
                v = V("str", g.fresh(f"{prefix}x"), True, lone=True)
                self.decl(v)
                g(f"bool {v.c}_esc = {leaf}_ok && {lf}.type == fbx::J_STRING && {lf}.esc;")
                ptr = self.pool_alloc(f"({v.c}_esc && alive) ? ({lf}.end - {lf}.beg) : 0u")
                g(f"if (alive && {leaf}_ok && {lf}.type == fbx::J_STRING) {{")
                g(f"if (!{lf}.esc) {{ {v.c} = fbx::Str{{{src.c}.p + {lf}.beg, {lf}.end - {lf}.beg}};"
                  f" {v.c}_n = false; }}")
                g(f"else if ({ptr}) {{ u32 lone = 0; u32 L = fbx::j_unescape({src.c}.p, {lf}.beg, "
                  f"{lf}.end, {ptr}, &lone); {v.c} = fbx::Str{{{ptr}, L}}; {v.c}_n = false; "
                  f"{v.c}_l = lone != 0; }}")
                g("}")
            elif e.kind is Kind.INT64:
                v = V("i64", g.fresh(f"{prefix}x"), True)
                self.decl(v)
                g(f"if (alive && {leaf}_ok && {lf}.type == fbx::J_INT) {{")
                g(f"i64 t; if (fbx::j_to_i64({src.c}.p, {lf}.beg, {lf}.end, &t)) "
                  f"{{ {v.c} = (u64)t; {v.c}_n = false; }}")
                g("}")
            elif e.kind is Kind.JSON:
                # json.dumps(value, sort_keys=True, separators=(",", ":")): measured,
                # allocated from the bump pool, written (viewpipe.py:266-267)
                v = V("str", g.fresh(f"{prefix}x"), True)
                self.decl(v)
                jl = g.fresh("jl")
                has = (f"alive && {leaf}_ok && {lf}.type != fbx::J_MISSING && "
                       f"{lf}.type != fbx::J_NULL")
                g(f"u32 {jl} = ({has}) ? fbx::json_canon({src.c}.p, {src.c}.n, {lf}, nullptr) : 0u;")
                g(f"if ({jl} == ~0u) {{")
                self.row_error(stage, "float_slow")
                g("}")
                ptr = self.pool_alloc(f"({has} && {jl} != ~0u) ? {jl} : 0u")
                g(f"if (({has}) && {jl} != ~0u && {ptr}) {{ fbx::json_canon({src.c}.p, {src.c}.n, {lf}, "
                  f"{ptr}); {v.c} = fbx::Str{{{ptr}, {jl}}}; {v.c}_n = false; }}")
            else:  # FLOAT32
                v = V("f32", g.fresh(f"{prefix}x"), True)
                self.decl(v)
                g(f"if (alive && {leaf}_ok) {{")
                g(f"u32 bits = 0; u32 fs = fbx::j_to_f32({src.c}.p, {lf}, &bits);")
                g(f"if (fs == 0u) {{ {v.c} = bits; {v.c}_n = false; }}")
                g(f"else if (fs == 2u) {{")
                self.row_error(stage, "float_overflow")
                g("} else if (fs == 3u) {")
                self.row_error(stage, "float_slow")
                g("}")
                g("}")
            out[e.output] = v
        return out

    # -- filter -------------------------------------------------------------------------
    def filter_expr(self, expr, vals: Mapping[str, V]) -> str:
        if isinstance(expr, BoolExpr):
            j = " && " if expr.kind == "and" else " || "
            return "(" + j.join(self.filter_expr(p, vals) for p in expr.parts) + ")"
        assert isinstance(expr, Comparison)
        v = vals[expr.column]
        nn = f"!{v.n}" if v.nullable else "true"
        op, lit = expr.op, expr.literal
        if v.t == "str":
            b = lit.encode("utf-8", "surrogatepass")
            k = self.g.const(b)
            return f"({nn} && (fbx::str_cmp({v.c}, {k}, {len(b)}u) {op} 0))"
        if v.t == "f32":
            bits = _f32_bits(float(lit))
            return f"({nn} && (__uint_as_float({v.c}) {op} __uint_as_float({bits}u)))"
        # Int64 column vs int / float literal: exact Python semantics
        x = f"((i64){v.c})"
        if isinstance(lit, float):
            if lit != lit:
                return "false" if op != "!=" else nn
            fr = Fraction(lit)
        else:
            fr = Fraction(lit)
        return f"({nn} && {self._int_cmp(x, op, fr)})"

    def _int_cmp(self, x: str, op: str, fr: Fraction) -> str:
        import math
        lo, hi = INT64_MIN, INT64_MAX
        if op in ("==", "!="):
            if fr.denominator != 1 or not lo <= fr.numerator <= hi:
                return "true" if op == "!=" else "false"
            return f"({x} {op} {_i64(fr.numerator)})"
        if op in ("<", ">="):
            c = math.ceil(fr)  # x < fr  <=>  x < ceil(fr)
            if c > hi:
                return "true" if op == "<" else "false"
            if c <= lo:
                return "false" if op == "<" else "true"
            return f"({x} {op} {_i64(c)})"
        c = math.floor(fr)  # x <= fr <=> x <= floor(fr) ; x > fr <=> x > floor(fr)
        if c >= hi:
            return "true" if op == "<=" else "false"
        if c < lo:
            return "false" if op == "<=" else "true"
        return f"({x} {op} {_i64(c)})"

    # -- clean ---------------------------------------------------------------------------
    def clean_view(self, view: ViewIR, prefix: str, loader, stage: str, used: set[str],
                   count_prefix: str) -> dict[str, V]:
        """Cleaned values of one row: loads, JSON extraction, fills, filter."""
        g = self.g
        ckinds = view.cleaned_kinds()
        raw: dict[str, V] = {}
        sources = sorted({e.source for e in view.extractions})
        need = set(used) | set(sources)
        if view.filter is not None:
            need |= _filter_columns(view.filter)
        for name, kind in view.kinds.items():
            if name in need:
                raw[name] = loader(name, kind)
        vals: dict[str, V] = dict(raw)
        if sources:
            g(f"bool {prefix}malformed = false;")
        for s in sources:
            exts = [e for e in view.extractions if e.source == s]
            vals.update(self.json_source(view, raw[s], exts, prefix, stage,
                                         f"{prefix}malformed = true;"))
        if sources:
            g(f"if (alive && {prefix}malformed) {{ alive = false; {count_prefix}malformed += 1u; }}")
        ext_out = {e.output for e in view.extractions}
        for name, fill in view.fills.items():
            if name in ext_out or name not in vals:
                continue  # an extraction output replaces the filled column
            vals[name] = self.apply_fill(vals[name], view.kinds[name], fill)
        if view.filter is not None:
            cond = self.filter_expr(view.filter, vals)
            g(f"if (alive && !({cond})) {{ alive = false; {count_prefix}filtered += 1u; }}")
        return {k: v for k, v in vals.items() if k in ckinds}

    def apply_fill(self, v: V, kind: Kind, fill) -> V:
        g = self.g
        out = V(v.t, g.fresh("f"), False, v.lone)
        if kind is Kind.INT64:
            if not INT64_MIN <= int(fill) <= INT64_MAX:
                raise UnsupportedOnDevice("Int64 fill value outside int64")
            g(f"u64 {out.c} = {v.n} ? {_u64(int(fill))} : {v.c};")
        elif kind is Kind.FLOAT32:
            g(f"u32 {out.c} = {v.n} ? {_f32_bits(float(fill))}u : {v.c};")
        else:
            b = str(fill).encode("utf-8", "surrogatepass")
            k = g.const(b)
            g(f"fbx::Str {out.c} = {v.n} ? fbx::Str{{{k}, {len(b)}u}} : {v.c};")
        if v.lone:
            g(f"bool {out.c}_l = !{v.n} && {v.l};")
        return out

    # -- join keys ----------------------------------------------------------------------
    def key_hash(self, vals: Sequence[V], kinds: Sequence[Kind], out: str):
        """Table hash of a join key (identical on the build and probe sides;
        equality is always re-checked on the canonical values)."""
        g = self.g
        g(f"u64 {out};")
        g("{")
        g("u64 h = 0x243F6A8885A308D3ull;")
        for v, k in zip(vals, kinds):
            if k is Kind.INT64:
                g(f"h = fbx::tbl_hash_u64(h, {v.c});")
            elif k is Kind.FLOAT32:
                g(f"h = fbx::tbl_hash_u64(h, (u64){v.c} | (1ull << 40));")
            else:
                g(f"h = fbx::tbl_hash_bytes(h, {v.c}.p, {v.c}.n);")
        g(f"{out} = fbx::table_tag(h);")
        g("}")

    def key_eq(self, a: Sequence[V], b: Sequence[V]) -> str:
        terms = []
        for x, y in zip(a, b):
            if x.t == "str":
                terms.append(f"fbx::str_eq({x.c}, {y.c})")
            else:
                terms.append(f"({x.c} == {y.c})")
        return " && ".join(terms) if terms else "true"

    # -- side views ----------------------------------------------------------------------
    def side_loader(self, k: int, row: str):
        g = self.g

        def load(name: str, kind: Kind) -> V:
            t = self.kind_t(kind)
            v = V(t, g.fresh(f"s{k}_{name}_"), True)
            self.decl(v)
            nul = g.p(f"side{k}.{name}.nulls", "const u8*")
            pre = self.prefetched.pop((k, name, row), None)
            if pre is not None:  # raw words loaded before the DAG: only the arithmetic here
                g(f"{v.c}_n = ({pre}_nb >> ({row} & 7u)) & 1u;")
                if kind is Kind.INT64:
                    g(f"{v.c} = {pre}_v;")
                elif kind is Kind.FLOAT32:
                    g(f"{v.c} = fbx::f32_canon_bits({pre}_v);")
                else:
                    data = g.p(f"side{k}.{name}.data", "const u8*")
                    g(f"{v.c} = fbx::Str{{{data} + {pre}_o0, {pre}_o1 - {pre}_o0}};")
                return v
            g(f"{v.c}_n = fbx::null_bit({nul}, {row});")
            if kind is Kind.INT64:
                g(f"{v.c} = fbx::ldg_u64({g.p(f'side{k}.{name}.data', 'const u64*')} + {row});")
            elif kind is Kind.FLOAT32:
                g(f"{v.c} = fbx::f32_canon_bits(fbx::ldg_u32("
                  f"{g.p(f'side{k}.{name}.data', 'const u32*')} + {row}));")
            else:
                offs = g.p(f"side{k}.{name}.offsets", "const u32*")
                data = g.p(f"side{k}.{name}.data", "const u8*")
                g(f"{{ u32 o0 = fbx::ldg_u32({offs} + {row}), o1 = fbx::ldg_u32({offs} + {row} + 1);"
                  f" {v.c} = fbx::Str{{{data} + o0, o1 - o0}}; }}")
            return v
        return load

    def prefetch_side_column(self, k: int, view: ViewIR, name: str, row: str):
        """Issue the raw loads of a joined column before the DAG (no arithmetic on
        them, so no warp waits here); the first reader does the rest."""
        g = self.g
        ext = {e.output for e in view.extractions}
        if name in ext or name not in view.kinds or (k, name, row) in self.prefetched:
            return
        kind = view.kinds[name]
        pre = g.fresh(f"pg{k}_")
        nul = g.p(f"side{k}.{name}.nulls", "const u8*")
        g(f"const u32 {pre}_nb = fbx::ldg_u8({nul} + ({row} >> 3));")
        if kind is Kind.INT64:
            g(f"const u64 {pre}_v = fbx::ldg_u64({g.p(f'side{k}.{name}.data', 'const u64*')} + {row});")
        elif kind is Kind.FLOAT32:
            g(f"const u32 {pre}_v = fbx::ldg_u32({g.p(f'side{k}.{name}.data', 'const u32*')} + {row});")
        else:
            offs = g.p(f"side{k}.{name}.offsets", "const u32*")
            g(f"const u32 {pre}_o0 = fbx::ldg_u32({offs} + {row}), {pre}_o1 = "
              f"fbx::ldg_u32({offs} + {row} + 1);")
        self.prefetched[(k, name, row)] = pre

    def side_value(self, k: int, view: ViewIR, name: str, row: str) -> V:
        """Cleaned value of side column `name` at side row `row` (gather)."""
        g = self.g
        ext = {e.output: e for e in view.extractions}
        if name in ext:
            e = ext[name]
            t = self.kind_t(e.kind)
            v = V(t, g.fresh(f"s{k}e_"), True, lone=(t == "str"))
            self.decl(v)
            if t == "str":
                g(f"{{ u64 pp = fbx::ldg_u64({g.p(f'side{k}.ext.{name}.ptr', 'const u64*')} + {row});"
                  f" u32 ll = fbx::ldg_u32({g.p(f'side{k}.ext.{name}.len', 'const u32*')} + {row});")
                g(f"  {v.c}_n = (ll == 0xFFFFFFFFu); {v.c}_l = (ll & 0x80000000u) != 0u && !{v.c}_n;"
                  f" {v.c} = fbx::Str{{(const u8*)pp, {v.c}_n ? 0u : (ll & 0x7FFFFFFFu)}}; }}")
            else:
                arr = g.p(f"side{k}.ext.{name}.val", "const u64*")
                g(f"{{ u64 w = fbx::ldg_u64({arr} + {row}); "
                  f"u8 nn = fbx::ldg_u8({g.p(f'side{k}.ext.{name}.null', 'const u8*')} + {row});"
                  f" {v.c} = ({'u32' if t == 'f32' else 'u64'})w; {v.c}_n = nn != 0; }}")
            return v
        v = self.side_loader(k, row)(name, view.kinds[name])
        if name in view.fills:
            v = self.apply_fill(v, view.kinds[name], view.fills[name])
        return v

    # ------------------------------------------------------------------------------------
    def side_prep_kernel(self, k: int, view: ViewIR, is_basic: bool) -> str:
        """Index one side view (or the basic view) into its HBM join table."""
        g = self.g
        name = f"fbx_side_prep_{k}"
        # a device function: every view's index build runs in ONE launch
        # (fbx_side_prep_all dispatches CTA ranges), so the small side views
        # build concurrently with the basic view instead of one after another
        g(f"static __device__ __forceinline__ void {name}(const fbx_params& P, const u32 BID, "
          "const u32 NBLK) {")
        g("fbx_state* ST = (fbx_state*)P.v[0];")
        g(f"const u64 n = {g.p(f'side{k}.rows')};")
        g(f"fbx::Slot* TBL = {g.p(f'side{k}.table', 'fbx::Slot*')};")
        g(f"const u64 MASK = {g.p(f'side{k}.mask')};")
        g(f"u8* POOL = {g.p('side_pool', 'u8*')}; const u64 POOL_CAP = {g.p('side_pool_cap')};")
        g("u32 nmal = 0, nfilt = 0, nidx = 0;")
        g("const u64 chunk = 0;")
        g("for (u64 base = (u64)BID * 256u; base < n; base += (u64)NBLK * 256u) {")
        g("const u64 srow = base + threadIdx.x;")
        g("bool alive = srow < n;")
        g("const u64 row = alive ? srow : 0ull;")
        g("__shared__ struct { fbx::BlockScanU32<256> scan; u64 pool_base; } sm;")
        g("constexpr int NT = 256;")
        g(f"u32 CUR_STAGE = {STAGE['prepare']}u, CUR_LAYER = 0u, CUR_RANK = 0u;")
        g("u32 malformed = 0, filtered = 0;")
        ckinds = view.cleaned_kinds()
        loader = self.side_loader(k, "row")
        used = set(view.keys)
        vals = self.clean_view(view, f"sp{k}_", loader, "prepare", used, "")
        g("nmal += malformed; nfilt += filtered;")
        # store extraction outputs for the gather side
        for e in view.extractions:
            v = vals[e.output]
            if v.t == "str":
                g(f"if (srow < n) {{ {g.p(f'side{k}.ext.{e.output}.ptr', 'u64*')}[row] = (u64){v.c}.p;"
                  f" {g.p(f'side{k}.ext.{e.output}.len', 'u32*')}[row] = (!alive || {v.n}) ? 0xFFFFFFFFu"
                  f" : ({v.c}.n | ({v.l} ? 0x80000000u : 0u)); }}")
            else:
                g(f"if (srow < n) {{ {g.p(f'side{k}.ext.{e.output}.val', 'u64*')}[row] = (u64){v.c};"
                  f" {g.p(f'side{k}.ext.{e.output}.null', 'u8*')}[row] = (!alive || {v.n}) ? 1 : 0; }}")
        keys = [vals[c] for c in view.keys]
        kk = [ckinds[c] for c in view.keys]
        null_any = " || ".join(v.n for v in keys if v.nullable) or "false"
        lone_any = " || ".join(v.l for v in keys if v.lone) or "false"
        g(f"if (alive && ({lone_any}) && !({null_any})) {{")
        self.row_error("prepare", "encode")
        g("}")
        g(f"if (alive && !({null_any})) {{")
        self.key_hash(keys, kk, "tag")
        if self.int_keyed(k):
            if is_basic:  # check_unique_ids over the basic view (pipeline.py:975-980)
                g(f"if (fbx::islot_insert((fbx::ISlot*)TBL, MASK, tag, (u64){keys[0].c}, (u32)row))")
                g(f"fbx::raise_err(ST, fbx::err_key(0ull, {STAGE['prepare']}u, 0u, 0u, "
                  f"{ERR['basic_dup']}u), (u64){keys[0].c});")
                g("++nidx;")
            else:
                g(f"fbx::islot_insert((fbx::ISlot*)TBL, MASK, tag, (u64){keys[0].c}, (u32)row); ++nidx;")
            g("}")
            g("}")
            g("fbx::block_side_counts(ST, nmal, nfilt, nidx);")
            g("}")
            return name
        g("u64 i = tag & MASK;")
        g("while (true) {")
        g("unsigned long long old = atomicCAS((unsigned long long*)&TBL[i].tag, 0ull, "
          "(unsigned long long)tag);")
        g("if (old == 0ull) { TBL[i].ref = (u32)row; __threadfence(); "
          "atomicExch(&TBL[i].aux, 1u); ++nidx; break; }")
        g("if (old == tag) {")
        g("u32 c; do { c = *((volatile u32*)&TBL[i].aux); } while (c == 0u);")
        g("const u64 other = *((volatile u32*)&TBL[i].ref);")
        other = [self.side_value(k, view, c, "other") for c in view.keys]
        g(f"if ({self.key_eq(keys, other)}) {{ atomicAdd(&TBL[i].aux, 1u); ++nidx; break; }}")
        g("}")
        g("i = (i + 1) & MASK;")
        g("}")
        g("}")
        g("}")
        g("fbx::block_side_counts(ST, nmal, nfilt, nidx);")
        g("}")
        return name

    def clean_rows_kernel(self, view: ViewIR) -> str:
        """``clean_views`` of a whole view (viewpipe.py:334-431), row-aligned, for
        the staged mode: per row the keep flag (not malformed, passes the filter)
        and every cleaned column -- fills applied, JSON extraction outputs coerced
        -- as value (Int64 / Float32) or pointer + length (Utf8 / Json), and a
        null byte (null slots hold 0 / the empty string).  The host compacts the kept rows into the
        cleaned view's FBXC image (fbx_select_rows / fbx_take / fbx_pack_nulls).
        A cleaned string holding a lone surrogate cannot be written as UTF-8:
        the staged clean stage fails with UnicodeEncodeError, as the reference's
        writer does."""
        g = self.g
        k = 0
        name = "fbx_clean_rows"
        g(f'extern "C" __global__ void __launch_bounds__(256) {name}(const fbx_params P) {{')
        g("fbx_state* ST = (fbx_state*)P.v[0];")
        g(f"const u64 n = {g.p('side0.rows')};")
        g(f"u8* POOL = {g.p('side_pool', 'u8*')}; const u64 POOL_CAP = {g.p('side_pool_cap')};")
        g(f"u8* KEEP = {g.p('clean.keep', 'u8*')};")
        g("u32 nmal = 0, nfilt = 0;")
        g("const u64 chunk = 0;")
        g("for (u64 base = (u64)blockIdx.x * 256u; base < n; base += (u64)gridDim.x * 256u) {")
        g("const u64 srow = base + threadIdx.x;")
        g("bool alive = srow < n;")
        g("const u64 row = alive ? srow : 0ull;")
        g("__shared__ struct { fbx::BlockScanU32<256> scan; u64 pool_base; } sm;")
        g("constexpr int NT = 256;")
        g(f"u32 CUR_STAGE = {STAGE['clean']}u, CUR_LAYER = 0u, CUR_RANK = 0u;")
        g("u32 malformed = 0, filtered = 0;")
        ckinds = view.cleaned_kinds()
        loader = self.side_loader(k, "row")
        vals = self.clean_view(view, "cl_", loader, "clean", set(ckinds), "")
        g("nmal += malformed; nfilt += filtered;")
        g("if (srow < n) {")
        g("KEEP[row] = alive ? 1u : 0u;")
        for c, kind in ckinds.items():
            v = vals[c]
            if v.t == "str":
                if v.lone:
                    g(f"if (alive && !{v.n} && {v.l}) {{")
                    self.row_error("clean", "encode")
                    g("}")
                g(f"{g.p(f'clean.{c}.ptr', 'u64*')}[row] = (u64){v.c}.p;")
                g(f"{g.p(f'clean.{c}.len', 'u32*')}[row] = {v.n} ? 0u : {v.c}.n;")
            else:  # a null slot holds 0, as the reference's Column.build writes it
                w = "u32" if kind is Kind.FLOAT32 else "u64"
                g(f"(({w}*){g.p(f'clean.{c}.val', 'u64*')})[row] = {v.n} ? ({w})0 : ({w}){v.c};")
            g(f"{g.p(f'clean.{c}.null', 'u8*')}[row] = {v.n} ? 1u : 0u;")
        g("}")
        g("}")
        g("fbx::block_side_counts(ST, nmal, nfilt, 0u);")
        g("}")
        return name

    def side_prep_dispatch(self, nviews: int):
        """fbx_side_prep_all: CTA b runs the index build of the view whose range
        [start_k, start_k + grid_k) holds b (side{k}.grid, set by the engine)."""
        g = self.g
        g('extern "C" __global__ void __launch_bounds__(256) fbx_side_prep_all(const fbx_params P) {')
        g("u32 b = blockIdx.x;")
        for k in range(nviews):
            g(f"{{ const u32 gk = (u32){g.p(f'side{k}.grid')};")
            g(f"if (b < gk) {{ fbx_side_prep_{k}(P, b, gk); return; }}")
            g("b -= gk; }")
        g("}")

    # -- operator library --------------------------------------------------------------
    def node_code(self, nd: NodeIR, args: list[V]) -> V:
        fn = nd.fn
        g = self.g
        stage_ctx = f"CUR_STAGE = {STAGE['extract']}u; CUR_LAYER = {nd.layer}u; CUR_RANK = {nd.rank}u;"
        g(f"// node {nd.name} [{fn.spec}] layer {nd.layer}")
        g(stage_ctx)
        err = lambda code: self.row_error("extract", code, nd.layer, nd.rank)  # noqa: E731
        op = fn.op
        if op == "id":
            return args[0]
        if op in ("mix", "fold"):
            a = args[0]
            if a.t in ("str", "f32"):
                out = V("u64", g.fresh("n"), True)
                self.decl(out)
                g(f"if (alive && !{a.n}) {{")
                err("type")
                g("}")
                return out
            t = "u64" if (op == "mix" or a.t == "u64") else "i64"
            out = V(t, g.fresh("n"), a.nullable)
            if op == "mix":
                g(f"u64 {out.c} = fbx::fnv_mix({a.c});")
            elif a.t == "u64":
                g(f"u64 {out.c} = ({a.c} >> 32) ^ ({a.c} & 0xFFFFFFFFull);")
            else:
                g(f"u64 {out.c} = (u64)(((i64){a.c}) >> 32) ^ ({a.c} & 0xFFFFFFFFull);")
            if a.nullable:
                g(f"bool {out.c}_n = {a.n};")
            return out
        if op == "token" and nd.name in getattr(self, "token_groups", {}) and args[0].t == "str":
            (col, delim), fields = self.token_groups[nd.name]
            gk = f"{col}|{delim}"
            a = args[0]
            self.pool_lane(nd, a)
            if gk not in self.token_done:
                base = g.fresh("tg")
                kk = len(fields)
                g(f"fbx::Str {base}[{kk}] = {{}};")
                g(f"{{ const u32 want[{kk}] = {{{', '.join(map(str, fields))}}};")
                cond = f"alive && !{a.n}" if a.nullable else "alive"
                g(f"if ({cond}) fbx::str_tokens<{kk}>({a.c}, {ord(delim)}u, want, {base}); }}")
                self.token_done[gk] = V("str", base, a.nullable, a.lone)
            grp = self.token_done[gk]
            out = V("str", g.fresh("n"), a.nullable, a.lone)
            g(f"fbx::Str {out.c} = {grp.c}[{fields.index(fn.index)}];")
            if out.nullable:
                g(f"bool {out.c}_n = {a.n} || !alive;")
            if out.lone:
                g(f"bool {out.c}_l = {a.l};")
                g(f"if (alive && !{out.n} && {out.l}) {{")
                err("encode")
                g("}")
            return out
        if op == "token":
            a = self.as_str(args[0], fn.spec)
            self.pool_lane(nd, a)
            if a.lower and fn.delim.isascii() and fn.delim.isalpha():
                a = self.materialize(a)  # a letter delimiter must see lowered bytes
            out = V("str", g.fresh("n"), a.nullable, a.lone, a.lower)
            self.decl(out)
            cond = f"alive && !{a.n}" if a.nullable else "alive"
            g(f"if ({cond}) {{")
            if len(fn.delim.encode("utf-8")) != 1:
                err("value")
            else:
                if a.lone:
                    g(f"if ({a.l}) {{")
                    err("encode")
                    g("}")
                g(f"{out.c} = fbx::str_token({a.c}, {ord(fn.delim)}u, {fn.index}u);")
                if out.nullable:
                    g(f"{out.c}_n = false;")
                if out.lone:
                    g(f"{out.c}_l = {a.l};")
            g("}")
            return out
        if op == "trim":
            a = self.as_str(args[0], fn.spec)
            out = V("str", g.fresh("n"), a.nullable, a.lone, a.lower)
            self.decl(out)
            cond = f"alive && !{a.n}" if a.nullable else "alive"
            g(f"if ({cond}) {{ {out.c} = fbx::str_trim({a.c});"
              + (f" {out.c}_n = false;" if out.nullable else "")
              + (f" {out.c}_l = {a.l};" if out.lone else "") + " }")
            return out
        if op == "lower":
            a = self.as_str(args[0], fn.spec)
            if a.lower:
                return a  # str.lower is idempotent (checked over all code points)
            cls = g.fresh("lc")
            cond = f"alive && !{a.n}" if a.nullable else "alive"
            g(f"u32 {cls} = ({cond}) ? fbx::str_lower_class({a.c}) : 0u;")
            # non-ASCII rows: full Unicode lower() materialised from the pool;
            # ASCII rows stay a lazy view, lowercased by their consumers
            sz = g.fresh("lz")
            g(f"const u32 {sz} = ({cls} == 2u) ? fbx::unicode_lower({a.c}, nullptr) : 0u;")
            ptr = self.pool_alloc(sz)
            out = V("str", g.fresh("n"), a.nullable, a.lone, lower=True)
            g(f"fbx::Str {out.c} = {a.c};")
            if a.nullable:
                g(f"bool {out.c}_n = {a.n};")
            if a.lone:
                g(f"bool {out.c}_l = {a.l};")
            g(f"if ({cls} == 2u && ({ptr} || {sz} == 0u)) {{ fbx::unicode_lower({a.c}, {ptr});"
              f" {out.c} = fbx::Str{{{ptr}, {sz}}}; }}")
            return out
        if op == "lookup":
            a = args[0]
            out = V("u64", g.fresh("n"), False)
            ti = self.ir.tables[fn.table]
            dflt = self.ir.table_defaults[fn.table]
            g(f"u64 {out.c} = {_u64(dflt)};")
            s = self.materialize(self.as_str(a, fn.spec))
            cond = f"alive && !{s.n}" if s.nullable else "alive"
            lone = f" && !{s.l}" if s.lone else ""
            g(f"if ({cond}{lone}) {{")
            if nd.name in self.dict_pf:
                _, _, off = self.dict_pf[nd.name]
                tag = f"dpf_{nd.name.replace('.', '_')}"
                g("fbx::cp_async_wait_all();")
                g(f"{out.c} = fbx::dict_lookup_pf({g.p(f'dict{ti}.slots', 'const fbx::Slot*')}, "
                  f"{g.p(f'dict{ti}.mask')}, {g.p(f'dict{ti}.keys', 'const u8*')}, {s.c}, "
                  f"{_u64(dflt)}, {tag}, (const fbx::Slot*)(dyn_smem + {off}u + 32u * threadIdx.x));")
            else:
                g(f"{out.c} = fbx::dict_lookup({g.p(f'dict{ti}.slots', 'const fbx::Slot*')}, "
                  f"{g.p(f'dict{ti}.mask')}, {g.p(f'dict{ti}.keys', 'const u8*')}, {s.c}, "
                  f"{_u64(dflt)});")
            g("}")
            return out
        if op == "hash":
            nullable = any(a.nullable for a in args)
            out = V("u64", g.fresh("n"), nullable)
            self.decl(out)
            nulls = [a.n for a in args if a.nullable]
            cond = "alive" + "".join(f" && !{x}" for x in nulls)
            lones = [a.l for a in args if a.t == "str" and a.lone]
            if lones:
                g(f"if (({cond}) && ({' || '.join(lones)})) {{")
                err("encode")
                g("}")
            # hashed unconditionally: a dead / null row's value is never read, and
            # every input is a valid (possibly empty) view -- no reconvergence
            # scaffolding around the FNV loops
            h0 = fnv1a64(fn.slot.to_bytes(2, "big"))
            g("{")
            g(f"fbx::Fnv h({_u64(h0)});")
            for i, a in enumerate(args):
                if i:
                    g("h.byte(0u);")
                if a.t == "str":
                    g(f"h.bytes{'_lower' if a.lower else ''}({a.c}.p, {a.c}.n);")
                elif a.t == "f32":
                    g(f"h.word_be({a.c});")
                else:
                    g(f"h.u64_be_int({a.c});")
            g(f"{out.c} = h.value();")
            g("}")
            if nullable:
                g(f"{out.c}_n = !({cond});")
            return out
        if op == "concat":
            parts = [self.as_str(a, fn.spec) for a in args]
            nullable = any(p.nullable for p in parts)
            lone = any(p.lone for p in parts)
            if len(parts) == 1:
                return parts[0]  # sep.join([s]) == s: a view
            out = V("str", g.fresh("n"), nullable, lone)
            self.decl(out)
            sep = fn.sep.encode("utf-8", "surrogatepass")
            nulls = [p.n for p in parts if p.nullable]
            ok = g.fresh("ok")
            g(f"bool {ok} = alive" + "".join(f" && !{x}" for x in nulls) + ";")
            total = " + ".join(f"{p.c}.n" for p in parts) + f" + {len(sep) * (len(parts) - 1)}u"
            ptr = self.pool_alloc(f"{ok} ? ({total}) : 0u")
            g(f"if ({ok} && {ptr}) {{")
            g(f"u8* d = {ptr};")
            k = g.const(sep) if sep else None
            for i, p in enumerate(parts):
                if i and sep:
                    g(f"for (u32 q = 0; q < {len(sep)}u; ++q) d[q] = {k}[q]; d += {len(sep)}u;")
                g(f"fbx::str_copy{'_lower' if p.lower else ''}(d, {p.c}); d += {p.c}.n;")
            g(f"{out.c} = fbx::Str{{{ptr}, {total}}};")
            if nullable:
                g(f"{out.c}_n = false;")
            if lone:
                g(f"{out.c}_l = " + " || ".join(p.l for p in parts if p.lone) + ";")
            g("}")
            return out
        raise UnsupportedOnDevice(f"function {fn.spec!r}")

    # ------------------------------------------------------------------------------------
    def probe(self, k: int, view: ViewIR, keys: list[V], kinds: list[Kind], row_var: str,
              cnt_var: str, pre: str | None):
        """Emit a hash-table probe of side table k; sets row_var / cnt_var.

        With ``pre`` the first slot (tag/ref/aux) was loaded in the prologue."""
        g = self.g
        if self.int_keyed(k):
            g(f"const fbx::ISlot* T = {g.p(f'side{k}.table', 'const fbx::ISlot*')};")
            g(f"const u64 MASK = {g.p(f'side{k}.mask')};")
            if pre:
                g(f"u64 tag = {pre}_tag;")
            else:
                self.key_hash(keys, kinds, "tag")
            g("u64 i = tag & MASK;")
            if pre and k in self.pf_slot:
                g("fbx::cp_async_wait_all();")
                g(f"fbx::ISlot s = *(const fbx::ISlot*)(dyn_smem + SPAN_BUDGET + "
                  f"{16 * self.nt * self.pf_slot[k]}u + 16u * threadIdx.x);")
            else:
                g("fbx::ISlot s = fbx::islot_ld(T + i);")
            g("while (true) {")
            g("if (s.aux == 0u) break;")
            g(f"if (s.key == (u64){keys[0].c}) {{ {cnt_var} = s.aux; {row_var} = s.ref; break; }}")
            g("i = (i + 1) & MASK;")
            g("s = fbx::islot_ld(T + i);")
            g("}")
            return
        g(f"const fbx::Slot* T = {g.p(f'side{k}.table', 'const fbx::Slot*')};")
        g(f"const u64 MASK = {g.p(f'side{k}.mask')};")
        if pre:
            g(f"u64 tag = {pre}_tag;")
        else:
            self.key_hash(keys, kinds, "tag")
        g("u64 i = tag & MASK;")
        g("bool first = true;")
        g("while (true) {")
        if pre:
            g(f"u64 t = first ? {pre}_t : __ldg(&T[i].tag);")
        else:
            g("u64 t = __ldg(&T[i].tag);")
        g("if (t == 0ull) break;")
        g("if (t == tag) {")
        if pre:
            g(f"const u64 other = first ? (u64){pre}_ref : (u64)__ldg(&T[i].ref);")
        else:
            g("const u64 other = __ldg(&T[i].ref);")
        other = [self.side_value(k, view, c, "other") for c in view.keys]
        if pre:
            g(f"if ({self.key_eq(keys, other)}) {{ {cnt_var} = first ? {pre}_aux : __ldg(&T[i].aux);"
              f" {row_var} = other; break; }}")
        else:
            g(f"if ({self.key_eq(keys, other)}) {{ {cnt_var} = __ldg(&T[i].aux); {row_var} = other;"
              " break; }")
        g("}")
        g("first = false;")
        g("i = (i + 1) & MASK;")
        g("}")

    def int_keyed(self, k: int) -> bool:
        """Table k is keyed by one Int64 column on both sides: 16-B ISlot layout
        (key stored in the slot, no key gather on the probe)."""
        ir = self.ir
        if k < len(ir.sides):
            sv = ir.sides[k]
            if len(ir.join_keys) != 1 or len(sv.keys) != 1:
                return False
            dk = ir.driver.cleaned_kinds()
            return (dk.get(ir.join_keys[0]) is Kind.INT64
                    and sv.cleaned_kinds().get(sv.keys[0]) is Kind.INT64)
        bv = ir.basic
        return (bv is not None and len(bv.keys) == 1
                and bv.cleaned_kinds().get(bv.keys[0]) is Kind.INT64)

    def raw_key_cols(self, cols) -> bool:
        drv = self.ir.driver
        needed = self.driver_needed()
        ext_out = {e.output for e in drv.extractions}
        return all(c in drv.kinds and c in needed and c not in ext_out and c not in drv.fills
                   for c in cols)

    def smem_prefetch_tables(self) -> list[int]:
        """Int-keyed tables whose first probe slot is copied to shared memory
        (cp.async) in the prologue: the probe then never waits on HBM."""
        ir = self.ir
        out = [k for k in range(len(ir.sides))
               if self.int_keyed(k) and self.raw_key_cols(ir.join_keys)]
        bk = len(ir.sides)
        if ir.basic is not None and self.int_keyed(bk) and self.raw_key_cols([ir.instance_column]):
            out.append(bk)
        return out

    def staged_columns(self) -> list[str]:
        ir = self.ir
        drv = ir.driver
        needed = self.driver_needed()
        return ([c for c, k in drv.kinds.items() if k.var_length and c in needed]
                if ir.stage_strings else [])[:16]

    def dict_prefetch_nodes(self) -> list[tuple[str, str, int]]:
        """lookup pre-ops keyed directly by a (filled) driver string column: their
        first dictionary slot is copied to shared memory right after the span
        staging lands, so the probe does not wait on HBM (query_dict: 1e7 keys)."""
        ir = self.ir
        drv = ir.driver
        ext_out = {e.output for e in drv.extractions}
        out = []
        for nd in ir.nodes:
            if nd.role != "pre" or nd.fn.op != "lookup" or len(nd.inputs) != 1:
                continue
            c = nd.inputs[0]
            k = drv.kinds.get(c)
            if (k not in (Kind.UTF8, Kind.JSON) or c in ext_out or c in ir.producer
                    or c not in self.staged):
                continue
            out.append((nd.name, c, ir.tables[nd.fn.table]))
        return out

    def prefetch(self, k: int, keys: list[V], kinds: list[Kind], name: str) -> str:
        """Prologue: hash the raw key and load the first probe slot."""
        g = self.g
        if k in self.pf_slot:
            g(f"u64 {name}_tag = 0;")
        else:
            g(f"u64 {name}_tag = 0, {name}_t = 0; u32 {name}_ref = 0, {name}_aux = 0;")
        nn = " && ".join(f"!{v.n}" for v in keys if v.nullable) or "true"
        g(f"if (inrange && {nn}) {{")
        self.key_hash(keys, kinds, "tg")
        g(f"{name}_tag = tg;")
        if k in self.pf_slot:
            g(f"const fbx::ISlot* T = {g.p(f'side{k}.table', 'const fbx::ISlot*')};")
            g(f"fbx::cp_async16(dyn_smem + SPAN_BUDGET + {16 * self.nt * self.pf_slot[k]}u"
              " + 16u * threadIdx.x, T + (tg & " + g.p(f'side{k}.mask') + "));")
            g("}")
            return name
        g(f"const fbx::Slot* T = {g.p(f'side{k}.table', 'const fbx::Slot*')};")
        g(f"const fbx::Slot* sl = T + (tg & {g.p(f'side{k}.mask')});")
        g(f"{name}_t = __ldg(&sl->tag); {name}_ref = __ldg(&sl->ref); {name}_aux = __ldg(&sl->aux);")
        g("}")
        return name

    def pipeline_kernel(self) -> str:
        ir, g = self.ir, self.g
        nt = self.nt
        drv = ir.driver
        dk = drv.cleaned_kinds()
        needed = self.driver_needed()
        self.staged = self.staged_columns()
        feats = sorted(ir.features.items(), key=lambda kv: (kv[1], kv[0]))
        K = max(1, len(feats))
        g(f"constexpr int NT = {nt};")
        g(f"constexpr u32 SPAN_BUDGET = {self.span_cap}u;")
        g(f"constexpr u32 DYN_SMEM = {self.dyn_smem}u;")
        g(f'extern "C" __global__ void __launch_bounds__(NT, {self.min_blocks}) '
          'fbx_pipeline(const fbx_params P) {')
        g("fbx_state* ST = (fbx_state*)P.v[0];")
        g(f"u64* STATUS = {g.p('tile_status', 'u64*')};")
        g(f"const u64 ROW_LO = {g.p('row_lo')}, ROW_HI = {g.p('row_hi')};")
        g(f"const u64 CHUNK0 = {g.p('chunk0')};")
        g(f"u8* POOL = {g.p('pool', 'u8*')}; const u64 POOL_CAP = {g.p('pool_cap')};")
        g("extern __shared__ __align__(16) u8 dyn_smem[];")
        g("__shared__ struct {")
        g("fbx::BlockScanU32<NT> scan;")
        g("fbx::TileReduce<NT> tred;")
        g("u64 pool_base; u32 tile; u64 ex_inst, ex_signs; u64 bar;")
        g("u32 rank[NT]; u32 soff[NT];")
        g("u64 span_lo[16]; u32 span_len[16];")
        g("u64 red[NT / 32][4];")
        g("} sm;")
        self.staged_plan = bool(self.staged)
        if self.pool_nodes:
            self.pool_decls()
        if self.phase_timers:
            g("u64 ph_t = clock64();")
        g("// tiles in blockIdx order: the hardware dispatches CTAs in order, so every")
        g("// predecessor a look-back waits on is resident or done (as CUB relies on)")
        bid = "blockIdx.x"
        g(f"const u32 TILE0 = (u32){g.p('tile_base')};  // this launch's first tile")
        g(f"const u32 tile = TILE0 + {bid};  // run-global tile id")
        if self.spc == 1:
            g(f"const u64 chunk = CHUNK0 + {bid};")
            g(f"const u64 row0 = ROW_LO + (u64){bid} * {ir.chunk}ull;")
            g(f"const u64 row_end = (row0 + {ir.chunk}ull < ROW_HI) ? row0 + {ir.chunk}ull : ROW_HI;")
        else:
            g(f"// sub-tile {bid} % {self.spc} of chunk {bid} / {self.spc} ({self.tile_rows} rows each)")
            g(f"const u64 chunk = CHUNK0 + {bid} / {self.spc}u;")
            g(f"const u64 cend0 = ROW_LO + (u64)({bid} / {self.spc}u + 1u) * {ir.chunk}ull;")
            g("const u64 cend = cend0 < ROW_HI ? cend0 : ROW_HI;")
            g(f"const u64 row0s = ROW_LO + (u64)({bid} / {self.spc}u) * {ir.chunk}ull + "
              f"(u64)({bid} % {self.spc}u) * {self.tile_rows}ull;")
            g("const u64 row0 = row0s < cend ? row0s : cend;")
            g(f"const u64 row_end = (row0 + {self.tile_rows}ull < cend) ? row0 + {self.tile_rows}ull : cend;")
        # (issuing the span TMA from the row sort's own offset loads, right after its
        # first barrier, measured 0.2-0.5 % slower: the copies are issued early
        # enough as it is)
        self.span_tma_early = False
        if self.staged:
            self.span_decls()
        if self.sort_rows and self.staged:
            # work-balanced warps: threads take the chunk's rows in order of their
            # string bytes (a 128-bucket counting sort), so the lanes of a warp run
            # the per-byte loops (JSON, tokens, FNV) for similar trip counts.  The
            # emission order is by instance id, independent of this mapping.
            # The offsets it loads also bound the chunk's string spans: the last
            # thread issues their TMA copies right after the first barrier, so the
            # copies overlap the rest of the sort (no extra barrier, no extra load).
            ns_ = len(self.staged)
            g("u32 RT;  // the chunk row this thread works on")
            g("{")
            g("__shared__ u32 srt_h[128]; __shared__ u16 srt_p[NT];")
            g(f"__shared__ u32 srt_lo[{ns_}], srt_hi[{ns_}];")
            g("for (u32 q = threadIdx.x; q < 128u; q += NT) srt_h[q] = 0u;")
            g("u32 L = 0u;")
            g("const u32 nrow = (u32)(row_end - row0);")
            g(f"if (threadIdx.x == 0 && nrow == 0u) {{ for (int i = 0; i < {ns_}; ++i) "
              "srt_lo[i] = srt_hi[i] = 0u; }")
            g(f"const bool in0 = threadIdx.x < {self.tile_rows}u && threadIdx.x < nrow;")
            g("if (in0) {")
            for i, c in enumerate(self.staged):
                offs = g.p(f"drv.{c}.offsets", "const u32*")
                g(f"{{ const u32 a = fbx::ldg_u32({offs} + row0 + threadIdx.x), "
                  f"b = fbx::ldg_u32({offs} + row0 + threadIdx.x + 1); L += b - a;")
                g(f"if (threadIdx.x == 0) srt_lo[{i}] = a; if (threadIdx.x + 1 == nrow) srt_hi[{i}] = b; }}")
            g("}")
            g("const u32 key = in0 ? (L >> 1 < 126u ? L >> 1 : 126u) : 127u;")
            g("__syncthreads();")
            if self.span_tma_early:
                g("if (threadIdx.x == NT - 1) {")
                self.span_tma(lambda i, offs: (f"srt_lo[{i}]", f"srt_hi[{i}]"))
                g("}")
            g("const u32 pos = atomicAdd(&srt_h[key], 1u);")
            g("__syncthreads();")
            g("if (threadIdx.x < 32u) {  // exclusive scan of the 128 buckets")
            g("const u32 a0 = srt_h[4 * threadIdx.x], a1 = srt_h[4 * threadIdx.x + 1], "
              "a2 = srt_h[4 * threadIdx.x + 2], a3 = srt_h[4 * threadIdx.x + 3];")
            g("u32 t = a0 + a1 + a2 + a3, x = t;")
            g("#pragma unroll")
            g("for (int d = 1; d < 32; d <<= 1) { const u32 y = __shfl_up_sync(0xFFFFFFFFu, x, d); "
              "if (threadIdx.x >= (u32)d) x += y; }")
            g("x -= t;")
            g("srt_h[4 * threadIdx.x] = x; srt_h[4 * threadIdx.x + 1] = x + a0; "
              "srt_h[4 * threadIdx.x + 2] = x + a0 + a1; srt_h[4 * threadIdx.x + 3] = x + a0 + a1 + a2;")
            g("}")
            g("__syncthreads();")
            g("srt_p[srt_h[key] + pos] = (u16)threadIdx.x;")
            g("__syncthreads();")
            g("RT = srt_p[threadIdx.x];")
            g("}")
        else:
            g("const u32 RT = threadIdx.x;")
        g("const u64 srow = row0 + RT;")
        g(f"const bool inrange = RT < {self.tile_rows}u && srow < row_end;")
        g("const u64 row = inrange ? srow : row0;")
        g("bool alive = inrange;")
        g("u32 malformed = 0, filtered = 0;")
        g(f"u32 CUR_STAGE = {STAGE['clean']}u, CUR_LAYER = 0u, CUR_RANK = 0u;")
        if self.staged and not self.span_tma_early:
            g("if (threadIdx.x == 0) {")
            self.span_tma(lambda i, offs: (f"fbx::ldg_u32({offs} + row0)",
                                           f"fbx::ldg_u32({offs} + row_end)"))
            g("}")
            g("__syncthreads();")
        # ---- prologue loads: every driver column this plan reads ----------------
        g("// ---- prologue: coalesced loads of the row's fixed columns / offsets ----")
        raw: dict[str, V] = {}
        for name, kind in drv.kinds.items():
            if name in needed:
                raw[name] = self.load_driver_column(name, kind)
        # ---- prefetch the first slot of every probe whose key is a raw column -----
        ext_out = {e.output for e in drv.extractions}

        def raw_key(cols):
            return all(c in raw and c not in ext_out and c not in drv.fills for c in cols)
        pre_side: dict[int, str | None] = {}
        for k, sv in enumerate(ir.sides):
            if raw_key(ir.join_keys):
                pre_side[k] = self.prefetch(k, [raw[c] for c in ir.join_keys],
                                            [dk[c] for c in ir.join_keys], f"pf{k}")
            else:
                pre_side[k] = None
        bk = len(ir.sides)
        pre_basic = None
        if ir.basic is not None and raw_key([ir.instance_column]):
            pre_basic = self.prefetch(bk, [raw[ir.instance_column]], [Kind.INT64], "pfb")
        if self.pf_slot:
            g("fbx::cp_async_commit();")
        if self.staged:
            g("fbx::mbar_wait(&sm.bar, 0u);")
        if self.dict_pf:
            g("// first dictionary slot of every lookup keyed by a driver string column,")
            g("// fetched now (cp.async) so the probe after the JSON finds it in smem")
            for name, (c, t, off) in self.dict_pf.items():
                v = raw[c]
                tag = f"dpf_{name.replace('.', '_')}"
                g(f"u64 {tag} = 0ull;")
                fills = self.ir.driver.fills
                if c in fills:
                    b = str(fills[c]).encode("utf-8", "surrogatepass")
                    kc = g.const(b)
                    key = f"({v.n} ? fbx::Str{{{kc}, {len(b)}u}} : {v.c})"
                    cond = "inrange"
                else:
                    key = v.c
                    cond = f"inrange && !{v.n}"
                g(f"if ({cond}) {{")
                g(f"const fbx::Str kk = {key};")
                g(f"{tag} = fbx::table_tag(fbx::tbl_hash_bytes(0x5DB2CEB4C16A9E87ull, kk.p, kk.n));")
                g(f"const fbx::Slot* sl = {g.p(f'dict{t}.slots', 'const fbx::Slot*')} + "
                  f"({tag} & {g.p(f'dict{t}.mask')});")
                g(f"u8* dst = dyn_smem + {off}u + 32u * threadIdx.x;")
                g("fbx::cp_async16(dst, sl); fbx::cp_async16(dst + 16, (const u8*)sl + 16);")
                g("}")
            g("fbx::cp_async_commit();")
        # ---- clean ------------------------------------------------------------------
        if self.phase_timers:
            g("FBX_PHASE(0);")
        g("// ---- clean (viewpipe.clean_views) ----")
        vals = self.clean_view(drv, "d_", lambda n, k: raw[n], "clean", needed, "")
        # ---- join -------------------------------------------------------------------
        if self.phase_timers:
            g("FBX_PHASE(1);")
        g(f"CUR_STAGE = {STAGE['join']}u;")
        env: dict[str, V] = dict(vals)
        side_rows: list[str] = []
        self.side_rows = side_rows
        idv0 = env.get(ir.instance_column)
        for k, sv in enumerate(ir.sides):
            g(f"// ---- join side view {sv.name!r} on {list(ir.join_keys)} ----")
            keys = [env[c] for c in ir.join_keys]
            kinds = [dk[c] for c in ir.join_keys]
            srow = f"sr{k}"
            g(f"u64 {srow} = 0ull;")
            null_any = " || ".join(v.n for v in keys if v.nullable) or "false"
            lone_any = " || ".join(v.l for v in keys if v.lone) or "false"
            g(f"if (alive && ({null_any})) alive = false;")
            g(f"if (alive && ({lone_any})) {{")
            self.row_error("join", "encode")
            g("}")
            g("if (alive) {")
            g("u32 cnt = 0;")
            self.probe(k, sv, keys, kinds, srow, "cnt", pre_side[k])
            g("if (cnt == 0u) alive = false;")
            g("else if (cnt > 1u) {")
            g(f"if (!{idv0.n}) {{")
            self.row_error("merge", "multi_match")
            g("} else { alive = false; }")
            g("}")
            g("}")
            side_rows.append(srow)
            for c in sv.cleaned_kinds():
                if c not in ir.join_keys:
                    env[c] = ("side", k, c)
        g("u32 joined = alive ? 1u : 0u;")
        self.env = env
        if self.pool_nodes:
            self.pool_join_site([env[c] for c in ir.join_keys] if ir.sides else [])
        # ---- basic merge probe (side-effect free; the drop is applied later) -------
        idv = env[ir.instance_column]
        if ir.basic is not None:
            g("// ---- basic-view probe on the instance id (merge_features) ----")
            g("u64 br = 0ull; bool bhit = false;")
            g(f"if (alive && !{idv.n}) {{")
            g("u32 bcnt = 0;")
            self.probe(bk, ir.basic, [idv], [Kind.INT64], "br", "bcnt", pre_basic)
            g("bhit = bcnt != 0u;")
            g("}")
            for c in ir.basic.cleaned_kinds():
                if c != ir.instance_column and c not in env:
                    env[c] = ("side", bk, c)
            side_rows.append("br")
        # eager gathers: every side / basic column the DAG or emit will read
        used_cols = set(ir.features)
        for nd in ir.nodes:
            used_cols |= set(nd.inputs)
        g("// ---- gathers of joined side / basic columns: loads issued before the DAG,")
        g("// their arithmetic at the first reader (driver-only nodes hide the latency)")
        for c in sorted(used_cols):
            if isinstance(env.get(c), tuple):
                if self.defer_gathers:
                    _, k, cc = env[c]
                    view = ir.sides[k] if k < len(ir.sides) else ir.basic
                    row = self.side_rows[k] if k < len(self.side_rows) else f"sr{k}"
                    self.prefetch_side_column(k, view, cc, row)
                else:
                    self.col(c, {})
        # ---- DAG --------------------------------------------------------------------
        g(f"CUR_STAGE = {STAGE['extract']}u;")
        if self.phase_timers:
            g("FBX_PHASE(2);")
        g("// ---- operator DAG: layer order (driver-only nodes first) ----")
        self.token_groups = self.plan_token_groups()
        self.token_done: dict[str, V] = {}
        node_out: dict[str, V] = {}
        for nd in self.node_schedule():
            if nd.role == "pre":
                args = [self.col(nd.inputs[0], node_out)]
            elif nd.role == "post":
                args = [node_out[nd.op]]
            else:
                pre = ir.pre_of.get(nd.op, {})
                args = [node_out[pre[i]] if i in pre else self.col(c, node_out)
                        for i, c in enumerate(nd.inputs)]
            node_out[nd.name] = self.node_code(nd, args)
        self.node_out = node_out
        for col, domain in ir.extract_outputs:
            v = node_out[ir.producer[col]]
            if domain == "u64" and v.t == "i64":
                g(f"if (alive && !{v.n} && (i64){v.c} < 0) {{")
                self.row_error("extract", "value")
                g("}")
        # ---- uniqueness check + merge ------------------------------------------------
        if self.phase_timers:
            g("FBX_PHASE(3);")
        g(f"CUR_STAGE = {STAGE['merge']}u;")
        lab = self.col(ir.label_column, node_out)
        g("// ---- check_unique_ids over the run (pipeline.py:1071, viewpipe.py:562) ----")
        g("// the winner of an id's slot stores its row; a later occurrence notes its")
        g("// row for fbx_dup_resolve and stays live (its rank keeps the emission")
        g("// positions of the chunks before the reported one exact)")
        g("// the first atomic is issued here; its result is only consumed at the very")
        g("// end of the kernel (collision probing + dup note), off the critical path")
        g(f"u64* IDS = {g.p('idset', 'u64*')}; const u64 IMASK = {g.p('idset_mask')};")
        g("u64 ids_slot = IMASK + 1; unsigned long long ids_old = 0ull;")
        g(f"const bool ids_on = alive && !{idv.n};")
        g("// one CAS for every id (id 0 -> its own slot, set 0 -> 1); no result copy")
        g(f"if ({idv.c} != 0ull) ids_slot = ({idv.c} * 0x9E3779B97F4A7C15ull) >> 20 & IMASK;")
        g("// rows that do not take part CAS a private dummy word (0 -> 0): no branch, so")
        g("// the result is never merged / copied right after the atomic")
        g(f"ids_old = atomicCAS((unsigned long long*)&IDS[ids_on ? ids_slot : IMASK + 2 + (row & 1023u)], "
          f"0ull, !ids_on ? 0ull : ({idv.c} == 0ull ? 1ull : (unsigned long long){idv.c}));")
        self._ids_tail = [
            "// ---- check_unique_ids: resolve the id-set insertion issued at the merge ----",
            "if (ids_on) {",
            "bool dup;",
            f"if ({idv.c} == 0ull) {{",
            "dup = ids_old != 0ull;",
            "} else {",
            f"while (ids_old != 0ull && ids_old != (unsigned long long){idv.c}) {{",
            "ids_slot = (ids_slot + 1) & IMASK;",
            f"ids_old = atomicCAS((unsigned long long*)&IDS[ids_slot], 0ull, (unsigned long long){idv.c});",
            "}",
            "dup = ids_old != 0ull;",
            "}",
            f"if (dup) fbx::dup_note(ST, {g.p('idset_d', 'u64*')} + 2 * ids_slot, row);",
            f"else {g.p('idset_w', 'u64*')}[ids_slot] = row;",
            "}",
        ]
        if ir.basic is not None:
            g(f"if (alive && ({idv.n} || !bhit)) alive = false;  // inner merge drops it")
        # ---- emit ---------------------------------------------------------------------
        g("// ---- emit_minibatch: sorted, de-duplicated (slot, sign) ----")
        g("// null / non-0/1 labels fail when the row's mini-batch is flushed: the row")
        g("// stays live for its emission position (raised after the look-back)")
        g(f"const u32 emit_bad = !alive ? 0u : ({lab.n} ? 1u : ({lab.c} > 1ull ? 2u : 0u));")
        fv = []
        for col, slot in feats:
            v = self.col(col, node_out)
            if v.t not in ("i64", "u64"):
                raise UnsupportedOnDevice(f"feature column {col!r} is not integer-valued")
            fv.append((slot, v))
        Kf = len(fv)
        g(f"u64 fsg[{max(Kf, 1)}]; u32 fpres = 0u;")
        i = 0
        while i < Kf:
            j = i
            while j < Kf and fv[j][0] == fv[i][0]:
                j += 1
            for q in range(i, j):
                v = fv[q][1]
                g(f"fsg[{q}] = {v.c}; if (!{v.n}) fpres |= {1 << q}u;")
            if j - i > 1:
                for a in range(i, j):
                    for b in range(i, j - 1 - (a - i)):
                        g(f"{{ bool pa = (fpres >> {b}) & 1u, pb = (fpres >> {b + 1}) & 1u;"
                          f" bool sw = (!pa && pb) || (pa && pb && fsg[{b}] > fsg[{b + 1}]);"
                          f" if (sw) {{ u64 t = fsg[{b}]; fsg[{b}] = fsg[{b + 1}]; fsg[{b + 1}] = t;"
                          f" fpres = (fpres & ~{(1 << b) | (1 << (b + 1))}u) | ((u32)pb << {b}) |"
                          f" ((u32)pa << {b + 1}); }} }}")
                for b in range(i + 1, j):
                    g(f"if (((fpres >> {b}) & 1u) && ((fpres >> {b - 1}) & 1u) && "
                      f"fsg[{b}] == fsg[{b - 1}]) fpres &= ~{1 << b}u;")
            i = j
        g("if (!alive) fpres = 0u;")
        g("const u32 m = alive ? __popc(fpres) : 0u;")

        # ---- tile: sort by instance id, offsets, look-back, write -----------------------
        if self.phase_timers:
            g("FBX_PHASE(4);")
        self.emission_order(idv, "alive", "m", "dyn_smem")
        # look-back by warp 0 while every warp (warp 0 after it) hashes its rows'
        # instance digests -- the digest is off the path to the aggregate publish
        if self.phase_timers:
            g("FBX_PHASE(5);")
        g("const u32 out_bytes = tile_signs * 10u + n_inst * 17u + 176u;")
        g("const bool staged_out = out_bytes <= DYN_SMEM;")
        self.emit_lookback()
        self.emit_digest(idv, lab, fv)
        g(f"u64* O_IDS = {g.p('out.ids', 'u64*')}; u8* O_LAB = {g.p('out.labels', 'u8*')};")
        g(f"u64* O_OFF = {g.p('out.offsets', 'u64*')}; u16* O_SLOT = {g.p('out.slots', 'u16*')};")
        g(f"u64* O_SIGN = {g.p('out.signs', 'u64*')};")
        g("// the look-back is launch-local (28-bit counts per launch); the run totals")
        g("// before this launch come from the previous launch's last tile (LB), so a")
        g("// run has no row limit.  Ring mode: the CSR of a launch lands at the start")
        g("// of its own output slot (offsets launch-local), for bounded-memory streams.")
        g(f"const u64* LB = {g.p('launch_base', 'const u64*')};")
        g("const u64 lb_i = LB[0], lb_s = LB[1];")
        g(f"const bool RING = {g.p('csr_ring')} != 0ull;")
        g("const u64 ei = (RING ? 0ull : lb_i) + sm.ex_inst, es = (RING ? 0ull : lb_s) + sm.ex_signs;")
        g("if (blockIdx.x == gridDim.x - 1u && threadIdx.x == 0u) {  // this launch's run totals")
        g(f"u64* LN = {g.p('launch_next', 'u64*')};")
        g("LN[0] = lb_i + sm.ex_inst + n_inst; LN[1] = lb_s + sm.ex_signs + tile_signs;")
        g("}")
        g(f"if (emit_bad) fbx::raise_emit(ST, lb_i + sm.ex_inst + myrank, emit_bad == 2u, {lab.c});")
        # sub-tiled chunks: the merge re-places label failures from the final order,
        # so a bad label is marked in the emitted label byte (0xFE null, 0xFF range;
        # such a run fails, its CSR is never handed out)
        labx = (f"(emit_bad ? (u8)(0xFDu + emit_bad) : (u8)({lab.c}))" if self.spc > 1
                else f"(u8)({lab.c})")
        g("u8* const st_sign = dyn_smem + ((u64)(O_SIGN + es) & 15u);")
        g("u8* const st_slot = st_sign + ((8u * tile_signs + 15u) & ~15u) + 16u - ((u64)(O_SIGN + es) & 15u) + ((u64)(O_SLOT + es) & 15u);")
        g("u8* const st_ids = st_slot + ((2u * tile_signs + 15u) & ~15u) + 16u - ((u64)(O_SLOT + es) & 15u) + ((u64)(O_IDS + ei) & 15u);")
        g("u8* const st_off = st_ids + ((8u * n_inst + 15u) & ~15u) + 16u - ((u64)(O_IDS + ei) & 15u) + ((u64)(O_OFF + ei) & 15u);")
        g("u8* const st_lab = st_off + ((8u * n_inst + 15u) & ~15u) + 16u - ((u64)(O_OFF + ei) & 15u) + ((u64)(O_LAB + ei) & 15u);")
        g("if (staged_out) {")
        g("if (alive) {")
        g("u64* s_sign = (u64*)st_sign; u16* s_slot = (u16*)st_slot;")
        g("const u32 r = myrank;")
        g("u32 so = myoff;")
        g(f"((u64*)st_ids)[r] = {idv.c}; st_lab[r] = {labx}; ((u64*)st_off)[r] = es + so;")
        for q, (slot, _) in enumerate(fv):
            g(f"if ((fpres >> {q}) & 1u) {{ s_slot[so] = (u16){slot}u; s_sign[so] = fsg[{q}]; ++so; }}")
        g("}")
        g("fbx::fence_async_smem();")
        g("__syncthreads();")
        if self.phase_timers:
            g("FBX_PHASE(6);")
        g("fbx::tile_out<NT>((u8*)(O_SIGN + es), st_sign, 8u * tile_signs);")
        g("fbx::tile_out<NT>((u8*)(O_SLOT + es), st_slot, 2u * tile_signs);")
        g("fbx::tile_out<NT>((u8*)(O_IDS + ei), st_ids, 8u * n_inst);")
        g("fbx::tile_out<NT>((u8*)(O_OFF + ei), st_off, 8u * n_inst);")
        g("fbx::tile_out<NT>(O_LAB + ei, st_lab, n_inst);")
        g("if (threadIdx.x == 0) fbx::bulk_commit();")
        g("} else if (alive) {")
        g("const u64 pos = ei + myrank;")
        g("u64 so = es + myoff;")
        g(f"O_IDS[pos] = {idv.c}; O_LAB[pos] = {labx};")
        g("O_OFF[pos] = so;")
        for q, (slot, _) in enumerate(fv):
            g(f"if ((fpres >> {q}) & 1u) {{ O_SLOT[so] = (u16){slot}u; O_SIGN[so] = fsg[{q}]; ++so; }}")
        g("}")
        g("if (threadIdx.x == 0) O_OFF[ei + n_inst] = es + tile_signs;")
        for line in self._ids_tail:
            g(line)
        if self.phase_timers:
            g("FBX_PHASE(7);")
        g("if (threadIdx.x == 0 && staged_out) fbx::bulk_wait_read();  // smem lives until read")
        if self.phase_timers:
            g("if (threadIdx.x == 0) { __threadfence(); if (atomicAdd(&fbx_ph_done, 1u) == gridDim.x - 1) {")
            g("__threadfence(); u64 t = 0; for (int q = 0; q < 10; ++q) t += fbx_ph[q];")
            g('for (int q = 0; q < 10; ++q) printf("FBX_PHASE %d %llu %.4f\\n", q, fbx_ph[q], (double)fbx_ph[q] / (double)t);')
            g("fbx_ph_done = 0; for (int q = 0; q < 10; ++q) fbx_ph[q] = 0; } }")
        g("}")
        return "fbx_pipeline"


    # ------------------------------------------------------------------------------
    def extract_rows_kernel(self) -> str:
        """``_extract_batch`` (pipeline.py:718-737): the DAG over an already cleaned
        and joined table, outputs row-aligned.  u64-domain outputs are written as
        Int64 images (two's-complement, ``wrap_u64``) with a warp-ballot null
        bitmap; str outputs are materialised into the pool as (pointer, length)
        and compacted into an FBXC Utf8 image by the host (scan + copy)."""
        ir, g = self.ir, self.g
        tbl = ir.driver
        self.staged = []
        g("constexpr int NT = 256;")
        g('extern "C" __global__ void __launch_bounds__(256) fbx_extract_rows(const fbx_params P) {')
        g("fbx_state* ST = (fbx_state*)P.v[0];")
        g(f"const u64 N = {g.p('rows')};")
        g(f"u8* POOL = {g.p('pool', 'u8*')}; const u64 POOL_CAP = {g.p('pool_cap')};")
        g("__shared__ struct { fbx::BlockScanU32<256> scan; u64 pool_base; } sm;")
        g("for (u64 base = (u64)blockIdx.x * 256u; base < N; base += (u64)gridDim.x * 256u) {")
        g("const u64 srow = base + threadIdx.x;")
        g("const bool inrange = srow < N;")
        g("const u64 row = inrange ? srow : base;")
        g("bool alive = inrange;")
        g("const u64 chunk = 0;")
        g(f"u32 CUR_STAGE = {STAGE['extract']}u, CUR_LAYER = 0u, CUR_RANK = 0u;")
        need = set()
        for nd in ir.nodes:
            need |= set(nd.inputs)
        env = {}
        for name, kind in tbl.kinds.items():
            if name in need:
                env[name] = self.load_driver_column(name, kind)
        self.env = env
        self.side_rows = []
        self.token_groups = self.plan_token_groups()
        self.token_done = {}
        node_out: dict[str, V] = {}
        for nd in ir.nodes:
            if nd.role == "pre":
                args = [self.col(nd.inputs[0], node_out)]
            elif nd.role == "post":
                args = [node_out[nd.op]]
            else:
                pre = ir.pre_of.get(nd.op, {})
                args = [node_out[pre[i]] if i in pre else self.col(c, node_out)
                        for i, c in enumerate(nd.inputs)]
            node_out[nd.name] = self.node_code(nd, args)
        g("// ---- outputs, row-aligned ----")
        for j, (col, domain) in enumerate(ir.extract_outputs):
            v = node_out[ir.producer[col]]
            nn = f"(!alive || {v.n})"
            if domain == "u64":
                if v.t == "i64":
                    g(f"if (alive && !{v.n} && (i64){v.c} < 0) {{")
                    self.row_error("extract", "value")
                    g("}")
                if v.t not in ("i64", "u64"):
                    raise UnsupportedOnDevice(f"output {col!r}: u64 domain on a {v.t} value")
                g(f"if (inrange) {g.p(f'out{j}.data', 'u64*')}[row] = {nn} ? 0ull : {v.c};")
            else:
                if v.t != "str":
                    raise UnsupportedOnDevice(f"output {col!r}: str domain on a {v.t} value")
                ptr = self.pool_alloc(f"{nn} ? 0u : {v.c}.n")
                g(f"if (inrange) {{ {g.p(f'out{j}.ptr', 'u64*')}[row] = (u64){ptr};"
                  f" {g.p(f'out{j}.len', 'u32*')}[row] = {nn} ? 0u : {v.c}.n; }}")
                g(f"if (!{nn} && {ptr}) fbx::str_copy{'_lower' if v.lower else ''}({ptr}, {v.c});")
                if v.lone:
                    g(f"if (!{nn} && {v.l}) {{ /* Utf8 column holds a lone surrogate: kept as WTF-8 */ }}")
            g("{")
            g(f"const u32 nb = __ballot_sync(0xFFFFFFFFu, inrange && {nn});")
            g(f"if ((threadIdx.x & 31u) == 0u && inrange) "
              f"((u32*){g.p(f'out{j}.nulls', 'u8*')})[row >> 5] = nb;")
            g("}")
        g("}")
        g("}")
        return "fbx_extract_rows"


    def emit_instance_digest(self, idv: V, lab: V, fv):
        """Instance digest (pipeline.py:375-382), straight-line over the row's
        features (registers)."""
        g = self.g
        g("u64 digest = 0ull;")
        g("if (alive) {")
        g("fbx::Fnv h;")
        g(f"h.u64_le({idv.c}); h.byte((u32)({lab.c} & 1ull));")
        for q, (slot, _) in enumerate(fv):
            g(f"if ((fpres >> {q}) & 1u) {{ h.u16_le({slot}u); h.u64_le(fsg[{q}]); }}")
        g("digest = h.value();")
        g("}")
        if self.phase_timers:
            g("FBX_PHASE(9);  // instance digests")

    def emit_digest(self, idv: V, lab: V, fv):
        """The block's counter reduction (digest XOR, clean / join counters)."""
        g = self.g
        self.emit_instance_digest(idv, lab, fv)
        g("{")
        g("// warp reductions (redux.sync): the XOR digest and three <=512 counters packed")
        g("const u32 r0l = __reduce_xor_sync(0xFFFFFFFFu, (u32)digest);")
        g("const u32 r0h = __reduce_xor_sync(0xFFFFFFFFu, (u32)(digest >> 32));")
        g("const u32 rc = __reduce_add_sync(0xFFFFFFFFu, malformed | (filtered << 10) | (joined << 20));")
        g("if ((threadIdx.x & 31u) == 0) { sm.red[threadIdx.x >> 5][0] = ((u64)r0h << 32) | r0l; "
          "sm.red[threadIdx.x >> 5][1] = rc & 0x3FFu; sm.red[threadIdx.x >> 5][2] = (rc >> 10) & 0x3FFu; "
          "sm.red[threadIdx.x >> 5][3] = rc >> 20; }")
        g("}")
        g("__syncthreads();")
        g("if (threadIdx.x == 0) {")
        g("u64 r0 = 0, r1 = 0, r2 = 0, r3 = 0;")
        g("for (int w = 0; w < NT / 32; ++w) { r0 ^= sm.red[w][0]; r1 += sm.red[w][1]; "
          "r2 += sm.red[w][2]; r3 += sm.red[w][3]; }")
        g("if (r0) atomicXor((unsigned long long*)&ST->digest, (unsigned long long)r0);")
        g("atomicAdd((unsigned long long*)&ST->instances, (unsigned long long)n_inst);")
        g("atomicAdd((unsigned long long*)&ST->signs, (unsigned long long)tile_signs);")
        g("if (r1) atomicAdd((unsigned long long*)&ST->malformed, (unsigned long long)r1);")
        g("if (r2) atomicAdd((unsigned long long*)&ST->filtered, (unsigned long long)r2);")
        g("if (r3) atomicAdd((unsigned long long*)&ST->joined, (unsigned long long)r3);")
        if self.pool_nodes:
            self.pool_tile_check()
        g("}")

    def emit_lookback(self):
        g = self.g
        g("if (threadIdx.x < 32u) {")
        g("u64 ei = 0, es = 0;")
        g("fbx::lookback(STATUS, tile, TILE0, n_inst, tile_signs, &ei, &es);")
        g("if (threadIdx.x == 0) { sm.ex_inst = ei; sm.ex_signs = es; }")
        g("}")
        if self.phase_timers:
            g("FBX_PHASE(8);  // look-back (warp 0 only)")

    def emission_order(self, idv: V, live: str, mm: str, scratch: str):
        """Tile counts + aggregate publish + rank / sign offset of every row (by
        ascending u64 instance id, viewpipe.py:521).  `live` / `mm`: which rows emit
        and their sign counts; `scratch`: shared memory for the rank pass."""
        g = self.g
        g("// ---- chunk emission order: ascending u64 instance id (viewpipe.py:521) ----")
        g(f"u64 skey = {live} ? {idv.c} : ~0ull;")
        g(f"u64* sbuf = (u64*)({scratch});")
        g("u32* hist = (u32*)(sbuf + NT); u32* bstart = hist + 1024; u16* bmv = (u16*)(bstart + 1024);")
        g("u32 myrank = 0, myoff = 0;")
        ir = self.ir
        fused = self.nt * max(1, len(ir.features)) < 65536
        if fused:
            g("// counts, signs and the ids' OR / AND in one reduction; the staged record")
            g("// spans are dead after its first barrier: the rank pass reuses that memory")
            g("u32 both; u64 kor, kand;")
            g(f"sm.tred.run(({live} ? 0x10000u : 0u) + {mm}, {live} ? skey : 0ull, {live} ? skey : ~0ull, "
              "&both, &kor, &kand, hist, 1024u);")
            g("const u32 n_inst = both >> 16, tile_signs = both & 0xFFFFu;")
        else:
            g(f"const u32 n_inst = sm.scan.sum({live} ? 1u : 0u);")
            g(f"const u32 tile_signs = sm.scan.sum({mm});")
        g("// publish the aggregate now: successors' look-back overlaps our sort")
        g("if (threadIdx.x == 0) fbx::publish_aggregate(STATUS, tile, TILE0, n_inst, tile_signs);")
        g("// Emitted ids are unique (else the run fails): a row's rank is the number")
        g("// of live ids below its own.  Adaptive radix buckets carrying the sign counts")
        g("// (rank and sign offset in one pass); bitonic sort + offset scan fallback.")
        if fused:
            g(f"if (!fbx::radix_rank_off<NT>(skey, {live}, {mm}, kor ^ kand, hist, bstart, sbuf, bmv, "
              "sm.scan, &myrank, &myoff)) {")
        else:
            g("{")
        g("const u64 sorted = fbx::bitonic_keys<NT>(skey, sbuf);")
        g("sbuf[2 * NT + threadIdx.x] = sorted;")
        g("__syncthreads();")
        g(f"myrank = {live} ? fbx::lower_rank<NT>(sbuf + 2 * NT, skey) : 0u;")
        g("sm.soff[threadIdx.x] = 0u;")
        g("__syncthreads();")
        g(f"if ({live}) sm.soff[myrank] = {mm};")
        g("__syncthreads();")
        g("const u32 s_off = sm.scan.exclusive(sm.soff[threadIdx.x]);")
        g("sm.rank[threadIdx.x] = s_off;  // sign offset by sorted position")
        g("__syncthreads();")
        g(f"myoff = {live} ? sm.rank[myrank] : 0u;")
        g("}")

    def node_schedule(self) -> list[NodeIR]:
        """Layer order, with nodes that need no joined column first (their work
        hides the latency of the side/basic gathers)."""
        ir = self.ir
        side_cols = set(self.env) - set(ir.driver.cleaned_kinds())
        dep: set[str] = set()
        for nd in ir.nodes:
            if nd.role == "post":
                if nd.op in dep:
                    dep.add(nd.name)
                continue
            reads = set(nd.inputs)
            pre = ir.pre_of.get(nd.op, {}) if nd.role == "body" else {}
            direct = {c for i, c in enumerate(nd.inputs) if i not in pre}
            if nd.role == "pre":
                direct = reads
            if any(c in side_cols or (c in ir.producer and ir.producer[c] in dep)
                   for c in direct) or any(pre[i] in dep for i in pre):
                dep.add(nd.name)
        first = [nd for nd in ir.nodes if nd.name not in dep]
        return first + [nd for nd in ir.nodes if nd.name in dep]

    def plan_token_groups(self) -> dict[str, tuple]:
        """token pre-calls that split the same column on the same delimiter are
        computed by one scan: node name -> (group key, field list)."""
        groups: dict[tuple, list[NodeIR]] = {}
        for nd in self.ir.nodes:
            if nd.role == "pre" and nd.fn.op == "token" and len(nd.fn.delim.encode()) == 1:
                groups.setdefault((nd.inputs[0], nd.fn.delim), []).append(nd)
        out = {}
        for key, nds in groups.items():
            if len(nds) < 2:
                continue
            fields = sorted({nd.fn.index for nd in nds})
            for nd in nds:
                out[nd.name] = (key, fields)
        return out

    def driver_needed(self) -> set[str]:
        """Driver (cleaned) columns the kernel must read."""
        ir = self.ir
        need = set(ir.join_keys) | {ir.instance_column, ir.label_column} | set(ir.features)
        for nd in ir.nodes:
            need |= set(nd.inputs)
        need |= {e.source for e in ir.driver.extractions}
        if ir.driver.filter is not None:
            need |= _filter_columns(ir.driver.filter)
        return need

    def col(self, name: str, node_out: Mapping[str, V]) -> V:
        ir = self.ir
        if name in ir.producer:
            return node_out[ir.producer[name]]
        v = self.env[name]
        if isinstance(v, tuple):  # lazily gathered side / basic column
            _, k, c = v
            view = ir.sides[k] if k < len(ir.sides) else ir.basic
            g = self.g
            row = self.side_rows[k] if k < len(self.side_rows) else f"sr{k}"
            g("// gather " + f"{view.name}.{c}")
            out = self.side_value(k, view, c, row)
            # side rows are only valid for joined rows
            if out.nullable:
                g(f"if (!alive) {out.c}_n = true;")
            self.env[name] = out
            return out
        return v

    def pool_program(self) -> tuple:
        return tuple((nd.layer, nd.rank, self.pool_plane_of[nd.name]) for nd in self.pool_nodes)

    # ------------------------------------------------------------------------------------
    def generate(self) -> Program:
        ir = self.ir
        self.globals: list[str] = []
        self.span_cap = 0
        needed = self.driver_needed()
        nstaged = sum(1 for c, k in ir.driver.kinds.items() if k.var_length and c in needed) \
            if ir.stage_strings else 0
        # shared-memory span budget per staged column (bytes, multiple of 16)
        self.span_cap = SPAN_BUDGET if nstaged else 0
        k = max(1, len(ir.features))
        # one dynamic region, reused: staged spans -> sort exchange -> CSR staging.
        # Sized so MIN_BLOCKS CTAs fit an SM (227 KB); a tile whose CSR does not
        # fit is written directly.
        per_cta = (227 * 1024) // self.min_blocks - STATIC_SMEM_EST - 1024
        need = max(self.span_cap, 24 * self.nt, 10 * self.nt + 8192, self.nt * (17 + 10 * k) + 64)
        rank_bytes = max(24 * self.nt, 10 * self.nt + 8192)  # bitonic 3*NT u64 | radix
        self.dyn_smem = max(self.span_cap, rank_bytes,
                            min(need, per_cta, OUT_BUDGET)) // 16 * 16
        self.dyn_smem = max(self.dyn_smem, (self.span_cap + 16 + 15) // 16 * 16)  # read slack
        # first probe slots of int-keyed tables land behind the staged spans
        self.pf_slot = {}
        if ir.mode != "extract":
            pf = self.smem_prefetch_tables()
            pf_need = self.span_cap + 16 * self.nt * len(pf)
            if pf and pf_need <= max(self.dyn_smem, per_cta):
                self.pf_slot = {k: j for j, k in enumerate(pf)}
                self.dyn_smem = max(self.dyn_smem, pf_need) // 16 * 16
            self.staged = self.staged_columns()
            dpf = self.dict_prefetch_nodes() if self.dict_prefetch else []
            base = self.span_cap + 16 * self.nt * len(self.pf_slot)
            d_need = base + 32 * self.nt * len(dpf)
            if dpf and d_need <= max(self.dyn_smem, per_cta):
                self.dict_pf = {name: (c, t, base + 32 * self.nt * j)
                                for j, (name, c, t) in enumerate(dpf)}
                self.dyn_smem = max(self.dyn_smem, d_need) // 16 * 16
        self.g.slot("state")  # slot 0
        if ir.mode == "clean":
            kname = self.clean_rows_kernel(ir.driver)
            consts = b"".join(self.g.consts)
            head = [library_source(), "", "// ===== generated plan =====",
                    f"__device__ const __align__(16) u8 K_STR[] = {_c_bytes(consts + bytes(16))};",
                    *self.globals, ""]
            return Program("\n".join(head + self.g.lines), dict(self.g.slots), 256, 0,
                           [kname], [], self.notes)
        if ir.mode == "extract":
            kname = self.extract_rows_kernel()
            consts = b"".join(self.g.consts)
            head = [library_source(), "", "// ===== generated plan =====",
                    f"__device__ const __align__(16) u8 K_STR[] = {_c_bytes(consts + bytes(16))};",
                    *self.globals, ""]
            return Program("\n".join(head + self.g.lines), dict(self.g.slots), 256, 0,
                           [kname], [], self.notes, ref_pool=self.pool_program(),
                           pool_kw=0xFFFFFFFF, pool_ni=self.pool_ni)
        side_names = []
        for k, sv in enumerate(ir.sides):
            side_names.append(self.side_prep_kernel(k, sv, False))
            self.g("")
        if ir.basic is not None:
            side_names.append(self.side_prep_kernel(len(ir.sides), ir.basic, True))
            self.g("")
        if side_names:
            self.side_prep_dispatch(len(side_names))
            self.g("")
        body_start = len(self.g.lines)
        kname = self.pipeline_kernel()
        consts = b"".join(self.g.consts)
        head = (["#ifndef FBX_POOL_WARP", "#define FBX_POOL_WARP", "#endif"] if self.pool_warp else []) + [library_source(), "",
                "// ===== generated plan =====",
                f"__device__ const __align__(16) u8 K_STR[] = {_c_bytes(consts + bytes(16))};",
                *self.globals, ""]
        src = "\n".join(head + self.g.lines)
        smem = self.dyn_smem
        del body_start
        nt_ = len(ir.sides) + (1 if ir.basic is not None else 0)
        return Program(src, dict(self.g.slots), self.nt, smem, [kname], side_names, self.notes,
                       tuple(k for k in range(nt_) if self.int_keyed(k)),
                       self.json_kind, self.spc, self.pool_program(), self.pool_kw,
                       self.pool_ni, self.tile_rows,
                       self.pool_sites * ((self.nt // 32) * 16 if self.pool_warp else 128))


def _filter_columns(expr) -> set[str]:
    if isinstance(expr, BoolExpr):
        out = set()
        for p in expr.parts:
            out |= _filter_columns(p)
        return out
    return {expr.column}


def generate(ir: PlanIR) -> Program:
    return PlanCodegen(ir).generate()
