"""FBXC column images: the host-side and H2D layout of every view.

A view is held as one *column image* per column, exactly the byte layout an
FBXC file stores (reference ``pkg/docs/fbxc_format.md``; writer
``columnstore.py:338-398``, reader ``columnstore.py:401-608``):

* ``nulls``   -- LSB-first bitmap, bit set = null (``columnstore.py:117-130``);
* ``data``    -- Int64 little-endian ``int64[n]`` / Float32 ``float32[n]`` /
  Utf8 and Json: the concatenated UTF-8 payload (``uint8[...]``);
* ``offsets`` -- var-length kinds only, ``uint32[n + 1]``.

Null slots hold the kind's zero value (``columnstore.py:90-95``), so payload
bytes are deterministic.  Images are numpy arrays so a row range of a column is
one contiguous span per segment: that span is what the engine copies to HBM
(no per-value decode on the host -- the reference decodes into Python lists,
``columnstore.py:579-602``).
"""

from __future__ import annotations

import enum
import mmap
import os
import struct
import zlib
from dataclasses import dataclass, field
from pathlib import Path
from typing import Iterable, Mapping, Sequence

import numpy as np

MAGIC = b"FBXC"
VERSION = 1
MASK64 = (1 << 64) - 1
INT64_MIN = -(1 << 63)
INT64_MAX = (1 << 63) - 1


class FormatError(ValueError):
    """A view file violates the FBXC format (``columnstore.py:35``)."""


class ChecksumError(FormatError):
    """Body CRC32 does not match the footer (``columnstore.py:51``)."""


class BadMagicError(FormatError):
    pass


class UnsupportedVersionError(FormatError):
    pass


class TruncatedError(FormatError):
    pass


class UnknownColumnError(KeyError):
    pass


class Kind(enum.IntEnum):
    """Column kinds; the integer is the on-disk code (``columnstore.py:59-63``)."""

    INT64 = 0
    FLOAT32 = 1
    UTF8 = 2
    JSON = 3

    @property
    def var_length(self) -> bool:
        return self >= Kind.UTF8

    @property
    def fixed_width(self) -> int | None:
        return {Kind.INT64: 8, Kind.FLOAT32: 4}.get(self)

    @classmethod
    def from_name(cls, name: str) -> "Kind":
        try:
            return cls[name.upper()]
        except KeyError:
            raise ValueError(f"unknown column kind {name!r}") from None


def wrap_u64(value: int) -> int:
    """u64 -> two's-complement Int64 image (``columnstore.py:100-104``)."""
    if not 0 <= value <= MASK64:
        raise ValueError(f"value {value} outside u64 range")
    return value - (1 << 64) if value > INT64_MAX else value


def unwrap_u64(value: int) -> int:
    """Int64 image (or u64) -> u64 (``columnstore.py:107-111``)."""
    if not INT64_MIN <= value <= MASK64:
        raise ValueError(f"value {value} outside wrapped u64 range")
    return value & MASK64


def canon_f32(value: float) -> float:
    """Round to float32 storage precision (``columnstore.py:97``)."""
    return struct.unpack("<f", struct.pack("<f", value))[0]


def bitmap_bytes(n: int) -> int:
    return (n + 7) >> 3


@dataclass
class ColumnImage:
    """One column as FBXC segments (numpy views, never Python lists)."""

    kind: Kind
    n: int
    nulls: np.ndarray  # uint8[bitmap_bytes(n)]
    data: np.ndarray  # int64[n] | float32[n] | uint8[payload]
    offsets: np.ndarray | None = None  # uint32[n+1] for var-length kinds

    def __post_init__(self):
        self.kind = Kind(self.kind)
        if self.nulls.dtype != np.uint8 or self.nulls.size < bitmap_bytes(self.n):
            raise FormatError("null bitmap too short")
        if self.kind.var_length:
            if self.offsets is None or self.offsets.size != self.n + 1:
                raise FormatError("var-length column needs n+1 offsets")
            if self.offsets.dtype != np.uint32:
                raise FormatError("offsets must be uint32")
        elif self.data.size != self.n:
            raise FormatError("fixed column payload length mismatch")

    # -- construction -----------------------------------------------------
    @classmethod
    def from_values(cls, kind: Kind, values: Sequence) -> "ColumnImage":
        """Canonicalise Python values (None = null) into an image."""
        kind = Kind(kind)
        n = len(values)
        null_mask = np.fromiter((v is None for v in values), dtype=bool, count=n)
        nulls = np.packbits(null_mask, bitorder="little") if n else np.zeros(0, np.uint8)
        if kind is Kind.INT64:
            data = np.array([0 if v is None else int(v) for v in values], dtype=np.int64)
            return cls(kind, n, nulls, data)
        if kind is Kind.FLOAT32:
            data = np.array([0.0 if v is None else float(v) for v in values], dtype=np.float32)
            return cls(kind, n, nulls, data)
        blobs = [b"" if v is None else v.encode("utf-8") for v in values]
        lens = np.fromiter((len(b) for b in blobs), dtype=np.uint64, count=n)
        offsets = np.zeros(n + 1, dtype=np.uint64)
        np.cumsum(lens, out=offsets[1:])
        if n and offsets[-1] > 0xFFFFFFFF:
            raise FormatError("var-length payload exceeds u32 offset range")
        data = np.frombuffer(b"".join(blobs), dtype=np.uint8).copy()
        return cls(kind, n, nulls, data, offsets.astype(np.uint32))

    # -- access -------------------------------------------------------------
    def null_mask(self) -> np.ndarray:
        return np.unpackbits(self.nulls, bitorder="little", count=self.n).astype(bool)

    def value(self, i: int):
        """Row i as the reference's Python value (``Column.get``)."""
        if self.nulls[i >> 3] >> (i & 7) & 1:
            return None
        if self.kind is Kind.INT64:
            return int(self.data[i])
        if self.kind is Kind.FLOAT32:
            return float(self.data[i])
        lo, hi = int(self.offsets[i]), int(self.offsets[i + 1])
        return bytes(self.data[lo:hi]).decode("utf-8")

    def to_pylist(self) -> list:
        return [self.value(i) for i in range(self.n)]

    def slice(self, lo: int, hi: int) -> "ColumnImage":
        """Rows [lo, hi) as a new image (bitmap re-based to bit 0)."""
        n = hi - lo
        mask = self.null_mask()[lo:hi]
        nulls = np.packbits(mask, bitorder="little") if n else np.zeros(0, np.uint8)
        if self.kind.var_length:
            base = int(self.offsets[lo])
            offs = (self.offsets[lo : hi + 1].astype(np.uint64) - base).astype(np.uint32)
            data = self.data[base : int(self.offsets[hi])]
            return ColumnImage(self.kind, n, nulls, data, offs)
        return ColumnImage(self.kind, n, nulls, self.data[lo:hi])

    def nbytes(self) -> int:
        total = bitmap_bytes(self.n) + self.data.nbytes
        if self.offsets is not None:
            total += self.offsets.nbytes
        return total

    def segments(self) -> list[tuple[str, bytes]]:
        parts = [("nulls", self.nulls[: bitmap_bytes(self.n)].tobytes())]
        if self.kind.var_length:
            parts.append(("offsets", self.offsets.tobytes()))
            base = int(self.offsets[0]) if self.n else 0
            if base:
                raise FormatError("write a re-based slice")
        parts.append(("data", np.ascontiguousarray(self.data).tobytes()))
        return parts


@dataclass
class ViewImage:
    """A view: ordered (name, kind) schema, key columns, column images."""

    columns: dict[str, ColumnImage]
    key_columns: tuple[str, ...] = ()
    order: tuple[str, ...] = field(default=())

    def __post_init__(self):
        if not self.order:
            self.order = tuple(self.columns)
        ns = {c.n for c in self.columns.values()}
        if len(ns) > 1:
            raise FormatError("columns have differing row counts")
        for k in self.key_columns:
            if k not in self.columns:
                raise FormatError(f"key column {k!r} not in view")

    @property
    def row_count(self) -> int:
        return next(iter(self.columns.values())).n if self.columns else 0

    @property
    def schema(self) -> tuple[tuple[str, Kind], ...]:
        return tuple((n, self.columns[n].kind) for n in self.order)

    def kind_of(self, name: str) -> Kind:
        try:
            return self.columns[name].kind
        except KeyError:
            raise UnknownColumnError(name) from None

    def project(self, wanted: Iterable[str] | None) -> "ViewImage":
        if wanted is None:
            return self
        wanted = set(wanted)
        missing = wanted - set(self.columns)
        if missing:
            raise UnknownColumnError(sorted(missing)[0])
        order = tuple(n for n in self.order if n in wanted)
        return ViewImage(
            {n: self.columns[n] for n in order},
            tuple(k for k in self.key_columns if k in wanted),
            order,
        )

    def slice(self, lo: int, hi: int) -> "ViewImage":
        return ViewImage(
            {n: self.columns[n].slice(lo, hi) for n in self.order},
            self.key_columns,
            self.order,
        )

    def nbytes(self) -> int:
        return sum(c.nbytes() for c in self.columns.values())

    @classmethod
    def from_pydict(
        cls,
        spec: Sequence[tuple[str, Kind]],
        data: Mapping[str, Sequence],
        key_columns: Sequence[str] = (),
    ) -> "ViewImage":
        cols = {name: ColumnImage.from_values(kind, data[name]) for name, kind in spec}
        return cls(cols, tuple(key_columns), tuple(n for n, _ in spec))


# -- FBXC files ---------------------------------------------------------------

_U16 = struct.Struct("<H")
_U32 = struct.Struct("<I")
_U64 = struct.Struct("<Q")
_SEG = struct.Struct("<QQ")


def write_view(view: ViewImage, path: str | Path) -> Path:
    """Serialise to FBXC; byte-identical to the reference writer's output."""
    path = Path(path)
    if not view.order:
        raise FormatError("cannot write a view with zero columns")
    head = bytearray(MAGIC)
    head += _U16.pack(VERSION) + _U64.pack(view.row_count)
    head += _U16.pack(len(view.order)) + _U16.pack(len(view.key_columns))
    for name in view.order:
        raw = name.encode("utf-8")
        head += bytes([int(view.columns[name].kind)]) + _U16.pack(len(raw)) + raw
    index = {n: i for i, n in enumerate(view.order)}
    for k in view.key_columns:
        head += _U16.pack(index[k])
    blobs = [blob for n in view.order for _, blob in view.columns[n].segments()]
    cursor = len(head) + 4 + _SEG.size * len(blobs)
    directory = bytearray(_U32.pack(len(blobs)))
    for blob in blobs:
        directory += _SEG.pack(cursor, len(blob))
        cursor += len(blob)
    body = b"".join(blobs)
    with open(path, "wb") as fh:
        fh.write(head)
        fh.write(directory)
        fh.write(body)
        fh.write(_U32.pack(zlib.crc32(body) & 0xFFFFFFFF))
    return path


@dataclass(frozen=True)
class ViewFile:
    path: Path
    schema: tuple[tuple[str, Kind], ...]
    key_columns: tuple[str, ...]
    row_count: int
    segments: dict[tuple[str, str], tuple[int, int]]
    body_offset: int
    body_bytes: int
    checksum: int


def open_view(path: str | Path) -> ViewFile:
    """Parse an FBXC header + directory (``columnstore.py:401-478``).

    Only the header, the directory and the 4-byte CRC trailer are read (the
    body is read later, span by span); the file length is checked against the
    directory."""
    path = Path(path)
    with open(path, "rb") as fh:
        size = os.fstat(fh.fileno()).st_size
        blob = fh.read(min(size, 1 << 16))

        def more(upto: int):
            # read on as the header needs; past the end of the file the parse below
            # fails exactly as the reference's does on its whole-file blob
            nonlocal blob
            if upto > len(blob):
                blob += fh.read(upto - len(blob))

        # the reference's checks and messages (columnstore.py:401-478)
        if len(blob) < 6:
            raise TruncatedError(f"{path}: too short for a header")
        if blob[:4] != MAGIC:
            raise BadMagicError(f"{path}: magic {bytes(blob[:4])!r}, expected {MAGIC!r}")
        (version,) = _U16.unpack_from(blob, 4)
        if version != VERSION:
            raise UnsupportedVersionError(f"{path}: version {version}, expected {VERSION}")
        try:
            pos = 6
            more(pos + 12)
            (rows,) = _U64.unpack_from(blob, pos)
            (ncols,) = _U16.unpack_from(blob, pos + 8)
            (nkeys,) = _U16.unpack_from(blob, pos + 10)
            pos += 12
            schema = []
            for _ in range(ncols):
                more(pos + 3)
                kind = Kind(blob[pos])
                (ln,) = _U16.unpack_from(blob, pos + 1)
                more(pos + 3 + ln)
                name = blob[pos + 3 : pos + 3 + ln].decode("utf-8")
                if len(name.encode("utf-8")) != ln:
                    raise TruncatedError(f"{path}: truncated column name")
                schema.append((name, kind))
                pos += 3 + ln
            keys = []
            for _ in range(nkeys):
                more(pos + 2)
                keys.append(schema[_U16.unpack_from(blob, pos)[0]][0])
                pos += 2
            more(pos + 4)
            (nseg,) = _U32.unpack_from(blob, pos)
            pos += 4
            more(pos + nseg * _SEG.size)
            spans = [_SEG.unpack_from(blob, pos + i * _SEG.size) for i in range(nseg)]
            pos += nseg * _SEG.size
        except (struct.error, IndexError, ValueError) as exc:
            if isinstance(exc, FormatError):
                raise
            raise TruncatedError(f"{path}: malformed header ({exc})") from None
        parts = [
            (n, p)
            for n, k in schema
            for p in (("nulls", "offsets", "data") if k.var_length else ("nulls", "data"))
        ]
        if len(parts) != nseg:
            raise FormatError(f"{path}: directory has {nseg} segments, schema implies "
                              f"{len(parts)}")
        cursor = pos
        segs = {}
        for key, (off, ln) in zip(parts, spans):
            if off != cursor:
                raise FormatError(f"{path}: segment {key[0]}/{key[1]} not contiguous")
            segs[key] = (off, ln)
            cursor += ln
        if cursor + 4 != size:
            raise TruncatedError(f"{path}: file is {size} bytes, layout implies {cursor + 4}")
        fh.seek(cursor)
        (crc,) = _U32.unpack(fh.read(4))
    return ViewFile(path, tuple(schema), tuple(keys), rows, segs, pos, cursor - pos, crc)


def read_view(
    source: str | Path | ViewFile,
    wanted: Iterable[str] | None = None,
    verify: bool = True,
) -> ViewImage:
    """Map an FBXC file into column images without decoding values.

    Segments are zero-copy numpy views over an mmap of the file.  With
    ``verify`` and a full read the body CRC32 is checked first, as the
    reference does for whole-body reads (``columnstore.py:554-562``).
    """
    vf = source if isinstance(source, ViewFile) else open_view(source)
    names = [n for n, _ in vf.schema]
    wanted_set = set(names) if wanted is None else set(wanted)
    unknown = wanted_set - set(names)
    if unknown:
        raise UnknownColumnError(sorted(unknown)[0])
    with open(vf.path, "rb") as fh:
        mm = mmap.mmap(fh.fileno(), 0, access=mmap.ACCESS_READ)
    buf = np.frombuffer(mm, dtype=np.uint8)
    if verify and wanted_set == set(names):
        crc = zlib.crc32(buf[vf.body_offset : vf.body_offset + vf.body_bytes]) & 0xFFFFFFFF
        if crc != vf.checksum:
            raise ChecksumError(f"{vf.path}: body CRC {crc:#010x} != footer {vf.checksum:#010x}")
    n = vf.row_count
    cols = {}
    for name, kind in vf.schema:
        if name not in wanted_set:
            continue
        o, ln = vf.segments[(name, "nulls")]
        nulls = buf[o : o + ln]
        o, ln = vf.segments[(name, "data")]
        raw = buf[o : o + ln]
        if kind is Kind.INT64:
            cols[name] = ColumnImage(kind, n, nulls, raw.view(np.int64))
        elif kind is Kind.FLOAT32:
            cols[name] = ColumnImage(kind, n, nulls, raw.view(np.float32))
        else:
            oo, oln = vf.segments[(name, "offsets")]
            cols[name] = ColumnImage(kind, n, nulls, raw, buf[oo : oo + oln].view(np.uint32))
    order = tuple(n for n, _ in vf.schema if n in wanted_set)
    return ViewImage(cols, tuple(k for k in vf.key_columns if k in wanted_set), order)


def schema_of(path: str | Path) -> tuple[tuple[str, Kind], ...]:
    return open_view(path).schema
