"""Exact Python model of ``fbx::json_canon`` (Json-kind extraction, viewpipe.py:266-267).

``json.dumps(json.loads(doc), sort_keys=True, separators=(",", ":"))`` computed the
device's way: ensure_ascii escaping of decoded code points, ints as written except
``-0``, floats as ``repr()`` of the correctly rounded double (``decimal_tables.f64_repr``),
``Infinity`` on overflow, objects emitted by selection (each step scans the members
for the smallest key above the last one emitted, the later duplicate winning) through
an explicit stack of open containers.  Checked against ``json.dumps`` in
tests/test_host.py; the device port is checked against the oracle on the GPU.
"""

from __future__ import annotations

import json
import random
import struct

from .decimal_tables import f64_repr

_WS = b" \t\n\r"
_SHORT = {8: "\\b", 12: "\\f", 10: "\\n", 13: "\\r", 9: "\\t"}
_UNESC = {0x62: 8, 0x66: 12, 0x6E: 10, 0x72: 13, 0x74: 9}


def json_canon(doc: bytes) -> str:
    s, n = doc, len(doc)

    def skip(i):
        while i < n and s[i] in _WS:
            i += 1
        return i

    def str_end(i):
        while s[i] != 0x22:
            i += 2 if s[i] == 0x5C else 1
        return i

    def value_end(i):
        c = s[i]
        if c == 0x22:
            return str_end(i + 1) + 1
        if c in b"{[":
            depth = 0
            while True:
                c = s[i]
                if c == 0x22:
                    i = str_end(i + 1) + 1
                    continue
                if c in b"{[":
                    depth += 1
                elif c in b"}]":
                    depth -= 1
                    if depth == 0:
                        return i + 1
                i += 1
        while i < n and s[i] not in b",}]" and s[i] not in _WS:
            i += 1
        return i

    def cps(b, e):
        out, i = [], b
        while i < e:
            c = s[i]
            if c != 0x5C:
                ln = 1 if c < 0x80 else 2 if c < 0xE0 else 3 if c < 0xF0 else 4
                out.append(ord(s[i:i + ln].decode("utf-8")))
                i += ln
                continue
            x = s[i + 1]
            if x != 0x75:
                out.append(_UNESC.get(x, x))
                i += 2
                continue
            cp = int(s[i + 2:i + 6], 16)
            i += 6
            if 0xD800 <= cp <= 0xDBFF and s[i:i + 2] == b"\\u":
                lo = int(s[i + 2:i + 6], 16)
                if 0xDC00 <= lo <= 0xDFFF:
                    cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00)
                    i += 6
            out.append(cp)
        return out

    def put_str(b, e):
        o = ['"']
        for cp in cps(b, e):
            if cp in (0x22, 0x5C):
                o.append("\\" + chr(cp))
            elif 0x20 <= cp <= 0x7E:
                o.append(chr(cp))
            elif cp in _SHORT:
                o.append(_SHORT[cp])
            elif cp < 0x10000:
                o.append(f"\\u{cp:04x}")
            else:
                v = cp - 0x10000
                o.append(f"\\u{0xD800 | (v >> 10):04x}\\u{0xDC00 | (v & 0x3FF):04x}")
        o.append('"')
        return "".join(o)

    def put_scalar(b, e):
        t = s[b:e].decode()
        if t[0] == '"':
            return put_str(b + 1, e - 1)
        if t == "-Infinity" or not (t[0] == "-" or t[0].isdigit()):
            return t
        if not any(ch in t for ch in ".eE"):
            return "0" if t == "-0" else t
        x = float(t)
        if x in (float("inf"), float("-inf")):
            return "Infinity" if x > 0 else "-Infinity"
        return f64_repr(struct.unpack("<Q", struct.pack("<d", x))[0])

    b = skip(0)
    if s[b] not in b"{[":
        return put_scalar(b, value_end(b))
    out = [chr(s[b])]
    st = [[s[b] == 0x7B, skip(b + 1), None, True]]  # object?, position, last key, first
    while st:
        f = st[-1]
        if not f[0]:
            i = f[1]
            if s[i] == 0x5D:
                out.append("]")
                st.pop()
                continue
            if not f[3]:
                out.append(",")
            f[3] = False
            vb, ve = i, value_end(i)
            nx = skip(ve)
            if s[nx] == 0x2C:
                nx = skip(nx + 1)
            f[1] = nx
        else:
            best, i = None, f[1]
            while s[i] != 0x7D:
                kb = i + 1
                ke = str_end(kb)
                vi = skip(skip(ke + 1) + 1)
                vend = value_end(vi)
                if f[3] or cps(kb, ke) > cps(*f[2]):
                    if best is None or cps(kb, ke) <= cps(best[0], best[1]):
                        best = (kb, ke, vi)
                i = skip(vend)
                if s[i] == 0x2C:
                    i = skip(i + 1)
            if best is None:
                out.append("}")
                st.pop()
                continue
            if not f[3]:
                out.append(",")
            f[3] = False
            f[2] = (best[0], best[1])
            out.append(put_str(best[0], best[1]) + ":")
            vb, ve = best[2], value_end(best[2])
        if s[vb] in b"{[":
            st.append([s[vb] == 0x7B, skip(vb + 1), None, True])
            out.append(chr(s[vb]))
        else:
            out.append(put_scalar(vb, ve))
    return "".join(out)


_KEYS = ["a", "b", "B", "é", "éx", "k\\u0041", "aa", "", "\U0001F600", "z",
         "\\ud83d\\ude00"]
_STRS = ["x", "é", " ", "tab\there", 'q"uote', "\x7f", "\U0001F600", "back\\slash", "",
         "ctl\x01"]


def random_json_docs(n: int, seed: int = 3) -> list[str]:
    """Random valid JSON documents: nested objects / arrays, duplicate keys,
    escapes, non-ASCII, floats of every magnitude, NaN / Infinity, whitespace."""
    rng = random.Random(seed)

    def scalar():
        r = rng.random()
        if r < 0.2:
            return json.dumps(rng.choice(_STRS), ensure_ascii=rng.random() < 0.5)
        if r < 0.3:
            return rng.choice(['"\\ud800"', '"\\u00E9"', '"\\/"', '"a\\u0000b"'])
        if r < 0.5:
            return str(rng.choice([0, 7, -12, 10 ** 20, -(10 ** 30), 123456789]))
        if r < 0.55:
            return "-0"
        if r < 0.8:
            m = rng.randrange(1, 10 ** rng.randrange(1, 18))
            return rng.choice([f"{m}e{rng.randrange(-330, 310)}", f"{m}.5", f"-{m}E+3",
                               f"0.{m}", f"{m}.0e-7", "1e400", "-1e400", "1e-400", "-0.0"])
        return rng.choice(["true", "false", "null", "NaN", "Infinity", "-Infinity"])

    def sp():
        return rng.choice(["", "", " ", "\n ", "\t"])

    def value(d):
        r = rng.random()
        if d < 4 and r < 0.3:
            items = [f'{sp()}"{rng.choice(_KEYS)}"{sp()}:{sp()}{value(d + 1)}{sp()}'
                     for _ in range(rng.randrange(0, 5))]
            return "{" + ",".join(items) + sp() + "}"
        if d < 4 and r < 0.45:
            return "[" + ",".join(sp() + value(d + 1) + sp()
                                  for _ in range(rng.randrange(0, 4))) + "]"
        return scalar()

    out = []
    while len(out) < n:
        doc = value(0)
        try:
            json.loads(doc)
        except ValueError:
            continue
        out.append(doc)
    return out


def check_json_canon(n: int, seed: int = 3) -> int:
    docs = random_json_docs(n, seed)
    for d in docs:
        want = json.dumps(json.loads(d), sort_keys=True, separators=(",", ":"))
        got = json_canon(d.encode("utf-8"))
        if got != want:
            raise AssertionError(f"json_canon({d!r}) = {got!r}, json.dumps = {want!r}")
    return len(docs)
