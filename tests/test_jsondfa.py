"""CPU: the JSON DFA (device tables + exact emulation) against CPython json.loads.

Fuzzed documents (random valid JSON, then byte-level mutations) must be
accepted / rejected exactly like json.loads, and the extracted dot-path leaves
must equal viewpipe._walk_path on the parsed value (viewpipe.py:254-261)."""

from __future__ import annotations

import json
import random

import pytest

import jsondfa as D

PATHS = [["u", "city"], ["u"], ["src"], ["u", "tier"], ["a", "b", "c"]]
_MISSING = object()


def _walk(doc, parts):
    for p in parts:
        if not isinstance(doc, dict) or p not in doc:
            return _MISSING
        doc = doc[p]
    return doc


def _rand_value(rng, depth=0):
    r = rng.random()
    if depth < 4 and r < 0.25:
        keys = rng.sample(["u", "city", "src", "tier", "a", "b", "c", "x", "é", "u"],
                          rng.randint(0, 4))
        return {k: _rand_value(rng, depth + 1) for k in keys}
    if depth < 4 and r < 0.35:
        return [_rand_value(rng, depth + 1) for _ in range(rng.randint(0, 3))]
    if r < 0.55:
        return rng.choice(["tokyo", "", "a\"b", "back\\slash", "tab\t", "é", "\U0001F600",
                           "x y", "ctl"])
    if r < 0.7:
        return rng.choice([0, -1, 7, 123456789, -0, 10**25, 2**63])
    if r < 0.85:
        return rng.choice([0.5, -1e-7, 1e300, 3.25, -0.0, 1e21])
    return rng.choice([True, False, None, float("nan"), float("inf"), float("-inf")])


MUTANTS = b'{}[]:,"\\ \t\n0123456789-+.eEtrufalsnNIy\x01x'


def _mutate(rng, s):
    b = bytearray(s.encode("utf-8"))
    for _ in range(rng.randint(1, 3)):
        if not b:
            break
        k = rng.randrange(len(b))
        op = rng.random()
        if op < 0.3:
            del b[k]
        elif op < 0.6:
            b.insert(k, rng.choice(MUTANTS))
        else:
            b[k] = rng.choice(b'{}[]:,"\\ 0-.eE\x7f')
    return bytes(b)


def _check(doc: bytes):
    try:
        text = doc.decode("utf-8")
    except UnicodeDecodeError:
        return  # FBXC columns hold valid UTF-8 only
    paths = [[p.encode() for p in q] for q in PATHS]
    status, leaves = D.emulate(doc, paths)
    try:
        val = json.loads(text)
        ok, exc = True, None
    except json.JSONDecodeError:
        ok, exc = False, "decode"
    except ValueError:
        ok, exc = False, "bigint"
    except RecursionError:
        return
    if exc == "bigint":
        assert status == D.JS_BIGINT, doc
        return
    if not ok:
        assert status == D.JS_MALFORMED, (doc, status)
        return
    assert status == D.JS_OK, (doc, status)
    for q, (t, b0, b1, esc) in zip(PATHS, leaves):
        want = _walk(val, q)
        if want is _MISSING:
            assert t == D.J_MISSING, (doc, q, t)
            continue
        if isinstance(want, (dict, list)):
            assert t == D.J_CONTAINER, (doc, q)
        elif want is True:
            assert t == D.J_TRUE
        elif want is False:
            assert t == D.J_FALSE
        elif want is None:
            assert t == D.J_NULL
        elif isinstance(want, str):
            assert t == D.J_STRING
            assert json.loads(b'"' + doc[b0:b1] + b'"') == want
            assert bool(esc) == (b"\\" in doc[b0:b1])
        elif isinstance(want, int):
            assert t == D.J_INT and int(doc[b0:b1]) == want, (doc, q)
        else:
            text = doc[b0:b1].decode()
            if t == D.J_NAN:
                assert want != want
            elif t in (D.J_POSINF, D.J_NEGINF):
                assert want == (float("inf") if t == D.J_POSINF else float("-inf"))
            else:
                assert t == D.J_FLOAT and (float(text) == want or want != want), (doc, q)


CORNERS = [b"", b" ", b"{}", b"[]", b"[1,]", b"{,}", b'{"a":1,}', b"01", b"-", b"-0", b"1.",
           b"1e", b"1e+", b"1E5", b".5", b"+1", b"0x1", b'"\\x"', b'"\\u12"', b'"\\u12G4"',
           b'"\\/"', b"NaN", b"-NaN", b"-Infinity", b"Infinityx", b"truex", b"nul",
           b'{"a" : 1 }', b'{"u":{"city":"x"}}x', b" [1] ", b'"s"', b'"\x01"',
           b'{"u":{"city":"tab\there"}}', b'{"u":{"city":"a"},"u":5}',
           b'{"\\u0075":{"city":"k"}}', b"1" * 4301, b"-" + b"1" * 4300, b"1" * 4300 + b".5",
           b"[" * 64 + b"]" * 64, b"[" * 65 + b"]" * 65, b'{"u":{"city":"q","city":"r"}}',
           b"[1 2]", b'{"a" 1}', b'{"a"::1}', b"[,1]", b"\xef\xbb\xbf{}",
           b'{"u":{"city":"x"}}\n\r\t ']


@pytest.mark.parametrize("doc", CORNERS)
def test_corner_documents(doc):
    if doc.count(b"[") > 64:
        assert D.emulate(doc, [])[0] == D.JS_DEEP
        return
    _check(doc)


def test_fuzz_against_json_loads():
    rng = random.Random(2210)
    for _ in range(4000):
        v = _rand_value(rng)
        s = json.dumps(v, ensure_ascii=rng.random() < 0.5,
                       separators=rng.choice([(",", ":"), (", ", ": "), (" ,", " : ")]))
        _check(s.encode("utf-8"))
        _check(_mutate(rng, s))
