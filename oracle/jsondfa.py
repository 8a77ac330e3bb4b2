"""TEST INFRASTRUCTURE: a table-driven restatement of CPython's json.loads
grammar with dot-path extraction (viewpipe.py:254-280, 359-368).

It was built as a candidate device parser (a byte-class / transition-table
DFA); measured on B200 it was ~35 % slower than the control-flow scanner in
fbx_core.cuh because lanes of a warp diverge on the per-byte action code, so
the product keeps the control-flow scanner.  The model stays here as an
independently fuzz-validated grammar (tests/test_jsondfa.py) used to generate
and classify JSON corner cases.

CPython's ``json.loads`` (strict) accepts exactly the documents this DFA
accepts (validated by fuzzing against json.loads in tests/test_jsondfa.py):
objects, arrays, strings with the eight escapes and ``\\uXXXX``, numbers
``-?(0|[1-9]\\d*)(\\.\\d+)?([eE][-+]?\\d+)?``, ``true false null NaN Infinity
-Infinity``, whitespace `` \\t\\n\\r`` between tokens, nothing after the value.
The container stack and dot-path bookkeeping are code, not table (depth <= 64
on the device).  Used by viewpipe.clean_views (viewpipe.py:359-368, 254-280).

Per byte the device does: class = CLS[byte]; entry = TR[state*NCLS + class];
state = entry & 63; rare action bits (entry >> 6) run the stack/extraction code.
``render_header()`` emits the tables for csrc/device/fbx_json_tables.cuh;
``emulate()`` is the exact algorithm of ``fbx::json_extract`` in Python.
"""

from __future__ import annotations

# ---- byte classes -----------------------------------------------------------
C_OTHER, C_SPACE, C_WSCTL, C_CTL, C_QUOTE, C_BSLASH, C_LBRACE, C_RBRACE, C_LBRACK, C_RBRACK, \
    C_COLON, C_COMMA, C_MINUS, C_PLUS, C_DOT, C_ZERO, C_DIGIT, C_e, C_E, C_a, C_b, C_cd, C_f, \
    C_HEXUP, C_t, C_r, C_u, C_l, C_s, C_n, C_N, C_I, C_i, C_y, C_SLASH = range(35)
NCLS = 35


def byte_class(c: int) -> int:
    ch = chr(c)
    table = {" ": C_SPACE, "\t": C_WSCTL, "\n": C_WSCTL, "\r": C_WSCTL, '"': C_QUOTE,
             "\\": C_BSLASH, "{": C_LBRACE, "}": C_RBRACE, "[": C_LBRACK, "]": C_RBRACK,
             ":": C_COLON, ",": C_COMMA, "-": C_MINUS, "+": C_PLUS, ".": C_DOT, "0": C_ZERO,
             "e": C_e, "E": C_E, "a": C_a, "b": C_b, "c": C_cd, "d": C_cd, "f": C_f,
             "A": C_HEXUP, "B": C_HEXUP, "C": C_HEXUP, "D": C_HEXUP, "F": C_HEXUP,
             "t": C_t, "r": C_r, "u": C_u, "l": C_l, "s": C_s, "n": C_n, "N": C_N, "I": C_I,
             "i": C_i, "y": C_y, "/": C_SLASH}
    if ch in table:
        return table[ch]
    if "1" <= ch <= "9":
        return C_DIGIT
    if c < 0x20:
        return C_CTL
    return C_OTHER


CLS = bytes(byte_class(c) for c in range(256))

# ---- states ---------------------------------------------------------------------
STATES = ["ERR", "V_TOP", "V", "V_ARR0", "K0", "K", "COLON", "AV_TOP", "AV_OBJ", "AV_ARR",
          "VSTR", "VSTR_ESC", "VSTR_U1", "VSTR_U2", "VSTR_U3", "VSTR_U4",
          "KSTR", "KSTR_ESC", "KSTR_U1", "KSTR_U2", "KSTR_U3", "KSTR_U4",
          "N_MINUS", "N_ZERO", "N_INT", "N_DOT", "N_FRAC", "N_E", "N_ESIGN", "N_EXP",
          "L_t", "L_tr", "L_tru", "L_f", "L_fa", "L_fal", "L_fals", "L_n", "L_nu", "L_nul",
          "L_N", "L_Na", "L_I", "L_In", "L_Inf", "L_Infi", "L_Infin", "L_Infini", "L_Infinit"]
S = {name: i for i, name in enumerate(STATES)}
assert len(STATES) <= 64

# action bits (entry >> 6)
A_VSTART = 1 << 0    # first byte of a value
A_PUSH = 1 << 1      # '{' / '['
A_POP = 1 << 2       # '}' / ']' closes the current container -> AV(context)
A_KSTART = 1 << 3    # opening quote of a key
A_KEND = 1 << 4      # closing quote of a key
A_VEND = 1 << 5      # a string / literal value ends with this byte -> AV(context)
A_REPROC = 1 << 6    # a number ended before this byte: -> AV(context), redo this byte
A_ESC = 1 << 7       # backslash inside a string
A_DIGIT = 1 << 8     # an integer-part digit (the 4300-digit int limit)

# value types (match fbx_core.cuh J_*)
J_MISSING, J_STRING, J_INT, J_FLOAT, J_TRUE, J_FALSE, J_NULL, J_CONTAINER, J_NAN, J_POSINF, \
    J_NEGINF = range(11)
LIT_TYPE = [0] * 64
LIT_TYPE[S["L_tru"]] = J_TRUE
LIT_TYPE[S["L_fals"]] = J_FALSE
LIT_TYPE[S["L_nul"]] = J_NULL
LIT_TYPE[S["L_Na"]] = J_NAN
LIT_TYPE[S["L_Infinit"]] = J_POSINF  # J_NEGINF when the value started with '-'

HEX = (C_ZERO, C_DIGIT, C_a, C_b, C_cd, C_e, C_f, C_E, C_HEXUP)
DIGITS = (C_ZERO, C_DIGIT)
NUM_END = (C_SPACE, C_WSCTL, C_COMMA, C_RBRACE, C_RBRACK)
WS = (C_SPACE, C_WSCTL)


def _build():
    tr = [[0] * NCLS for _ in STATES]  # 0 = ERR, no action

    def put(state, classes, nxt, act=0):
        for c in classes:
            tr[S[state]][c] = S[nxt] | (act << 6)

    for v in ("V_TOP", "V", "V_ARR0"):
        put(v, WS, v)
        put(v, (C_QUOTE,), "VSTR", A_VSTART)
        put(v, (C_LBRACE,), "K0", A_VSTART | A_PUSH)
        put(v, (C_LBRACK,), "V_ARR0", A_VSTART | A_PUSH)
        put(v, (C_MINUS,), "N_MINUS", A_VSTART)
        put(v, (C_ZERO,), "N_ZERO", A_VSTART | A_DIGIT)
        put(v, (C_DIGIT,), "N_INT", A_VSTART | A_DIGIT)
        put(v, (C_t,), "L_t", A_VSTART)
        put(v, (C_f,), "L_f", A_VSTART)
        put(v, (C_n,), "L_n", A_VSTART)
        put(v, (C_N,), "L_N", A_VSTART)
        put(v, (C_I,), "L_I", A_VSTART)
    put("V_ARR0", (C_RBRACK,), "AV_TOP", A_POP)  # next state resolved by code
    put("K0", WS, "K0")
    put("K0", (C_QUOTE,), "KSTR", A_KSTART)
    put("K0", (C_RBRACE,), "AV_TOP", A_POP)
    put("K", WS, "K")
    put("K", (C_QUOTE,), "KSTR", A_KSTART)
    put("COLON", WS, "COLON")
    put("COLON", (C_COLON,), "V")
    put("AV_TOP", WS, "AV_TOP")
    put("AV_OBJ", WS, "AV_OBJ")
    put("AV_OBJ", (C_COMMA,), "K")
    put("AV_OBJ", (C_RBRACE,), "AV_TOP", A_POP)
    put("AV_ARR", WS, "AV_ARR")
    put("AV_ARR", (C_COMMA,), "V")
    put("AV_ARR", (C_RBRACK,), "AV_TOP", A_POP)
    for p, end_state, end_act in (("VSTR", "AV_TOP", A_VEND), ("KSTR", "COLON", A_KEND)):
        inside = [c for c in range(NCLS) if c not in (C_QUOTE, C_BSLASH, C_CTL, C_WSCTL)]
        put(p, inside, p)
        put(p, (C_QUOTE,), end_state, end_act)
        put(p, (C_BSLASH,), p + "_ESC", A_ESC)
        put(p + "_ESC", (C_QUOTE, C_BSLASH, C_SLASH, C_b, C_f, C_n, C_r, C_t), p)
        put(p + "_ESC", (C_u,), p + "_U1")
        put(p + "_U1", HEX, p + "_U2")
        put(p + "_U2", HEX, p + "_U3")
        put(p + "_U3", HEX, p + "_U4")
        put(p + "_U4", HEX, p)
    put("N_MINUS", (C_ZERO,), "N_ZERO", A_DIGIT)
    put("N_MINUS", (C_DIGIT,), "N_INT", A_DIGIT)
    put("N_MINUS", (C_I,), "L_I")
    for st in ("N_ZERO", "N_INT", "N_FRAC", "N_EXP"):
        put(st, NUM_END, "AV_TOP", A_REPROC)
    put("N_INT", DIGITS, "N_INT", A_DIGIT)
    for st in ("N_ZERO", "N_INT"):
        put(st, (C_DOT,), "N_DOT")
    for st in ("N_ZERO", "N_INT", "N_FRAC"):
        put(st, (C_e, C_E), "N_E")
    put("N_DOT", DIGITS, "N_FRAC")
    put("N_FRAC", DIGITS, "N_FRAC")
    put("N_E", (C_PLUS, C_MINUS), "N_ESIGN")
    put("N_E", DIGITS, "N_EXP")
    put("N_ESIGN", DIGITS, "N_EXP")
    put("N_EXP", DIGITS, "N_EXP")
    chains = [("t", "r", "u", "e"), ("f", "a", "l", "s", "e"), ("n", "u", "l", "l"),
              ("N", "a", "N"), ("I", "n", "f", "i", "n", "i", "t", "y")]
    names = {("t",): "L_t", ("t", "r"): "L_tr", ("t", "r", "u"): "L_tru",
             ("f",): "L_f", ("f", "a"): "L_fa", ("f", "a", "l"): "L_fal",
             ("f", "a", "l", "s"): "L_fals", ("n",): "L_n", ("n", "u"): "L_nu",
             ("n", "u", "l"): "L_nul", ("N",): "L_N", ("N", "a"): "L_Na"}
    word = "Infinity"
    for k in range(1, len(word)):
        names[tuple(word[:k])] = "L_" + word[:k]
    for ch in chains:
        for k in range(1, len(ch)):
            st = names[ch[:k]]
            c = byte_class(ord(ch[k]))
            if k + 1 < len(ch):
                put(st, (c,), names[ch[:k + 1]])
            else:
                put(st, (c,), "AV_TOP", A_VEND)
    return tr


TR = _build()
NUM_STATES = {S["N_ZERO"], S["N_INT"], S["N_FRAC"], S["N_EXP"]}

# emulate() return codes (fbx_core.cuh JS_*)
JS_OK, JS_MALFORMED, JS_BIGINT, JS_DEEP = range(4)
MAX_DEPTH = 64


def emulate(doc: bytes, paths: list[list[bytes]]):
    """Exact Python model of fbx::json_extract: (status, [(type, beg, end, esc)])."""
    np_ = len(paths)
    leaf = [(J_MISSING, 0, 0, 0)] * np_
    n = len(doc)
    s = S["V_TOP"]
    depth = 0
    kind = 0          # bit d: container at depth d+1 is an object
    live = [0] * 9    # live path mask of the object at depth d (1..8)
    leafm = 0         # paths whose leaf is the value about to start
    descm = (1 << np_) - 1
    top = True
    vbeg = 0
    vneg = False
    kbeg = 0
    esc = 0
    digits = 0
    pend = 0          # leaf paths of the value in progress (recorded at its end)

    def av():
        if depth == 0:
            return S["AV_TOP"]
        return S["AV_OBJ"] if (kind >> (depth - 1)) & 1 else S["AV_ARR"]

    i = 0
    while i < n:
        c = doc[i]
        e = TR[s][CLS[c]]
        act = e >> 6
        if act & A_REPROC:  # a number ended just before this byte
            t = J_INT if s in (S["N_ZERO"], S["N_INT"]) else J_FLOAT
            if digits > 4300 and t == J_INT:
                return JS_BIGINT, leaf
            for p in range(np_):
                if pend >> p & 1:
                    leaf[p] = (t, vbeg, i, 0)
            pend = 0
            s = av()
            e = TR[s][CLS[c]]
            act = e >> 6
        ns = e & 63
        if act:
            if act & A_VSTART:
                vbeg, esc, digits, vneg = i, 0, 0, c == ord("-")
                pend = leafm
                top_now = top
                top = False
                if act & A_PUSH:
                    obj = c == ord("{")
                    if depth >= MAX_DEPTH:
                        return JS_DEEP, leaf
                    for p in range(np_):
                        if pend >> p & 1:
                            leaf[p] = (J_CONTAINER, i, i, 0)
                    pend = 0
                    kind = kind | (1 << depth) if obj else kind & ~(1 << depth)
                    depth += 1
                    if depth <= 8:
                        live[depth] = ((1 << np_) - 1 if top_now else descm) if obj else 0
                leafm, descm = 0, 0
            elif act & A_PUSH:
                pass
            if act & A_DIGIT:
                digits += 1
            if act & A_ESC:
                esc = 1
            if act & A_KSTART:
                kbeg, esc = i + 1, 0
            if act & A_KEND:
                leafm, descm = 0, 0
                if depth <= 8 and live[depth]:
                    key = doc[kbeg:i]
                    if esc:
                        import json as _j
                        key = _j.loads(b'"' + key + b'"').encode("utf-8", "surrogatepass")
                    sidx = depth - 1
                    for p in range(np_):
                        if not live[depth] >> p & 1 or sidx >= len(paths[p]):
                            continue
                        if key != paths[p][sidx]:
                            continue
                        leaf[p] = (J_MISSING, 0, 0, 0)
                        if sidx + 1 == len(paths[p]):
                            leafm |= 1 << p
                        else:
                            descm |= 1 << p
            if act & A_VEND:
                if s in (S["VSTR"],):
                    t, b0, b1 = J_STRING, vbeg + 1, i
                else:
                    t = LIT_TYPE[s]
                    if t == J_POSINF and vneg:
                        t = J_NEGINF
                    b0, b1 = vbeg, i + 1
                for p in range(np_):
                    if pend >> p & 1:
                        leaf[p] = (t, b0, b1, esc)
                pend = 0
                ns = av()
            if act & A_POP:
                depth -= 1
                ns = av()
        s = ns
        if s == S["ERR"]:
            return JS_MALFORMED, leaf
        i += 1
    if s in NUM_STATES:
        t = J_INT if s in (S["N_ZERO"], S["N_INT"]) else J_FLOAT
        if digits > 4300 and t == J_INT:
            return JS_BIGINT, leaf
        for p in range(np_):
            if pend >> p & 1:
                leaf[p] = (t, vbeg, n, 0)
        s = av()
    if s != S["AV_TOP"] or depth != 0:
        return JS_MALFORMED, leaf
    return JS_OK, leaf


def render_header() -> str:
    """csrc/device/fbx_json_tables.cuh (generated; do not edit)."""
    cls = ",".join(str(b) for b in CLS)
    rows = ",\n  ".join(",".join(str(e) for e in row) for row in TR)
    lit = ",".join(str(x) for x in LIT_TYPE)
    names = "\n".join(f"#define JS_{name} {i}" for i, name in enumerate(STATES))
    return f"""// fbx_json_tables.cuh -- GENERATED by paper_2210_07768_b200/jsondfa.py; do not edit.
#pragma once
namespace fbx {{
{names}
constexpr u32 JNCLS = {NCLS};
constexpr u32 JA_VSTART = {A_VSTART}, JA_PUSH = {A_PUSH}, JA_POP = {A_POP}, JA_KSTART = {A_KSTART},
              JA_KEND = {A_KEND}, JA_VEND = {A_VEND}, JA_REPROC = {A_REPROC}, JA_ESC = {A_ESC},
              JA_DIGIT = {A_DIGIT};
__device__ const unsigned char JCLS[256] = {{{cls}}};
__device__ const unsigned short JTR[{len(STATES)} * {NCLS}] = {{
  {rows}}};
__device__ const unsigned char JLIT[64] = {{{lit}}};
}}  // namespace fbx
"""


if __name__ == "__main__":
    from pathlib import Path
    print(render_header()[:400])
