"""Correctly rounded decimal -> binary64 on the device (JSON Float32 leaves).

CPython's ``float(text)`` is correctly rounded (viewpipe.py:278-279 then
canon_f32).  The device uses a bracketing variant of Eisel-Lemire: with
``T[q] = floor(10**q * 2**s_q)`` normalised to 128 bits, a decimal
``w * 10**q`` (w < 2**64, the first 19 significant digits; more digits widen
the bracket to [w, w+1)) lies in ``[w*T, (w+1)*T + w + 1) / 2**s_q``.  Rounding
to nearest-even is monotone, so when both ends of the bracket round to the same
double that double is the exact answer; otherwise (a rounding boundary within
~2**-120 relative of the value) the device reports "needs a bignum" (never
observed on random inputs; tests/test_host.py checks 200k cases against float()).

``render()`` writes csrc/device/fbx_pow10.cuh; ``to_double()`` is the exact
Python model of ``fbx::dec_to_double``.
"""

from __future__ import annotations

import math
import struct
from pathlib import Path

QMIN, QMAX = -342, 308
HEADER = Path(__file__).resolve().parent / "csrc" / "device" / "fbx_pow10.cuh"


def table() -> list[tuple[int, int]]:
    """(T_q, s_q) for q in [QMIN, QMAX]: T = floor(10^q * 2^s), 2^127 <= T < 2^128."""
    out = []
    for q in range(QMIN, QMAX + 1):
        if q >= 0:
            v = 10 ** q
            s = 127 - (v.bit_length() - 1)
            t = v << s if s >= 0 else v >> -s
        else:
            d = 10 ** (-q)
            s = 127 + d.bit_length()
            t = (1 << s) // d
            while t >= 1 << 128:
                s -= 1
                t = (1 << s) // d
            while t < 1 << 127:
                s += 1
                t = (1 << s) // d
        assert (1 << 127) <= t < (1 << 128), q
        out.append((t, s))
    return out


_T = None


def _round53(p: int, e: int):
    """Round p * 2^e (p > 0 integer) to binary64: returns (bits) or None on overflow."""
    msb = p.bit_length() - 1
    exp = msb + e  # value in [2^exp, 2^(exp+1))
    if exp > 1023:
        return None
    if exp >= -1022:
        shift = msb - 52
    else:  # subnormal: fixed quantum 2^-1074
        shift = -1074 - e
    if shift <= 0:
        m = p << -shift
    else:
        m = p >> shift
        rem = p - (m << shift)
        half = 1 << (shift - 1)
        if rem > half or (rem == half and (m & 1)):
            m += 1
    q_exp = e + shift  # value = m * 2^q_exp
    if m == 0:
        return 0
    if m >= 1 << 53:  # mantissa overflow from rounding
        m >>= 1
        q_exp += 1
    if m >= 1 << 52:
        be = q_exp + 52 + 1075 - 52 - 1 + 1  # biased exponent
        be = q_exp + 1075
        if be >= 2047:
            return None
        return (be << 52) | (m & ((1 << 52) - 1))
    return m  # subnormal: biased exponent 0


def to_double(w: int, q: int, exact: bool):
    """(bits | None for overflow | 'slow') of w*10^q (exact=False: value in [w, w+1)*10^q)."""
    global _T
    if _T is None:
        _T = table()
    if w == 0:
        return 0
    if q < QMIN:
        return 0 if exact or (w + 1) * 10 ** 19 < 10 ** 19 * 2 else "slow"
    if q > QMAX:
        return None
    t, s = _T[q - QMIN]
    t_exact = 0 <= q and t == (10 ** q << s if s >= 0 else -1)
    lo = w * t
    hi = (w + (0 if exact else 1)) * (t + (0 if t_exact else 1)) - (0 if exact and t_exact else 1)
    a = _round53(lo, -s)
    b = _round53(hi, -s)
    if a == b:
        return a
    if not exact or a is None:
        return "slow"
    # exact decision against the midpoint of a and its successor (fbx::dec_to_double_tie)
    from fractions import Fraction
    ea_b = (a >> 52) & 0x7FF
    ma = ((a & ((1 << 52) - 1)) | (1 << 52)) if ea_b else (a & ((1 << 52) - 1))
    ea = ea_b - 1075 if ea_b else -1074
    mid = Fraction(2 * ma + 1) * Fraction(2) ** (ea - 1)
    v = Fraction(w) * Fraction(10) ** q
    r = a if v < mid else a + 1 if v > mid else (a + 1 if ma & 1 else a)
    return None if (r & 0x7FFFFFFFFFFFFFFF) >= 0x7FF0000000000000 else r


def decimal_parts(text: str):
    """Significand (first 19 significant digits), decimal exponent, exactness."""
    m = text.lstrip("-")
    if "e" in m or "E" in m:
        mant, _, ex = m.replace("E", "e").partition("e")
        ex = int(ex)
    else:
        mant, ex = m, 0
    ip, _, fp = mant.partition(".")
    digits = (ip + fp).lstrip("0")
    ex -= len(fp)
    if not digits:
        return 0, 0, True
    tail = digits[19:]
    ex += len(tail)
    return int(digits[:19]), ex, not tail.strip("0")


def f32_repr(bits: int) -> str:
    """Exact Python model of ``fbx::f32_repr``: ``repr(float)`` of a float32 value.

    str() of a Float32 value reaching lower/trim/token/concat/lookup
    (featureops.py:298-299, 318, 336) is CPython's shortest round-trip repr of
    the value widened to binary64 (``_Py_dg_dtoa`` mode 0 + ``format_float_short``).
    Widened, the value is ``f * 2**e`` with ``f`` even, so its round-to-nearest
    interval ``[L, H]`` is closed.  In units of ``2**t`` (t = e - 2) the interval
    and the value are the integers L, V, H < 2**55.  With K chosen so that
    ``H * 2**t / 10**K < 10**19``, the 19-digit windows ``floor(X * 2**t / 10**K)``
    plus a sticky bit decide exactly, for every p, whether a multiple of
    ``10**(K+p)`` lies in [L, H]; the largest such p gives the shortest digit
    string, and the candidate nearest V (ties to even) is the repr digits.
    """
    s, ex, m = bits >> 31, (bits >> 23) & 0xFF, bits & 0x7FFFFF
    if ex == 255:
        return "nan" if m else ("-inf" if s else "inf")
    if ex == 0 and m == 0:
        return "-0.0" if s else "0.0"
    mant, e2 = ((m | 0x800000), ex - 150) if ex else (m, -149)
    bl = mant.bit_length()
    f, e = mant << (53 - bl), e2 - (53 - bl)
    lo, v, hi, t = 4 * f - (1 if f == 1 << 52 else 2), 4 * f, 4 * f + 2, e - 2
    k = (((hi.bit_length() - 1 + t) * 78913) >> 18) - 17  # floor(log10 2^x) - 17

    def window(x: int) -> tuple[int, bool]:
        if k >= 0:
            if t >= 0:
                q, r = divmod(x << t, 10 ** k)
                return q, r != 0
            q, r = divmod(x >> -t, 10 ** k)
            return q, r != 0 or (x & ((1 << -t) - 1)) != 0
        p5, sh = x * 5 ** -k, t - k
        if sh >= 0:
            return p5 << sh, False
        return p5 >> -sh, (p5 & ((1 << -sh) - 1)) != 0

    (wl, sl), (wv, sv), (wh, _) = window(lo), window(v), window(hi)
    for p in range(19, 0, -1):
        p10 = 10 ** p
        top = wh // p10
        bot = wl // p10 + (1 if (wl % p10 or sl) else 0)
        if bot <= top:
            w, r = divmod(wv, p10)
            if r > p10 // 2 or (r == p10 // 2 and (sv or (w & 1))):
                w += 1
            w = min(max(w, bot), top)
            break
    digits = str(w)
    nd = len(digits)
    decpt = nd + k + p
    out = "-" if s else ""
    if decpt <= -4 or decpt > 16:
        x = decpt - 1
        return (out + digits[0] + ("." + digits[1:] if nd > 1 else "")
                + ("e-" if x < 0 else "e+") + f"{abs(x):02d}")
    if decpt <= 0:
        return out + "0." + "0" * -decpt + digits
    if decpt < nd:
        return out + digits[:decpt] + "." + digits[decpt:]
    return out + digits + "0" * (decpt - nd) + ".0"


def check_f32_repr(n: int = 100000, seed: int = 5) -> int:
    """Compare ``f32_repr`` with repr() on edge and random float32 bit patterns."""
    import random
    rng = random.Random(seed)
    cases = [0, 1, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00000, 0xFFC00001, 0x7F7FFFFF]
    for ex in range(255):
        cases += [ex << 23, (ex << 23) | 1, (ex << 23) | 0x7FFFFF, (ex << 23) | 0x400000]
    cases += [rng.getrandbits(32) for _ in range(n)]
    for b in cases:
        want = repr(struct.unpack("<f", struct.pack("<I", b))[0])
        assert f32_repr(b) == want, (hex(b), f32_repr(b), want)
    return len(cases)


def render() -> str:
    rows = table()
    hi = ",".join(f"0x{t >> 64:016X}ull" for t, _ in rows)
    lo = ",".join(f"0x{t & ((1 << 64) - 1):016X}ull" for t, _ in rows)
    sh = ",".join(str(s) for _, s in rows)
    ex = ",".join("1" if (QMIN + i >= 0 and s >= 0 and t == (10 ** (QMIN + i)) << s) else "0"
                  for i, (t, s) in enumerate(rows))
    return "\n".join([
        "// fbx_pow10.cuh -- GENERATED by paper_2210_07768_b200/decimal_tables.py; do not edit.",
        "#pragma once",
        "namespace fbx {",
        f"constexpr int P10_QMIN = {QMIN}, P10_QMAX = {QMAX};",
        f"__device__ const u64 P10_HI[{len(rows)}] = {{{hi}}};",
        f"__device__ const u64 P10_LO[{len(rows)}] = {{{lo}}};",
        f"__device__ const short P10_S[{len(rows)}] = {{{sh}}};",
        f"__device__ const unsigned char P10_EXACT[{len(rows)}] = {{{ex}}};",
        "}  // namespace fbx", ""])


def check_random(n: int = 20000, seed: int = 3) -> int:
    """Compare the model with float() on random decimal strings; returns #slow."""
    import random
    rng = random.Random(seed)
    slow = 0
    for _ in range(n):
        nd = rng.choice([1, 2, 5, 9, 15, 17, 19, 20, 25, 40])
        digits = "".join(rng.choice("0123456789") for _ in range(nd)).lstrip("0") or "0"
        e = rng.choice([0, rng.randint(-30, 30), rng.randint(-350, 320)])
        text = f"{digits}e{e}" if rng.random() < 0.5 else (
            digits[:max(1, nd // 2)] + "." + digits[max(1, nd // 2):] + "0" if nd > 1 else digits)
        ref = float(text)
        w, q, exact = decimal_parts(text)
        got = to_double(w, q, exact)
        if got == "slow":
            slow += 1
            continue
        want = None if math.isinf(ref) else struct.unpack("<Q", struct.pack("<d", ref))[0]
        assert got == want, (text, got, want)
    return slow


if __name__ == "__main__":
    HEADER.write_text(render())
    print("wrote", HEADER, "slow:", check_random())


def f64_repr(bits: int) -> str:
    """Exact Python model of ``fbx::f64_repr``: ``repr(float)`` of a binary64 value.

    The f32 scheme of :func:`f32_repr` generalised: subnormals keep their fixed
    spacing (no normalisation), the round-to-nearest interval is closed only for
    an even mantissa (ties-to-even parsing), and the windows need big integers
    (the device uses 36 x 32-bit limbs: x << t < 2^1030, x * 5^341 < 2^850).
    """
    s, ex, m = bits >> 63, (bits >> 52) & 0x7FF, bits & ((1 << 52) - 1)
    if ex == 0x7FF:
        return "nan" if m else ("-inf" if s else "inf")
    if ex == 0 and m == 0:
        return "-0.0" if s else "0.0"
    f, e = ((m | (1 << 52)), ex - 1075) if ex else (m, -1074)
    closed = (f & 1) == 0
    lo = 4 * f - (1 if (m == 0 and ex > 1) else 2)
    v, hi, t = 4 * f, 4 * f + 2, e - 2
    k = (((hi.bit_length() - 1 + t) * 78913) >> 18) - 17

    def window(x: int) -> tuple[int, bool]:
        if k >= 0:
            if t >= 0:
                q, r = divmod(x << t, 10 ** k)
                return q, r != 0
            q, r = divmod(x >> -t, 10 ** k)
            return q, r != 0 or (x & ((1 << -t) - 1)) != 0
        p5, sh = x * 5 ** -k, t - k
        if sh >= 0:
            return p5 << sh, False
        return p5 >> -sh, (p5 & ((1 << -sh) - 1)) != 0

    (wl, sl), (wv, sv), (wh, sh_) = window(lo), window(v), window(hi)
    for p in range(19, 0, -1):
        p10 = 10 ** p
        if closed:
            top = wh // p10
            bot = wl // p10 + (1 if (wl % p10 or sl) else 0)
        else:
            top = wh // p10 - (1 if (wh % p10 == 0 and not sh_) else 0)
            bot = wl // p10 + 1
        if bot <= top:
            w, r = divmod(wv, p10)
            if r > p10 // 2 or (r == p10 // 2 and (sv or (w & 1))):
                w += 1
            w = min(max(w, bot), top)
            break
    else:  # p = 0: the window digits themselves (unreachable for binary64)
        p, w = 0, wv
    digits = str(w)
    nd = len(digits)
    decpt = nd + k + p
    out = "-" if s else ""
    if decpt <= -4 or decpt > 16:
        x = decpt - 1
        return (out + digits[0] + ("." + digits[1:] if nd > 1 else "")
                + ("e-" if x < 0 else "e+") + f"{abs(x):02d}")
    if decpt <= 0:
        return out + "0." + "0" * -decpt + digits
    if decpt < nd:
        return out + digits[:decpt] + "." + digits[decpt:]
    return out + digits + "0" * (decpt - nd) + ".0"


def check_f64_repr(n: int, seed: int = 5) -> int:
    """f64_repr == repr() on random bit patterns, random decimals and edge cases."""
    import random
    import struct
    rng = random.Random(seed)
    cases = [0x0000000000000001, 0x000FFFFFFFFFFFFF, 0x0010000000000000, 0x7FEFFFFFFFFFFFFF,
             0x3FF0000000000000, 0x4340000000000000, 0x3CB0000000000000, 0x0020000000000000]
    for x in (0.1, 0.2, 0.3, 1e16, 1e17, 9007199254740993.0, 5e-324, 1.7976931348623157e308,
              2.2250738585072014e-308, 1e-5, 1e-4, 123456789012345680.0, 0.30000000000000004,
              1.5, 100000.0, 1e22, 1e23, 2 ** 63, 2 ** 64, 4.35, 0.001, 9.999999999999999e22):
        cases.append(struct.unpack("<Q", struct.pack("<d", x))[0])
    for _ in range(n):
        cases.append(rng.getrandbits(64))
        d = rng.choice([1, 2, 3, 5, 8, 12, 15, 16, 17, 18, 20])
        cases.append(struct.unpack("<Q", struct.pack(
            "<d", float(f"{rng.randrange(10 ** d)}e{rng.randrange(-330, 310)}")))[0])
    checked = 0
    for b in cases:
        x = struct.unpack("<d", struct.pack("<Q", b))[0]
        want = repr(x)
        got = f64_repr(b)
        if got != want:
            raise AssertionError(f"f64_repr({b:#018x}) = {got!r}, repr = {want!r}")
        checked += 1
    return checked
