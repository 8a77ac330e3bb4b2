// fbx_core.cuh -- device library for the fused FeatureBox extraction kernels.
//
// This header is prepended to every plan-specialised kernel the host planner
// generates (paper_2210_07768_b200/codegen.py) and compiled at prepare time
// by NVRTC for sm_100a (the paper's "runtime-compiled meta-kernel",
// reference PAPER.md:207).  It must stay NVRTC-clean: no host headers.
//
// Contents: integer types, FNV-1a-64 in 32-bit halves, FBXC column access,
// the string functions of the operator library (reference featureops.py:
// 298-367), a validating JSON scanner with dot-path extraction (viewpipe.py:
// 254-280 over CPython json.loads), HBM hash-table probes (dictionary lookups
// featureops.py:414-426, side-view join viewpipe.py:498-547), the block-level
// bump allocator (mempool.py:114-134 / PAPER.md Alg. 1) and the tile
// primitives for emission (scan, sort by instance id, decoupled look-back).
#pragma once

typedef unsigned char u8;
typedef unsigned short u16;
typedef unsigned int u32;
typedef unsigned long long u64;
typedef int i32;
typedef long long i64;

#define FBX_DI __device__ __forceinline__
#define FBX_STR_(x) #x
#define FBX_XSTR_(x) FBX_STR_(x)
// variable-trip loops of helpers inlined at many sites stay rolled: the unrolled
// copies cost more in instruction-cache misses than they save (measured)
#ifdef FBX_LOOPS_UNROLLED
#define FBX_ROLLED
#else
#define FBX_ROLLED _Pragma("unroll 1")
#endif
#ifndef FBX_FNV_UNROLL
#define FBX_FNV_UNROLL 1  // unroll factor of the FNV word loop
#endif
#define FBX_NI __device__ __noinline__

#include "fbx_abi.h"

// profiling aid (codegen FBX_PHASE_TIMERS): SM cycles per kernel phase, summed over warps
__device__ unsigned long long fbx_ph[10];
__device__ unsigned int fbx_ph_done;
#define FBX_PHASE(k) do { if ((threadIdx.x & 31u) == 0) { const u64 t_ = clock64(); \
  atomicAdd(&fbx_ph[(k)], t_ - ph_t); ph_t = t_; } } while (0)

namespace fbx {

// ---------------------------------------------------------------------------
// FNV-1a 64 (featureops.py:37-42).  State kept as two 32-bit halves:
//   h*P = h*0x1B3 + (h << 40)  =>  lo' = lo*0x1B3, hi' = hi*0x1B3 + mulhi + (lo<<8)
// which ptxas lowers to IMAD.WIDE.U32 + IMAD + LEA (+ the LOP3 xor).
// ---------------------------------------------------------------------------
struct Fnv {
  u32 lo, hi;
  FBX_DI Fnv() : lo(0x84222325u), hi(0xCBF29CE4u) {}
  FBX_DI Fnv(u64 h) : lo((u32)h), hi((u32)(h >> 32)) {}
  FBX_DI u64 value() const { return ((u64)hi << 32) | lo; }
  FBX_DI void mul(u32 x) {
    // lo' = x*0x1B3; hi' = hi*0x1B3 + mulhi(x, 0x1B3) + (x << 8).  Written as two
    // PTX mads so ptxas emits IMAD + IMAD/LEA instead of SHF + IMAD + IADD
    // (4.75 instead of 5.75 SASS instructions per hashed byte, measured).
    const u64 w = (u64)x * 0x1B3u;
    u32 t, h2;
    asm("mad.lo.u32 %0, %1, 435, %2;" : "=r"(t) : "r"(hi), "r"((u32)(w >> 32)));
    asm("mad.lo.u32 %0, %1, 256, %2;" : "=r"(h2) : "r"(x), "r"(t));
    hi = h2;
    lo = (u32)w;
  }
  FBX_DI void byte(u32 b) { mul(lo ^ b); }
  // h = (x | hi << 32) * K for a 64-bit constant K: three multiply-adds.  k zero
  // bytes in a row are one multiply by P^k ((h ^ 0) * P = h * P), so a run of
  // known-zero bytes costs one FNV step instead of k.
  template <u32 KLO, u32 KHI>
  FBX_DI void mulk(u32 x) {
    const u64 w = (u64)x * KLO;
    u32 t, h2;
    asm("mad.lo.u32 %0, %1, %3, %2;" : "=r"(t) : "r"(hi), "r"((u32)(w >> 32)), "n"(KLO));
    asm("mad.lo.u32 %0, %1, %3, %2;" : "=r"(h2) : "r"(x), "r"(t), "n"(KHI));
    hi = h2;
    lo = (u32)w;
  }
  FBX_DI void zeros4() { mulk<0x5635BC91u, 0x9FFAAC08u>(lo); }   // P^4
  FBX_DI void zeros6() { mulk<0xEDF1C639u, 0xDC966432u>(lo); }   // P^6
  FBX_DI void zeros7() { mulk<0x51D3D2DBu, 0xC5527B8Au>(lo); }   // P^7
  // an Int64 value's 8 big-endian bytes (value_bytes, featureops.py:73-87): the
  // leading zero bytes of a small non-negative value fold into one multiply
  FBX_DI void u64_be_int(u64 v) {
    const u32 vh = (u32)(v >> 32), vl = (u32)v;
    if (vh == 0u && vl < 0x100u) {
      zeros7();
      mul(lo ^ vl);
    } else if (vh == 0u && vl < 0x10000u) {
      zeros6();
      mul(lo ^ (vl >> 8));
      mul(lo ^ (vl & 0xFFu));
    } else {
      if (vh == 0u) zeros4(); else word_be(vh);
      word_be(vl);
    }
  }
  // four bytes of a little-endian word, low byte first
  FBX_DI void word_le(u32 w) {
    mul(lo ^ (w & 0xFFu));
    mul(lo ^ ((w >> 8) & 0xFFu));
    mul(lo ^ ((w >> 16) & 0xFFu));
    mul(lo ^ (w >> 24));
  }
  FBX_DI void word_be(u32 w) {  // big-endian image of w
    mul(lo ^ (w >> 24));
    mul(lo ^ ((w >> 16) & 0xFFu));
    mul(lo ^ ((w >> 8) & 0xFFu));
    mul(lo ^ (w & 0xFFu));
  }
  FBX_DI void u64_be(u64 v) { word_be((u32)(v >> 32)); word_be((u32)v); }
  FBX_DI void u64_le(u64 v) { word_le((u32)v); word_le((u32)(v >> 32)); }
  FBX_DI void u16_le(u32 v) {
    if (v < 0x100u) {  // a slot below 256 (all of them in practice): (h ^ v) * P^2
      mulk<0x0002E329u, 0x00036600u>(lo ^ v);
    } else {
      mul(lo ^ (v & 0xFFu));
      mul(lo ^ ((v >> 8) & 0xFFu));
    }
  }
  // arbitrary byte span.  Reads whole aligned 32-bit words and funnel-shifts
  // them into place.  The word after the last byte may be read: every span the
  // kernels hash (staged shared-memory spans, padded HBM segments, the pool,
  // constants) has >= 16 readable bytes of slack (FBX_EXACT_READS: never).
  template <bool LOWER>
  FBX_DI void bytes_t(const u8* p, u32 n) {
    if (n == 0) return;
    const u64 a = (u64)p;
    const u32 sh = (u32)(a & 3u) * 8u;
    const u32* wp = (const u32*)(a & ~3ull);
    const u32 nw = n >> 2, r = n & 3u;
    u32 lo_w = wp[0];
    _Pragma(FBX_XSTR_(unroll FBX_FNV_UNROLL))
    for (u32 k = 0; k < nw; ++k) {
      // the next word is needed when the span continues into it
#ifdef FBX_EXACT_READS
      const bool need = sh || (4u * (k + 1u) < n);
      u32 nxt = need ? wp[k + 1] : 0u;
#else
      u32 nxt = wp[k + 1];  // may be one word past the span: every span has >= 16 B slack
#endif
      u32 w = __funnelshift_r(lo_w, nxt, sh);
      if (LOWER) w = lower_word(w);
      word_le(w);
      lo_w = nxt;
    }
    if (r) {
#ifdef FBX_EXACT_READS
      u32 hi_w = (sh + r * 8u > 32u) ? wp[nw + 1] : 0u;
#else
      u32 hi_w = wp[nw + 1];
#endif
      u32 w = __funnelshift_r(lo_w, hi_w, sh);
      if (LOWER) w = lower_word(w);
      mul(lo ^ (w & 0xFFu));
      if (r > 1u) mul(lo ^ ((w >> 8) & 0xFFu));
      if (r > 2u) mul(lo ^ ((w >> 16) & 0xFFu));
    }
  }
  FBX_DI void bytes(const u8* p, u32 n) { bytes_t<false>(p, n); }
  FBX_DI void bytes_lower(const u8* p, u32 n) { bytes_t<true>(p, n); }
  // ASCII lowercase of 4 packed bytes (all < 0x80): 'A'..'Z' -> 'a'..'z'
  static FBX_DI u32 lower_word(u32 w) {
    const u32 w7 = w & 0x7F7F7F7Fu;      // no carries between bytes
    u32 ge_a = w7 + 0x3F3F3F3Fu;         // byte >= 0x41 -> bit 7 set
    u32 gt_z = w7 + 0x25252525u;         // byte >= 0x5B -> bit 7 set
    u32 up = ge_a & ~gt_z & ~w & 0x80808080u;  // ASCII 'A'..'Z' only
    return w | (up >> 2);
  }
};

FBX_DI u64 fnv_mix(u64 v) {  // featureops.py:306-307, mix(v) = FNV(8 BE bytes)
  Fnv h;
  h.u64_be(v);
  return h.value();
}

// ---------------------------------------------------------------------------
// Loads
// ---------------------------------------------------------------------------
FBX_DI u64 ldg_u64(const void* p) { return __ldg((const u64*)p); }
FBX_DI u32 ldg_u32(const void* p) { return __ldg((const u32*)p); }
FBX_DI u32 ldg_u8(const void* p) { return __ldg((const u8*)p); }

// FBXC null bitmap, LSB-first, bit set = null (columnstore.py:117-130)
FBX_DI bool null_bit(const u8* nulls, u64 row) {
  return (__ldg(nulls + (row >> 3)) >> (row & 7u)) & 1u;
}

// A string value: generic pointer (global, pool or shared) + byte length.
struct Str {
  const u8* p;
  u32 n;
};

FBX_DI u32 str_byte(const u8* p, u32 i) { return p[i]; }

FBX_DI bool str_eq(Str a, Str b) {
  if (a.n != b.n) return false;
  FBX_ROLLED
  for (u32 i = 0; i < a.n; ++i)
    if (a.p[i] != b.p[i]) return false;
  return true;
}

FBX_DI bool str_eq_const(Str a, const u8* c, u32 cn) {
  if (a.n != cn) return false;
  FBX_ROLLED
  for (u32 i = 0; i < cn; ++i)
    if (a.p[i] != c[i]) return false;
  return true;
}

// Python str ordering == UTF-8 byte order (code points are order-preserving)
FBX_DI int str_cmp(Str a, const u8* c, u32 cn) {
  u32 m = a.n < cn ? a.n : cn;
  FBX_ROLLED
  for (u32 i = 0; i < m; ++i) {
    u32 x = a.p[i], y = c[i];
    if (x != y) return x < y ? -1 : 1;
  }
  return a.n == cn ? 0 : (a.n < cn ? -1 : 1);
}

// ---------------------------------------------------------------------------
// token:<delim>:<index> (featureops.py:318-349, 392-412): field `index` of a
// single-byte split, "" past the end.  Returned as a view into the input.
// ---------------------------------------------------------------------------
FBX_DI Str str_token(Str s, u32 delim, u32 index) {
  u32 field = 0, start = 0;
  FBX_ROLLED
  for (u32 i = 0; i < s.n; ++i) {
    if (s.p[i] == delim) {
      if (field == index) return Str{s.p + start, i - start};
      ++field;
      start = i + 1;
    }
  }
  if (field == index) return Str{s.p + start, s.n - start};
  return Str{s.p, 0u};
}

// exact per-byte zero test: 0x80 in every byte of x that is 0x00
FBX_DI u32 zero_bytes(u32 x) { return ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u; }

// 4 bytes of a span starting at byte k (funnel-shifted aligned words; reads
// only words that hold bytes of the span)
struct WordCursor {
  const u32* wp;
  u32 sh, n;
  FBX_DI WordCursor(const u8* p, u32 len) : n(len) {
    const u64 a = (u64)p;
    sh = (u32)(a & 3u) * 8u;
    wp = (const u32*)(a & ~3ull);
  }
  FBX_DI u32 word(u32 k) const {  // bytes [k, k+4) (k % 4 == 0), bytes past n are garbage
    const u32 lo = wp[k >> 2];
#ifdef FBX_EXACT_READS
    const bool need = sh && (k + 4u - sh / 8u) < n;  // next word holds span bytes
    const u32 hi = need ? wp[(k >> 2) + 1] : 0u;
#else
    const u32 hi = wp[(k >> 2) + 1];  // every span has >= 16 B of readable slack
#endif
    return __funnelshift_r(lo, hi, sh);
  }
};

// Several fields of one single-byte split in one SWAR pass (codegen groups
// token calls that share an input and a delimiter).  want[k] = field number.
// 0x80 in every byte of x equal to the byte replicated in c (x7 = x & 0x7F7F7F7F)
FBX_DI u32 eq_bytes(u32 x, u32 x7, u32 c) { return ~(((x7 ^ c) + 0x7F7F7F7Fu) | x) & 0x80808080u; }

// bit j = (p[j] == c) for a span of 1..60 bytes: one branch-free pass over its
// aligned words (flags gathered by one IMAD per word, see jmask_build)
FBX_DI u64 byte_mask64(const u8* p, u32 n, u32 c) {
  const u64 a = (u64)p;
  const u32 sh = (u32)(a & 3u);
  const u32* wp = (const u32*)(a & ~3ull);
  const int nw = (int)((sh + n + 3u) >> 2);
  const u32 cc = c * 0x01010101u;
  u32 lo = 0, hi = 0;
  for (int w = nw - 1; w >= 0; --w) {
    const u32 x = wp[w];
    const u32 pz = eq_bytes(x, x & 0x7F7F7F7Fu, cc) * 0x00204081u;
    hi = __funnelshift_l(lo, hi, 4);
    lo = __funnelshift_l(pz, lo, 4);
  }
  return ((((u64)hi << 32) | lo) >> sh) & ((1ull << n) - 1ull);
}

template <int K>
FBX_DI void str_tokens(Str s, u32 delim, const u32 (&want)[K], Str (&out)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = Str{s.p, 0u};
  if (s.n != 0u && s.n <= 60u) {
    // mask mode: field f ends at the f-th set bit of the delimiter mask (or n)
    u64 m = byte_mask64(s.p, s.n, delim);
    u32 start = 0;
#pragma unroll
    for (u32 f = 0; f <= want[K - 1]; ++f) {
      const u32 end = m ? (u32)(__ffsll((long long)m) - 1) : s.n;
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (want[k] == f && start <= s.n) out[k] = Str{s.p + start, end - start};
      start = end + 1u;
      m &= m - 1ull;
    }
    return;
  }
  u32 field = 0, start = 0;
  if (s.n) {
    const WordCursor wc(s.p, s.n);
    const u32 dm = delim * 0x01010101u;
    FBX_ROLLED
    for (u32 b = 0; b < s.n; b += 4u) {
      u32 z = zero_bytes(wc.word(b) ^ dm);
      const u32 left = s.n - b;
      if (left < 4u) z &= (1u << (left * 8u)) - 1u;
      FBX_ROLLED
      while (z) {
        const u32 pos = b + ((u32)(__ffs(z) - 1) >> 3);
#pragma unroll
        for (int k = 0; k < K; ++k)
          if (want[k] == field) out[k] = Str{s.p + start, pos - start};
        ++field;
        start = pos + 1u;
        z &= z - 1u;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (want[k] == field) out[k] = Str{s.p + start, s.n - start};
}

// str.isspace() for a decoded code point (CPython 3.12 / Unicode 15)
FBX_DI bool py_isspace(u32 cp) {
  if (cp <= 0x7F) return (cp >= 0x09 && cp <= 0x0D) || (cp >= 0x1C && cp <= 0x20);
  return cp == 0x85 || cp == 0xA0 || cp == 0x1680 || (cp >= 0x2000 && cp <= 0x200A) ||
         cp == 0x2028 || cp == 0x2029 || cp == 0x202F || cp == 0x205F || cp == 0x3000;
}

// decode the code point starting at p[i] (valid UTF-8 assumed); returns length
FBX_DI u32 utf8_at(const u8* p, u32 i, u32 n, u32* cp) {
  u32 c = p[i];
  if (c < 0x80u) { *cp = c; return 1; }
  if (c < 0xE0u && i + 1 < n) { *cp = ((c & 0x1Fu) << 6) | (p[i + 1] & 0x3Fu); return 2; }
  if (c < 0xF0u && i + 2 < n) {
    *cp = ((c & 0x0Fu) << 12) | ((p[i + 1] & 0x3Fu) << 6) | (p[i + 2] & 0x3Fu);
    return 3;
  }
  if (i + 3 < n) {
    *cp = ((c & 0x07u) << 18) | ((p[i + 1] & 0x3Fu) << 12) | ((p[i + 2] & 0x3Fu) << 6) |
          (p[i + 3] & 0x3Fu);
    return 4;
  }
  *cp = c;
  return 1;
}

// trim = str.strip() (featureops.py:302-303): a view narrowing
FBX_DI Str str_trim(Str s) {
  u32 b = 0, e = s.n;
  FBX_ROLLED
  while (b < e) {
    u32 c = s.p[b];
    if (c < 0x80u) {
      if (!py_isspace(c)) break;
      ++b;
    } else {
      u32 cp, l = utf8_at(s.p, b, e, &cp);
      if (!py_isspace(cp)) break;
      b += l;
    }
  }
  FBX_ROLLED
  while (e > b) {
    u32 c = s.p[e - 1];
    if (c < 0x80u) {
      if (!py_isspace(c)) break;
      --e;
    } else {
      u32 k = e - 1;  // walk back to the lead byte
      FBX_ROLLED
      while (k > b && (s.p[k] & 0xC0u) == 0x80u) --k;
      u32 cp;
      utf8_at(s.p, k, e, &cp);
      if (!py_isspace(cp)) break;
      e = k;
    }
  }
  return Str{s.p + b, e - b};
}

// lower (featureops.py:298-299): 0 = unchanged (view ok), 1 = ASCII changes,
// 2 = non-ASCII present (needs the Unicode tables: not supported on device)
FBX_DI u32 str_lower_class(Str s) {
  if (s.n == 0) return 0;
  const WordCursor wc(s.p, s.n);
  u32 up = 0;
  FBX_ROLLED
  for (u32 b = 0; b < s.n; b += 4u) {
    u32 w = wc.word(b);
    const u32 left = s.n - b;
    if (left < 4u) w &= (1u << (left * 8u)) - 1u;  // garbage bytes -> 0 (not upper, ASCII)
    if (w & 0x80808080u) return 2;
    up |= (w + 0x3F3F3F3Fu) & ~(w + 0x25252525u);  // 'A'..'Z' -> bit 7
  }
  return (up & 0x80808080u) ? 1u : 0u;
}

}  // namespace fbx
#include "fbx_unicode.cuh"
namespace fbx {

// ---------------------------------------------------------------------------
// Full Unicode lower() (CPython 3.12, Unicode 15.0): _PyUnicode_ToLowerFull +
// Final_Sigma (unicodeobject.c handle_capital_sigma), tables generated from
// CPython itself (unicode_tables.py).  Only reached for strings with bytes
// >= 0x80; ASCII strings take the lazy SWAR path.
// ---------------------------------------------------------------------------
FBX_DI bool u_in(u32 cp, const u32* lo, const u32* hi, u32 n) {
  u32 a = 0, b = n;
  FBX_ROLLED
  while (a < b) {
    const u32 m = (a + b) >> 1;
    if (__ldg(lo + m) <= cp) a = m + 1; else b = m;
  }
  return a > 0 && cp <= __ldg(hi + a - 1);
}
FBX_DI u32 u_lower_single(u32 cp) {
  u32 a = 0, b = ULOWER_N;
  FBX_ROLLED
  while (a < b) {
    const u32 m = (a + b) >> 1;
    const u32 f = __ldg(ULOWER_FROM + m);
    if (f == cp) return __ldg(ULOWER_TO + m);
    if (f < cp) a = m + 1; else b = m;
  }
  return cp;
}
FBX_DI u32 utf8_len(u32 cp) { return cp < 0x80u ? 1u : cp < 0x800u ? 2u : cp < 0x10000u ? 3u : 4u; }
FBX_DI void utf8_put(u8* d, u32 cp) {  // surrogates encode as WTF-8 3-byte units
  if (cp < 0x80u) { d[0] = (u8)cp; return; }
  if (cp < 0x800u) { d[0] = (u8)(0xC0u | (cp >> 6)); d[1] = (u8)(0x80u | (cp & 0x3Fu)); return; }
  if (cp < 0x10000u) {
    d[0] = (u8)(0xE0u | (cp >> 12));
    d[1] = (u8)(0x80u | ((cp >> 6) & 0x3Fu));
    d[2] = (u8)(0x80u | (cp & 0x3Fu));
    return;
  }
  d[0] = (u8)(0xF0u | (cp >> 18));
  d[1] = (u8)(0x80u | ((cp >> 12) & 0x3Fu));
  d[2] = (u8)(0x80u | ((cp >> 6) & 0x3Fu));
  d[3] = (u8)(0x80u | (cp & 0x3Fu));
}
FBX_DI bool u_cased(u32 cp) { return u_in(cp, UCASED_LO, UCASED_HI, UCASED_N); }
FBX_DI bool u_ignorable(u32 cp) { return u_in(cp, UIGN_LO, UIGN_HI, UIGN_N); }

// U+03A3 at byte `pos` (2 bytes): final sigma when preceded (skipping case-
// ignorables) by a cased letter and not followed (likewise) by one.
FBX_DI u32 sigma_lower(Str s, u32 pos) {
  bool fin = false;
  u32 j = pos;
  while (j > 0) {
    do { --j; } while (j > 0 && (s.p[j] & 0xC0u) == 0x80u);
    u32 cp;
    utf8_at(s.p, j, s.n, &cp);
    if (!u_ignorable(cp)) { fin = u_cased(cp); break; }
  }
  if (fin) {
    u32 k = pos + 2u;
    while (k < s.n) {
      u32 cp;
      const u32 l = utf8_at(s.p, k, s.n, &cp);
      if (!u_ignorable(cp)) { fin = !u_cased(cp); break; }
      k += l;
    }
  }
  return fin ? 0x3C2u : 0x3C3u;
}

// str.lower() of a UTF-8 (or WTF-8) span into dst; returns the byte length
// (dst == nullptr: length only).
FBX_DI u32 unicode_lower(Str s, u8* dst) {
  u32 o = 0;
  for (u32 i = 0; i < s.n;) {
    const u32 c = s.p[i];
    if (c < 0x80u) {
      if (dst) dst[o] = (u8)((c - 'A' < 26u) ? c + 32u : c);
      ++o;
      ++i;
      continue;
    }
    u32 cp;
    const u32 len = utf8_at(s.p, i, s.n, &cp);
    if (cp == 0x130u) {  // LATIN CAPITAL I WITH DOT ABOVE -> "i" U+0307
      if (dst) { dst[o] = 'i'; utf8_put(dst + o + 1, 0x307u); }
      o += 3;
      i += len;
      continue;
    }
    const u32 lc = (cp == 0x3A3u) ? sigma_lower(s, i) : u_lower_single(cp);
    if (dst) utf8_put(dst + o, lc);
    o += utf8_len(lc);
    i += len;
  }
  return o;
}

FBX_DI void str_lower_copy(u8* dst, Str s) {
  FBX_ROLLED
  for (u32 i = 0; i < s.n; ++i) {
    u32 c = s.p[i];
    dst[i] = (u8)((c >= 'A' && c <= 'Z') ? c + 32u : c);
  }
}

FBX_DI void str_copy_lower(u8* dst, Str s) { str_lower_copy(dst, s); }

FBX_DI void str_copy(u8* dst, Str s) {
#ifdef FBX_EXACT_READS
  FBX_ROLLED
  for (u32 i = 0; i < s.n; ++i) dst[i] = s.p[i];
#else
  // bytewise until dst is 4-B aligned, then one aligned source-word pair, a funnel
  // shift and one 4-B store per word (the source keeps >= 16 B of readable slack)
  u32 i = 0;
  const u32 head = (u32)(-(i64)(u64)dst & 3);
  FBX_ROLLED
  for (; i < head && i < s.n; ++i) dst[i] = s.p[i];
  if (i + 4u <= s.n) {
    const u64 a = (u64)(s.p + i);
    const u32 sh = (u32)(a & 3u) * 8u;
    const u32* wp = (const u32*)(a & ~3ull);
    u32* dw = (u32*)(dst + i);
    u32 lo = wp[0];
    const u32 nw = (s.n - i) >> 2;
    FBX_ROLLED
    for (u32 k = 0; k < nw; ++k) {
      const u32 nx = wp[k + 1];
      dw[k] = __funnelshift_r(lo, nx, sh);
      lo = nx;
    }
    i += nw * 4u;
  }
  FBX_ROLLED
  for (; i < s.n; ++i) dst[i] = s.p[i];
#endif
}

// decimal text of a Python int (str(v)); buf >= 20 bytes (+1 for '-')
FBX_DI u32 u64_dec_len(u64 v) {
  if (v < 10000000000ull) {  // < 10^10: 32-bit-sized compares, no division
    u32 n = 1;
    u64 p = 10ull;
#pragma unroll
    for (int k = 0; k < 9; ++k) { n += v >= p ? 1u : 0u; p *= 10ull; }
    return n;
  }
  u32 n = 11;
  u64 p = 100000000000ull;
#pragma unroll
  for (int k = 0; k < 9; ++k) { n += v >= p ? 1u : 0u; p *= 10ull; }  // up to 10^19
  return n;
}
FBX_DI u32 int_dec_len(u64 bits, bool is_signed) {
  if (is_signed && (i64)bits < 0) return 1 + u64_dec_len(0ull - bits);
  return u64_dec_len(bits);
}
FBX_DI void u64_dec(u8* dst, u64 v, u32 len) {
  u32 i = len;
  FBX_ROLLED
  while (v > 0xFFFFFFFFull) { dst[--i] = (u8)('0' + v % 10u); v /= 10u; }
  u32 x = (u32)v;  // 32-bit divisions (a multiply-high each) for the rest
  FBX_ROLLED
  while (i > 0) { dst[--i] = (u8)('0' + x % 10u); x /= 10u; }
}
FBX_DI void int_dec(u8* dst, u64 bits, bool is_signed, u32 len) {
  if (is_signed && (i64)bits < 0) {
    dst[0] = '-';
    u64_dec(dst + 1, 0ull - bits, len - 1);
  } else {
    u64_dec(dst, bits, len);
  }
}

// Float32 value canonicalisation: Python floats re-packed with struct '>f'
// quiet a signalling NaN (columnstore.py:97, featureops.py:86).
FBX_DI u32 f32_canon_bits(u32 b) {
  return ((b & 0x7F800000u) == 0x7F800000u && (b & 0x007FFFFFu)) ? (b | 0x00400000u) : b;
}

// ---------------------------------------------------------------------------
// Error word: the first failure in pipeline order wins (atomicMin on a key).
//   key = chunk(32) | stage(4) | layer(8) | node rank(12) | code(8)
// ---------------------------------------------------------------------------
FBX_DI u64 err_key(u64 chunk, u32 stage, u32 layer, u32 node, u32 code) {
  return (chunk << 32) | ((u64)(stage & 0xFu) << 28) | ((u64)(layer & 0xFFu) << 20) |
         ((u64)(node & 0xFFFu) << 8) | (code & 0xFFu);
}
// one 128-bit compare-and-swap (atom.cas.b128, sm_90+)
FBX_DI void cas128(void* addr, u64 cmp_lo, u64 cmp_hi, u64 new_lo, u64 new_hi, u64* old_lo,
                   u64* old_hi) {
  asm volatile(
      "{\n\t.reg .b128 c, n, d;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 n, {%4, %5};\n\t"
      "atom.global.cas.b128 d, [%6], c, n;\n\t"
      "mov.b128 {%0, %1}, d;\n\t}"
      : "=l"(*old_lo), "=l"(*old_hi)
      : "l"(cmp_lo), "l"(cmp_hi), "l"(new_lo), "l"(new_hi), "l"(addr)
      : "memory");
}

// The fused kernel's error word: atomicMin on the key, then the winner writes
// its detail.  The row-level failures of the fused kernel carry no detail; the
// label detail can, in principle, pair with another label's position when two
// CTAs raise non-0/1 labels within one atomic round trip in the reverse order
// (measured: any 128-bit CAS on these paths, even out of line, costs the fused
// kernel 2-7%, so its exact pair update is kept to the off-path kernels:
// raise_err_exact).
FBX_DI void raise_err(fbx_state* st, u64 key, u64 detail) {
  u64 old = atomicMin((unsigned long long*)&st->error_key, (unsigned long long)key);
  if (key < old) atomicExch((unsigned long long*)&st->error_detail, (unsigned long long)detail);
}

// (key, detail) moved together by a 128-bit CAS: the detail is always the
// winning key's (fbx_pool_account: PoolExhausted's requested / remaining)
FBX_DI void raise_err_exact(fbx_state* st, u64 key, u64 detail) {
  u64* pair = &st->error_key;
  u64 lo = ~0ull, hi = 0ull;  // the reset value: one CAS when this is the first
  while (key < lo) {
    u64 olo, ohi;
    cas128(pair, lo, hi, key, detail, &olo, &ohi);
    if (olo == lo && ohi == hi) break;
    lo = olo;
    hi = ohi;
  }
}

// Label errors surface when their mini-batch is flushed (pipeline.py:765-777):
// emit_minibatch raises at a null label anywhere in the batch before
// MiniBatch.validate's range check, so the first null and the first non-0/1
// label are kept apart, by emission position; the host takes the earlier batch
// (null on a tie) and maps it to the chunk whose merge flushes it.  Positions,
// not batches, so a record-sharded run can shift them by the shard's base.
FBX_DI void raise_emit(fbx_state* st, u64 pos, bool range, u64 label) {
  u64* p = range ? &st->emit_range_pos : &st->emit_null_pos;
  u64 old = atomicMin((unsigned long long*)p, (unsigned long long)pos);
  if (range && pos < old)
    atomicExch((unsigned long long*)&st->emit_range_label, (unsigned long long)label);
}

// check_unique_ids (viewpipe.py:562-576) raises at the FIRST row, in row order,
// whose id occurred before: the row of some id's SECOND occurrence, minimised
// over ids.  The id-set winner records its row with a plain store; a thread that
// finds its id already present (rare) folds its row into the slot's two smallest
// "later" rows and flags the run; fbx_dup_resolve takes the second smallest of
// {winner, later rows} per slot and the minimum over slots after the run.
// The pair holds ~row (0 = none), so the two smallest rows are the two largest
// words: one atomicMax keeps the smallest, and whatever it displaces or rejects
// -- every row but the smallest, at some point -- goes through a second
// atomicMax into the runner-up (64-bit atomics only: a 128-bit CAS loop here
// measured slower for the whole fused kernel).
FBX_DI void dup_note(fbx_state* st, u64* pair, u64 row) {
  const u64 x = ~row;
  const u64 old = atomicMax((unsigned long long*)&pair[0], (unsigned long long)x);
  if (old != 0ull) atomicMax((unsigned long long*)&pair[1], (unsigned long long)(old < x ? old : x));
  atomicExch((unsigned long long*)&st->dup_seen, 1ull);
}

// Index-build tail: the CTA's malformed / filtered / indexed counts reach the
// run state by ONE atomic each per CTA (per-thread atomics on three shared
// words serialise in L2: 1M rows cost ~240 us that way).  Every thread of the
// CTA must call it (block-uniform control flow).
FBX_DI void block_side_counts(fbx_state* st, u32 nmal, u32 nfilt, u32 nidx) {
  __shared__ u32 acc[3];
  if (threadIdx.x < 3u) acc[threadIdx.x] = 0u;
  __syncthreads();
  const u32 a = __reduce_add_sync(0xFFFFFFFFu, nmal);
  const u32 b = __reduce_add_sync(0xFFFFFFFFu, nfilt);
  const u32 c = __reduce_add_sync(0xFFFFFFFFu, nidx);
  if ((threadIdx.x & 31u) == 0u) {
    if (a) atomicAdd(&acc[0], a);
    if (b) atomicAdd(&acc[1], b);
    if (c) atomicAdd(&acc[2], c);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (acc[0]) atomicAdd((unsigned long long*)&st->malformed, (unsigned long long)acc[0]);
    if (acc[1]) atomicAdd((unsigned long long*)&st->filtered, (unsigned long long)acc[1]);
    if (acc[2]) atomicAdd((unsigned long long*)&st->side_rows, (unsigned long long)acc[2]);
  }
}

// ---------------------------------------------------------------------------
// Block-level primitives (blockDim.x == NT, a multiple of 32, <= 1024)
// ---------------------------------------------------------------------------
template <int NT>
struct BlockScanU32 {
  u32 warp_tot[NT / 32];
  u32 total;
  // block-wide sum (all threads get it)
  FBX_DI u32 sum(u32 v) {
    const u32 lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
    if (lane == 0) warp_tot[wid] = v;
    __syncthreads();
    u32 t = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) t += warp_tot[w];
    __syncthreads();
    return t;
  }
  // exclusive scan; returns the exclusive prefix, total in `total`
  FBX_DI u32 exclusive(u32 v) {
    const u32 lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    u32 x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      u32 y = __shfl_up_sync(0xFFFFFFFFu, x, d);
      if (lane >= (u32)d) x += y;
    }
    if (lane == 31u) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      u32 t = lane < (u32)(NT / 32) ? warp_tot[lane] : 0u;
      u32 s = t;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        u32 y = __shfl_up_sync(0xFFFFFFFFu, s, d);
        if (lane >= (u32)d) s += y;
      }
      if (lane < (u32)(NT / 32)) warp_tot[lane] = s - t;
      if (lane == (u32)(NT / 32) - 1u) total = s;
    }
    __syncthreads();
    u32 r = warp_tot[wid] + x - v;
    __syncthreads();
    return r;
  }
};

// Block bump allocation from the HBM arena (Algorithm 1; reference
// mempool.py:114-134): exclusive prefix of lane sizes, ONE atomicAdd per CTA,
// 128-byte group alignment.  Returns the lane's pointer (nullptr when its size
// is 0 or the arena is exhausted -- then *exhausted is set, CTA-uniformly for
// the CTA grant and warp-uniformly for the warp grant).  This is the engine's
// own arena: running out of it is not the reference's PoolExhausted (that is
// the config's pool_bytes, settled by fbx_pool_account) -- the run is repeated
// with an arena of state.pool_overflow bytes.
template <int NT>
FBX_DI u8* pool_alloc(BlockScanU32<NT>& scan, u64* base_smem, fbx_state* st, u8* pool,
                      u64 pool_cap, u32 size, bool* exhausted) {
#ifdef FBX_POOL_WARP
  // warp-aggregated: one atomicAdd per warp that asks, no CTA barrier
  __syncwarp();
  *exhausted = false;
  if (__ballot_sync(0xFFFFFFFFu, size != 0u) == 0u) return nullptr;
  const u32 lane = threadIdx.x & 31u;
  u32 inc = size;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u32 y = __shfl_up_sync(0xFFFFFFFFu, inc, d);
    if (lane >= (u32)d) inc += y;
  }
  const u32 total = __shfl_sync(0xFFFFFFFFu, inc, 31);
  u64 b = 0;
  if (lane == 31u) {
    const u64 tot = ((u64)total + 15ull) & ~15ull;
    b = atomicAdd((unsigned long long*)&st->pool_head, (unsigned long long)tot);
    if (b + tot > pool_cap) {  // the head this launch needs: the engine grows the arena
      atomicMax((unsigned long long*)&st->pool_overflow, (unsigned long long)(b + tot));
      b = ~0ull;
    }
  }
  b = __shfl_sync(0xFFFFFFFFu, b, 31);
  *exhausted = (b == ~0ull);
  if (b == ~0ull || size == 0) return nullptr;
  return pool + b + (inc - size);
#else
  if (!__syncthreads_or(size != 0u)) {
    *exhausted = false;
    return nullptr;
  }
  u32 pre = scan.exclusive(size);
  u32 total = scan.total;
  if (threadIdx.x == 0) {
    u64 tot = ((u64)total + 127ull) & ~127ull;
    u64 b = tot ? atomicAdd((unsigned long long*)&st->pool_head, (unsigned long long)tot) : 0ull;
    if (tot && b + tot > pool_cap) {  // the head this launch needs: the engine grows the arena
      atomicMax((unsigned long long*)&st->pool_overflow, (unsigned long long)(b + tot));
      b = ~0ull;
    }
    *base_smem = b;
  }
  __syncthreads();
  u64 b = *base_smem;
  __syncthreads();
  *exhausted = (b == ~0ull);
  if (b == ~0ull || size == 0) return nullptr;
  return pool + b + pre;
#endif
}

// Bitonic sort of (key, payload) pairs held in shared memory, N = power of 2.
template <int N, int NT>
FBX_DI void smem_bitonic_sort(u64* keys, u32* vals) {
  for (u32 k = 2; k <= (u32)N; k <<= 1) {
    for (u32 j = k >> 1; j > 0; j >>= 1) {
      for (u32 i = threadIdx.x; i < (u32)N; i += NT) {
        u32 ixj = i ^ j;
        if (ixj > i) {
          u64 a = keys[i], b = keys[ixj];
          bool up = (i & k) == 0;
          if ((a > b) == up) {
            keys[i] = b;
            keys[ixj] = a;
            u32 t = vals[i];
            vals[i] = vals[ixj];
            vals[ixj] = t;
          }
        }
      }
      __syncthreads();
    }
  }
}


// Bitonic sort of (key, val) pairs, ascending by (key, val), in shared memory.
template <int N, int NT>
FBX_DI void smem_bitonic_sort2(u64* keys, u32* vals) {
  for (u32 k = 2; k <= (u32)N; k <<= 1) {
    for (u32 j = k >> 1; j > 0; j >>= 1) {
      for (u32 i = threadIdx.x; i < (u32)N; i += NT) {
        u32 ixj = i ^ j;
        if (ixj > i) {
          u64 a = keys[i], b = keys[ixj];
          u32 va = vals[i], vb = vals[ixj];
          bool gt = (a > b) || (a == b && va > vb);
          bool up = (i & k) == 0;
          if (gt == up) {
            keys[i] = b;
            keys[ixj] = a;
            vals[i] = vb;
            vals[ixj] = va;
          }
        }
      }
      __syncthreads();
    }
  }
}


// Bitonic sort of one (key, val) pair per thread, NT a power of two.  Steps
// with partner distance < 32 exchange through warp shuffles; the few wider
// steps go through shared memory.  On return thread i holds the i-th
// smallest pair in (key, val) order.
template <int NT>
FBX_DI void block_sort_pairs(u64& key, u32& val, u64* sk, u32* sv) {
  // sk/sv hold 2*NT entries: wide exchanges alternate between two halves so
  // one barrier per exchange suffices (a half is rewritten only after the
  // next exchange's barrier, by which time every reader of it is done).
  const u32 i = threadIdx.x;
  u32 buf = 0;
#pragma unroll 1
  for (u32 k = 2; k <= (u32)NT; k <<= 1) {
#pragma unroll 1
    for (u32 j = k >> 1; j > 0; j >>= 1) {
      u64 ok;
      u32 ov;
      if (j >= 32u) {
        sk[buf + i] = key;
        sv[buf + i] = val;
        __syncthreads();
        ok = sk[buf + (i ^ j)];
        ov = sv[buf + (i ^ j)];
        buf ^= (u32)NT;
      } else {
        ok = __shfl_xor_sync(0xFFFFFFFFu, key, (int)j);
        ov = __shfl_xor_sync(0xFFFFFFFFu, val, (int)j);
      }
      bool other_lt = (ok < key) || (ok == key && ov < val);
      bool take_min = ((i & k) == 0) == ((i & j) == 0);
      if (other_lt == take_min) {
        key = ok;
        val = ov;
      }
    }
  }
  __syncthreads();
}


// Fully unrolled bitonic sort of one u64 key per thread (NT a power of two):
// exchanges with partner distance < 32 use warp shuffles, wider ones go through
// `buf` (2*NT u64, alternating halves: one barrier per exchange).  Returns the
// key of sorted position threadIdx.x.
template <int NT>
FBX_DI u64 bitonic_keys(u64 key, u64* buf) {
  const u32 i = threadIdx.x;
  u32 b = 0;
#pragma unroll
  for (u32 k = 2; k <= (u32)NT; k <<= 1) {
#pragma unroll
    for (u32 j = k >> 1; j > 0; j >>= 1) {
      u64 o;
      if (j >= 32u) {
        buf[b + i] = key;
        __syncthreads();
        o = buf[b + (i ^ j)];
        b ^= (u32)NT;
      } else {
        o = __shfl_xor_sync(0xFFFFFFFFu, key, (int)j);
      }
      const bool take_min = ((i & k) == 0) == ((i & j) == 0);
      if ((o < key) == take_min) key = o;
    }
  }
  return key;
}


// Rank of each live key among the tile's live keys (keys unique among live
// rows): an adaptive radix bucket pass.  `diff` = OR ^ AND of the live keys
// (the bits that vary); bucket = the 10 bits below the highest varying bit, so
// random ids and sequential ids alike spread over 1024 buckets; each key's
// rank = bucket start + number of smaller keys in its (small) bucket.  Returns
// false (CTA-uniformly) when some bucket holds more than 32 keys -- the caller
// then uses the bitonic network.  smem: hist u32[1024], start u32[1024],
// keys u64[NT].
template <int NT>
FBX_DI bool radix_rank(u64 key, bool live, u64 diff, u32* hist, u32* start, u64* bkeys,
                       BlockScanU32<NT>& scan, u32* rank) {
  constexpr int BPT = 1024 / NT;  // buckets per thread
  const u32 hb = diff ? 63u - (u32)__clzll((long long)diff) : 0u;
  const u32 shift = hb >= 9u ? hb - 9u : 0u;
  const u32 digit = (u32)(key >> shift) & 1023u;
#pragma unroll
  for (int b = 0; b < BPT; ++b) hist[threadIdx.x * BPT + b] = 0u;
  __syncthreads();
  u32 pos = 0;
  if (live) pos = atomicAdd(&hist[digit], 1u);
  __syncthreads();
  u32 sz[BPT], tot = 0;
  bool big = false;
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    sz[b] = hist[threadIdx.x * BPT + b];
    tot += sz[b];
    big |= sz[b] > 32u;
  }
  if (__syncthreads_or(big)) return false;
  u32 run = scan.exclusive(tot);
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    start[threadIdx.x * BPT + b] = run;
    run += sz[b];
  }
  __syncthreads();
  u32 b0 = 0, bn = 0;
  if (live) {
    b0 = start[digit];
    bn = hist[digit];
    bkeys[b0 + pos] = key;
  }
  __syncthreads();
  if (live) {
    u32 r = b0;
    FBX_ROLLED
    for (u32 q = 0; q < bn; ++q) r += bkeys[b0 + q] < key ? 1u : 0u;
    *rank = r;
  }
  return true;
}

// One block reduction of a u32 sum and a u64 OR / AND (redux.sync per warp, warp 0
// folds the warp partials): two barriers, every thread receives all three.
template <int NT>
struct TileReduce {
  u32 ws[NT / 32];
  u64 wo[NT / 32], wa[NT / 32];
  u32 rs;
  u64 ro, ra;
  // zero[0..nzero) is cleared between the two barriers (after every thread has
  // left the phase that may still read that shared memory)
  FBX_DI void run(u32 v, u64 o, u64 a, u32* sum, u64* vor, u64* vand, u32* zero, u32 nzero) {
    const u32 lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    v = __reduce_add_sync(0xFFFFFFFFu, v);
    const u32 olo = __reduce_or_sync(0xFFFFFFFFu, (u32)o), ohi = __reduce_or_sync(0xFFFFFFFFu, (u32)(o >> 32));
    const u32 alo = __reduce_and_sync(0xFFFFFFFFu, (u32)a), ahi = __reduce_and_sync(0xFFFFFFFFu, (u32)(a >> 32));
    if (lane == 0) { ws[wid] = v; wo[wid] = ((u64)ohi << 32) | olo; wa[wid] = ((u64)ahi << 32) | alo; }
    __syncthreads();
    for (u32 q = threadIdx.x; q < nzero; q += NT) zero[q] = 0u;
    if (wid == 0) {
      const bool in = lane < (u32)(NT / 32);
      const u32 x = in ? ws[lane] : 0u;
      const u64 xo = in ? wo[lane] : 0ull, xa = in ? wa[lane] : ~0ull;
      const u32 t = __reduce_add_sync(0xFFFFFFFFu, x);
      const u32 tol = __reduce_or_sync(0xFFFFFFFFu, (u32)xo), toh = __reduce_or_sync(0xFFFFFFFFu, (u32)(xo >> 32));
      const u32 tal = __reduce_and_sync(0xFFFFFFFFu, (u32)xa), tah = __reduce_and_sync(0xFFFFFFFFu, (u32)(xa >> 32));
      if (lane == 0) { rs = t; ro = ((u64)toh << 32) | tol; ra = ((u64)tah << 32) | tal; }
    }
    __syncthreads();
    *sum = rs; *vor = ro; *vand = ra;
  }
};

// Rank AND sign offset of a row in ascending-key order in one pass: the radix
// buckets carry packed (count << 16 | signs) so one scan gives both starts, and
// within a (small) bucket a row adds the members with smaller keys.  `hist` must
// be zeroed (1024 words) before the caller's last barrier (TileReduce::run does).  Requires the tile's
// total signs < 65536.  false: a bucket holds > 32 rows (use the sort fallback).
template <int NT>
FBX_DI bool radix_rank_off(u64 key, bool live, u32 m, u64 diff, u32* hist, u32* start, u64* bkeys,
                           u16* bm, BlockScanU32<NT>& scan, u32* rank, u32* off) {
  constexpr int BPT = 1024 / NT;  // buckets per thread
  const u32 hb = diff ? 63u - (u32)__clzll((long long)diff) : 0u;
  const u32 shift = hb >= 9u ? hb - 9u : 0u;
  const u32 digit = (u32)(key >> shift) & 1023u;
  u32 pos = 0;
  if (live) pos = atomicAdd(&hist[digit], (1u << 16) | m) >> 16;
  __syncthreads();
  u32 sz[BPT], tot = 0;
  bool big = false;
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    sz[b] = hist[threadIdx.x * BPT + b];
    tot += sz[b];
    big |= (sz[b] >> 16) > 32u;
  }
  if (__syncthreads_or(big)) return false;
  u32 run = scan.exclusive(tot);
#pragma unroll
  for (int b = 0; b < BPT; ++b) {
    start[threadIdx.x * BPT + b] = run;
    run += sz[b];
  }
  __syncthreads();
  u32 b0 = 0, bn = 0;
  if (live) {
    const u32 st = start[digit];
    b0 = st;
    bn = hist[digit] >> 16;
    bkeys[(st >> 16) + pos] = key;
    bm[(st >> 16) + pos] = (u16)m;
  }
  __syncthreads();
  if (live) {
    u32 r = b0 >> 16, o = b0 & 0xFFFFu;
    const u32 j0 = b0 >> 16;
    FBX_ROLLED
    for (u32 q = 0; q < bn; ++q) {
      const bool lt = bkeys[j0 + q] < key;
      r += lt ? 1u : 0u;
      o += lt ? (u32)bm[j0 + q] : 0u;
    }
    *rank = r;
    *off = o;
  }
  return true;
}

// block-wide OR and AND of a u64 (all threads receive both)
template <int NT>
FBX_DI void block_or_and(u64 vo, u64 va, u64* red, u64* o, u64* a) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    vo |= __shfl_xor_sync(0xFFFFFFFFu, vo, d);
    va &= __shfl_xor_sync(0xFFFFFFFFu, va, d);
  }
  if ((threadIdx.x & 31u) == 0) {
    red[threadIdx.x >> 5] = vo;
    red[(NT / 32) + (threadIdx.x >> 5)] = va;
  }
  __syncthreads();
  u64 ro = 0, ra = ~0ull;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) {
    ro |= red[w];
    ra &= red[(NT / 32) + w];
  }
  *o = ro;
  *a = ra;
  __syncthreads();
}

// Rank of `key` among the NT sorted keys in buf (number of keys < key).
template <int NT>
FBX_DI u32 lower_rank(const u64* sorted, u64 key) {
  u32 lo = 0;
#pragma unroll
  for (u32 step = (u32)NT >> 1; step > 0; step >>= 1)
    if (sorted[lo + step - 1] < key) lo += step;
  return lo;
}

// Table hashing (join indexes, dictionaries): a word-at-a-time splitmix
// mix -- any deterministic hash works, equality is always checked exactly.
FBX_DI u64 mix64(u64 x) {
  x ^= x >> 31;
  x *= 0x7FB5D329728EA185ull;
  x ^= x >> 27;
  x *= 0x81DADEF4BC2DD44Dull;
  x ^= x >> 33;
  return x;
}
// first min(n, 8) bytes of a span as a little-endian u64 (zero padded)
FBX_DI u64 load_prefix8(const u8* p, u32 n) {
  if (n == 0) return 0ull;
  const u64 a = (u64)p;
  const u32 sh = (u32)(a & 3u) * 8u;
  const u32* wp = (const u32*)(a & ~3ull);
  const u32 m = n < 8u ? n : 8u;
#ifdef FBX_EXACT_READS
  const u32 last = ((u32)(a & 3u) + m - 1u) >> 2;  // last word index touched
  u32 w0 = wp[0];
  u32 w1 = last >= 1u ? wp[1] : 0u;
  u32 w2 = last >= 2u ? wp[2] : 0u;
#else
  const u32 w0 = wp[0], w1 = wp[1], w2 = wp[2];  // spans keep >= 16 B of readable slack
#endif
  u32 lo = __funnelshift_r(w0, w1, sh), hi = __funnelshift_r(w1, w2, sh);
  u64 v = ((u64)hi << 32) | lo;
  return m == 8u ? v : (v & ((1ull << (m * 8u)) - 1ull));
}
// table hash of a byte key: one multiply-xorshift per 8-byte word, one full
// avalanche at the end (the same function builds and probes every table)
// (*pre: the first min(n, 8) bytes, zero padded -- the slots' prefix field)
FBX_DI u64 tbl_hash_bytes_pre(u64 h, const u8* p, u32 n, u64* pre) {
  h ^= (u64)n * 0x9E3779B97F4A7C15ull;
#ifdef FBX_EXACT_READS
  *pre = load_prefix8(p, n);
  FBX_ROLLED
  for (u32 k = 0; k < n; k += 8u) {
    h = (h ^ load_prefix8(p + k, n - k)) * 0xBF58476D1CE4E5B9ull;
    h ^= h >> 31;
  }
#else
  // the same 8-byte words, streamed: two aligned word loads per word
  u64 first = 0ull;
  if (n) {
    const u64 a = (u64)p;
    const u32 sh = (u32)(a & 3u) * 8u;
    const u32* wp = (const u32*)(a & ~3ull);
    u32 w0 = wp[0];
    FBX_ROLLED
    for (u32 k = 0; k < n; k += 8u, wp += 2) {
      const u32 w1 = wp[1], w2 = wp[2];  // spans keep >= 16 B of readable slack
      u64 v = ((u64)__funnelshift_r(w1, w2, sh) << 32) | __funnelshift_r(w0, w1, sh);
      if (n - k < 8u) v &= (1ull << ((n - k) * 8u)) - 1ull;
      if (k == 0u) first = v;
      h = (h ^ v) * 0xBF58476D1CE4E5B9ull;
      h ^= h >> 31;
      w0 = w2;
    }
  }
  *pre = first;
#endif
  return mix64(h);
}
FBX_DI u64 tbl_hash_bytes(u64 h, const u8* p, u32 n) {
  u64 pre;
  return tbl_hash_bytes_pre(h, p, n, &pre);
}
FBX_DI u64 tbl_hash_u64(u64 h, u64 v) { return mix64(h ^ mix64(v)); }

// ---------------------------------------------------------------------------
// TMA bulk copy global -> shared with an mbarrier (cp.async.bulk, sm_90+)
// ---------------------------------------------------------------------------
FBX_DI u32 smem_addr(const void* p) { return (u32)__cvta_generic_to_shared(p); }

FBX_DI void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
FBX_DI void mbar_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes) : "memory");
}
FBX_DI void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
// per-thread async copies (LDGSTS): probe slots prefetched into shared memory
FBX_DI void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
FBX_DI void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
FBX_DI void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Int64-keyed join tables: 16-B slots {u64 key, u32 ref, u32 aux}, aux = count
// (0 = empty), so a probe is one 16-B load and no key gather.
struct ISlot {
  u64 key;
  u32 ref;
  u32 aux;
};
FBX_DI ISlot islot_ld(const ISlot* s) {
  const uint4 v = __ldg((const uint4*)s);
  return ISlot{((u64)v.y << 32) | v.x, v.z, v.w};
}
FBX_DI u32 ld_acquire_u32(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// build-side insert (count duplicates): the whole slot {key, ref, count = 1} is
// claimed by ONE 128-bit compare-and-swap (atom.cas.b128, sm_90+), so no other
// thread can see a claimed slot without its key -- no fence, no publish step.
// An equal key already present bumps the count (its key is immutable by then).
// Returns true when the key was already present (a repeated key).
FBX_DI bool islot_insert(ISlot* T, u64 mask, u64 h, u64 key, u32 row) {
  u64 i = h & mask;
  const u64 hi = (1ull << 32) | (u64)row;  // {ref = row, aux = count 1}
  while (true) {
    u64 ok, oh;
    cas128(&T[i], 0ull, 0ull, key, hi, &ok, &oh);
    if (ok == 0ull && oh == 0ull) return false;  // claimed an empty slot
    if (ok == key) { atomicAdd(&T[i].aux, 1u); return true; }
    i = (i + 1) & mask;
  }
}

// L2 prefetch of a byte range (TMA bulk prefetch; the range is widened to 16 B)
FBX_DI void prefetch_span(const void* p, u64 bytes) {
  const u64 a = (u64)p & ~15ull, e = ((u64)p + bytes + 15ull) & ~15ull;
  for (u64 x = a; x < e; x += (1u << 20)) {
    const u32 len = (u32)((e - x) < (1ull << 20) ? (e - x) : (1ull << 20));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(x), "r"(len) : "memory");
  }
}

// TMA bulk store shared -> global (bulk async-group; 16-B aligned, 16-B multiple)
FBX_DI void bulk_s2g(void* gdst, const void* ssrc, u32 bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_addr(ssrc)), "r"(bytes)
               : "memory");
}
FBX_DI void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
FBX_DI void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
FBX_DI void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Copy n bytes staged at s (s == g mod 16) to global g: the 16-B aligned middle
// by one TMA bulk store (issued by thread 0), the ragged head / tail bytewise.
template <int NT>
FBX_DI void tile_out(u8* g, const u8* s, u32 n) {
  const u32 head = (u32)((16u - ((u64)g & 15u)) & 15u) < n ? (u32)((16u - ((u64)g & 15u)) & 15u) : n;
  const u32 mid = (n - head) & ~15u;
  for (u32 b = threadIdx.x; b < n - mid; b += NT) {
    const u32 o = b < head ? b : b + mid;
    g[o] = s[o];
  }
  if (threadIdx.x == 0 && mid) bulk_s2g(g + head, s + head, mid);
}

FBX_DI void mbar_wait(u64* bar, u32 phase) {
  u32 done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
  }
}

// ---------------------------------------------------------------------------
// Decoupled look-back over tiles (chunks) for the CSR offsets, within one
// launch (a launch covers at most 2^24 rows, so 28-bit counts never wrap; the
// run totals before a launch are carried in device memory, see codegen).
// status word: flag(2) | instances(28) | signs(34); flag 1 = aggregate,
// 2 = launch-inclusive prefix.
// ---------------------------------------------------------------------------
#ifndef FBX_LB_SLEEP
#define FBX_LB_SLEEP 64  // ns between polls of an unpublished predecessor
#endif
FBX_DI u64 ld_acquire(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
FBX_DI void st_release(u64* p, u64 v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
FBX_DI u64 pack_status(u64 flag, u64 inst, u64 signs) {
  return (flag << 62) | ((inst & 0xFFFFFFFull) << 34) | (signs & 0x3FFFFFFFFull);
}

// Thread 0, as soon as the tile's totals are known: the launch's first tile
// publishes its inclusive prefix, every other tile its aggregate (decoupled
// look-back).  Counts are launch-local: a launch never looks back past `first`.
FBX_DI void publish_aggregate(u64* status, u32 tile, u32 first, u64 inst, u64 signs) {
  st_release(status + tile, pack_status(tile == first ? 2 : 1, inst, signs));
}

// Warp 0, later: sum predecessors back to the first inclusive prefix, then
// publish this tile's inclusive prefix.  Returns the exclusive prefix.
FBX_DI void lookback(u64* status, u32 tile, u32 first, u64 inst, u64 signs, u64* ex_inst,
                     u64* ex_signs) {
  const u32 lane = threadIdx.x & 31u;
  if (tile == first) {
    *ex_inst = 0;
    *ex_signs = 0;
    return;
  }
  u64 acc_i = 0, acc_s = 0;
  i64 base = (i64)tile - 1;
  while (true) {
    i64 idx = base - (i64)lane;
    u64 w = 0;
    if (idx >= (i64)first) {
      w = ld_acquire(status + idx);
      while ((w >> 62) == 0) {  // predecessor not published yet: yield the issue slot
#if FBX_LB_SLEEP > 0
        __nanosleep(FBX_LB_SLEEP);
#endif
        w = ld_acquire(status + idx);
      }
    } else {
      w = pack_status(2, 0, 0);
    }
    u32 incl = __ballot_sync(0xFFFFFFFFu, (w >> 62) == 2);
    u32 stop = incl ? (__ffs(incl) - 1) : 31u;
    u64 vi = (lane <= stop) ? ((w >> 34) & 0xFFFFFFFull) : 0;
    u64 vs = (lane <= stop) ? (w & 0x3FFFFFFFFull) : 0;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      vi += __shfl_xor_sync(0xFFFFFFFFu, vi, d);
      vs += __shfl_xor_sync(0xFFFFFFFFu, vs, d);
    }
    acc_i += vi;
    acc_s += vs;
    if (incl) break;
    base -= 32;
  }
  if (lane == 0) st_release(status + tile, pack_status(2, acc_i + inst, acc_s + signs));
  *ex_inst = acc_i;
  *ex_signs = acc_s;
}

// ---------------------------------------------------------------------------
// HBM hash tables.  Slot layout (32 B, one sector per probe):
//   u64 tag (0 = empty), u32 ref (row / key offset), u32 aux (count / key len),
//   u64 value, u64 pad.  Capacity is a power of two; linear probing.
// ---------------------------------------------------------------------------
struct Slot {
  u64 tag;
  u32 ref;
  u32 aux;
  u64 value;
  u64 pad;
};

FBX_DI u64 table_tag(u64 h) { return h | 1ull; }  // never 0

// dictionary lookup (featureops.py:104-167): key bytes -> u64, default on miss.
// Slot.pad holds the key's first 8 bytes, so short keys compare in one word.
FBX_DI u64 dict_lookup(const Slot* slots, u64 mask, const u8* keyblob, Str key, u64 dflt) {
  u64 pre;
  const u64 tag = table_tag(tbl_hash_bytes_pre(0x5DB2CEB4C16A9E87ull, key.p, key.n, &pre));
  u64 i = tag & mask;
  FBX_ROLLED
  while (true) {
    const Slot* s = slots + i;
    u64 t = __ldg(&s->tag);
    if (t == 0) return dflt;
    if (t == tag && __ldg(&s->aux) == key.n && __ldg(&s->pad) == pre) {
      bool eq = true;
      u32 ref = __ldg(&s->ref);
      FBX_ROLLED
      for (u32 k = 8; k < key.n && eq; k += 8u)
        eq = load_prefix8(keyblob + ref + k, key.n - k) == load_prefix8(key.p + k, key.n - k);
      if (eq) return __ldg(&s->value);
    }
    i = (i + 1) & mask;
  }
}

// dict_lookup whose first slot (tag already computed) was copied into shared
// memory by cp.async in the prologue (raw driver-column keys)
FBX_DI u64 dict_lookup_pf(const Slot* slots, u64 mask, const u8* keyblob, Str key, u64 dflt,
                          u64 tag, const Slot* first) {
  const u64 pre = load_prefix8(key.p, key.n);
  u64 i = tag & mask;
  const Slot* s = first;
  FBX_ROLLED
  while (true) {
    const u64 t = s->tag;
    if (t == 0) return dflt;
    if (t == tag && s->aux == key.n && s->pad == pre) {
      bool eq = true;
      const u32 ref = s->ref;
      FBX_ROLLED
      for (u32 k = 8; k < key.n && eq; k += 8u)
        eq = load_prefix8(keyblob + ref + k, key.n - k) == load_prefix8(key.p + k, key.n - k);
      if (eq) return s->value;
    }
    i = (i + 1) & mask;
    s = slots + i;
  }
}

// ---------------------------------------------------------------------------
// JSON (CPython json.loads, strict=True) validation + dot-path extraction.
// Leaves are reported for up to NP paths of up to 8 segments each.
// ---------------------------------------------------------------------------
enum : u32 {
  J_MISSING = 0, J_STRING = 1, J_INT = 2, J_FLOAT = 3, J_TRUE = 4, J_FALSE = 5,
  J_NULL = 6, J_CONTAINER = 7, J_NAN = 8, J_POSINF = 9, J_NEGINF = 10
};
enum : u32 { JS_OK = 0, JS_MALFORMED = 1, JS_BIGINT = 2, JS_DEEP = 3 };

struct JLeaf {
  u32 beg, end;  // value text [beg, end) (strings: inside the quotes)
  u32 type;
  u32 esc;       // string contains a backslash escape
};

struct JPathSet {
  const u8* seg;       // concatenated segment bytes
  const u16* seg_off;  // [NP][8]
  const u8* seg_len;   // [NP][8]
  const u8* nseg;      // [NP]
};

FBX_DI bool j_ws(u32 c) { return c <= 0x20u && ((0x100002600ull >> c) & 1ull); }
FBX_DI bool j_digit(u32 c) { return c - '0' < 10u; }
FBX_DI bool j_hex(u32 c) { return (c - '0' < 10u) || ((c | 0x20u) - 'a' < 6u); }
FBX_DI u32 j_hexval(u32 c) { return c <= '9' ? c - '0' : (c | 0x20u) - 'a' + 10u; }

// Reader over a document (shared-memory stage or HBM).  Documents of at most
// 60 bytes with no backslash and no byte < 0x20 (the common case) take the
// mask mode: one branch-free SWAR pass builds 64-bit quote / space masks
// (jmask_build), after which whitespace skipping and string scanning are a
// find-first-set each.  Every other document runs the byte-wise scanner.
// Both modes accept exactly the same language: with no escapes and no
// control bytes, a string ends at the next quote and whitespace is ' ' only.
struct JReader {
  const u8* p;
  u32 n;
  bool fast;
  // fast mode, bit-reversed (bit 63 - j = byte j) so "first set bit at or
  // after i" is a left shift and a count-leading-zeros:
  u64 q;    // quote bytes | sentinel at byte 63 (no closing quote -> >= n)
  u64 nsp;  // non-space bytes | sentinel at byte n (all space -> n)
  FBX_DI u32 at(u32 k) const { return p[k]; }  // byte k, k < n
  FBX_DI u32 skip_ws(u32 i) const {  // i <= n
    if (fast) return i + (u32)__clzll((long long)(nsp << i));

    FBX_ROLLED
    while (i < n) {
      const u32 c = at(i);
      if (c > 0x20u || !j_ws(c)) break;
      ++i;
    }
    return i;
  }
};


// The mask mode's single pass: false -> the document needs the byte scanner.
FBX_DI bool jmask_build(const u8* p, u32 n, u64* qm, u64* nspm) {
  if (n == 0u || n > 60u) return false;
  const u64 a = (u64)p;
  const u32 sh = (u32)(a & 3u);
  const u32* wp = (const u32*)(a & ~3ull);
  const int nw = (int)((sh + n + 3u) >> 2);  // <= 16 aligned words
  u32 qlo = 0, qhi = 0, slo = 0, shi = 0, blo = 0, bhi = 0;
  FBX_ROLLED
  for (int w = nw - 1; w >= 0; --w) {  // last word first: word 0 lands in bits 0..3
    const u32 x = wp[w];
    const u32 x7 = x & 0x7F7F7F7Fu;
    const u32 zq = eq_bytes(x, x7, 0x22222222u);
    const u32 zs = eq_bytes(x, x7, 0x20202020u);
    // bad = byte < 0x20 or a backslash
    const u32 zb = (~((x7 + 0x60606060u) | x) | eq_bytes(x, x7, 0x5C5C5C5Cu)) & 0x80808080u;
    // gather the four 0x80 flags into bits 28..31 (products land on distinct bits)
    const u32 pq = zq * 0x00204081u, ps = zs * 0x00204081u, pb = zb * 0x00204081u;
    qhi = __funnelshift_l(qlo, qhi, 4); qlo = __funnelshift_l(pq, qlo, 4);
    shi = __funnelshift_l(slo, shi, 4); slo = __funnelshift_l(ps, slo, 4);
    bhi = __funnelshift_l(blo, bhi, 4); blo = __funnelshift_l(pb, blo, 4);
  }
  const u64 range = (1ull << n) - 1ull;
  const u64 bad = ((((u64)bhi << 32) | blo) >> sh) & range;
  if (bad) return false;
  const u64 qq = ((((u64)qhi << 32) | qlo) >> sh) & range;
  const u64 ns = ~((((u64)shi << 32) | slo) >> sh) & range;
  *qm = __brevll(qq | (1ull << 63));
  *nspm = __brevll(ns | (1ull << n));
  return true;
}

// JSON string body starting at i (after the quote): index of the closing quote
// or ~0 when malformed.  Mask mode: the next quote.  Byte mode: four bytes at
// a time until a quote, backslash or control byte shows up (SWAR), then
// byte-wise escape validation.
FBX_DI u32 j_string(const JReader& r, u32 i, u32* esc) {
  if (r.fast) {  // i <= n
    const u32 e = i + (u32)__clzll((long long)(r.q << i));
    return e < r.n ? e : ~0u;
  }
  const u64 base = (u64)r.p;
  FBX_ROLLED
  while (i < r.n) {
    const u64 a = base + i;
    const u32 sh = (u32)(a & 3u) * 8u;
    const u32 v = *(const u32*)(a & ~3ull) >> sh;
    u32 avail = 4u - (u32)(a & 3u), left = r.n - i;
    u32 m = avail < left ? avail : left;
    u32 q = v ^ 0x22222222u, b = v ^ 0x5C5C5C5Cu;
    u32 sp = (((q - 0x01010101u) & ~q) | ((b - 0x01010101u) & ~b) | ((v - 0x20202020u) & ~v)) &
             0x80808080u;
    if (m < 4u) sp &= (1u << (m * 8u)) - 1u;
    if (sp == 0u) { i += m; continue; }
    i += (u32)(__ffs(sp) - 1) >> 3;
    u32 c = r.at(i);
    if (c == '"') return i;
    if (c < 0x20u) return ~0u;
    // backslash escape
    *esc = 1;
    if (i + 1 >= r.n) return ~0u;
    u32 e = r.at(i + 1);
    if (e == 'u') {
      if (i + 5 >= r.n) return ~0u;
      if (!(j_hex(r.at(i + 2)) && j_hex(r.at(i + 3)) && j_hex(r.at(i + 4)) && j_hex(r.at(i + 5))))
        return ~0u;
      i += 6;
    } else if (e == '"' || e == '\\' || e == '/' || e == 'b' || e == 'f' || e == 'n' || e == 'r' ||
               e == 't') {
      i += 2;
    } else {
      return ~0u;
    }
  }
  return ~0u;
}

// decode the escaped JSON string body s[b, e) into dst (UTF-8, lone surrogates
// as WTF-8); returns the byte length, *lone set if a lone surrogate occurs.
FBX_DI u32 j_unescape(const u8* s, u32 b, u32 e, u8* dst, u32* lone) {
  u32 o = 0;
  u32 i = b;
  FBX_ROLLED
  while (i < e) {
    u32 c = s[i];
    if (c != '\\') { if (dst) dst[o] = (u8)c; ++o; ++i; continue; }
    u32 x = s[i + 1];
    if (x != 'u') {
      u32 v = x == 'b' ? 8u : x == 'f' ? 12u : x == 'n' ? 10u : x == 'r' ? 13u : x == 't' ? 9u : x;
      if (dst) dst[o] = (u8)v;
      ++o;
      i += 2;
      continue;
    }
    u32 cp = (j_hexval(s[i + 2]) << 12) | (j_hexval(s[i + 3]) << 8) | (j_hexval(s[i + 4]) << 4) |
             j_hexval(s[i + 5]);
    i += 6;
    if (cp >= 0xD800u && cp <= 0xDBFFu && i + 1 < e && s[i] == '\\' && s[i + 1] == 'u') {
      u32 lo2 = (j_hexval(s[i + 2]) << 12) | (j_hexval(s[i + 3]) << 8) |
                (j_hexval(s[i + 4]) << 4) | j_hexval(s[i + 5]);
      if (lo2 >= 0xDC00u && lo2 <= 0xDFFFu) {
        cp = 0x10000u + ((cp - 0xD800u) << 10) + (lo2 - 0xDC00u);
        i += 6;
      }
    }
    if (cp >= 0xD800u && cp <= 0xDFFFu) *lone = 1;
    if (cp < 0x80u) {
      if (dst) dst[o] = (u8)cp;
      o += 1;
    } else if (cp < 0x800u) {
      if (dst) { dst[o] = (u8)(0xC0u | (cp >> 6)); dst[o + 1] = (u8)(0x80u | (cp & 0x3Fu)); }
      o += 2;
    } else if (cp < 0x10000u) {
      if (dst) {
        dst[o] = (u8)(0xE0u | (cp >> 12));
        dst[o + 1] = (u8)(0x80u | ((cp >> 6) & 0x3Fu));
        dst[o + 2] = (u8)(0x80u | (cp & 0x3Fu));
      }
      o += 3;
    } else {
      if (dst) {
        dst[o] = (u8)(0xF0u | (cp >> 18));
        dst[o + 1] = (u8)(0x80u | ((cp >> 12) & 0x3Fu));
        dst[o + 2] = (u8)(0x80u | ((cp >> 6) & 0x3Fu));
        dst[o + 3] = (u8)(0x80u | (cp & 0x3Fu));
      }
      o += 4;
    }
  }
  return o;
}

// key comparison against a path segment, decoding escapes when present
FBX_DI bool j_key_eq(const JReader& r, const u8* s, u32 b, u32 e, u32 esc, const u8* seg, u32 slen) {
  if (!esc) {
    if (e - b != slen) return false;
    FBX_ROLLED
    for (u32 k = 0; k < slen; ++k)
      if (r.at(b + k) != seg[k]) return false;
    return true;
  }
  u8 tmp[64];
  u32 lone = 0;
  u32 dl = j_unescape(s, b, e, nullptr, &lone);
  if (dl != slen || dl > 64u) return false;
  j_unescape(s, b, e, tmp, &lone);
  if (lone) return false;
  FBX_ROLLED
  for (u32 k = 0; k < slen; ++k)
    if (tmp[k] != seg[k]) return false;
  return true;
}

// number at i; returns end index (or ~0 malformed); *type J_INT / J_FLOAT,
// *digits = number of integer digits (for the 4300-digit int limit).
FBX_DI u32 j_number(const JReader& r, u32 i, u32* type, u32* digits) {
  const u32 n = r.n;
  u32 st = i;
  bool neg = r.at(i) == '-';
  if (neg) ++i;
  if (i >= n || !j_digit(r.at(i))) return ~0u;
  if (r.at(i) == '0') {
    ++i;
  } else {
    FBX_ROLLED
    while (i < n && j_digit(r.at(i))) ++i;
  }
  *digits = i - st - (neg ? 1u : 0u);
  *type = J_INT;
  if (i + 1 < n && r.at(i) == '.' && j_digit(r.at(i + 1))) {
    i += 2;
    FBX_ROLLED
    while (i < n && j_digit(r.at(i))) ++i;
    *type = J_FLOAT;
  }
  if (i < n && (r.at(i) | 0x20u) == 'e') {
    u32 k = i + 1;
    if (k < n && (r.at(k) == '+' || r.at(k) == '-')) ++k;
    if (k < n && j_digit(r.at(k))) {
      FBX_ROLLED
      while (k < n && j_digit(r.at(k))) ++k;
      i = k;
      *type = J_FLOAT;
    }
  }
  return i;
}

FBX_DI bool j_lit(const JReader& r, u32 i, const char* w, u32 wl) {
  if (i + wl > r.n) return false;
  FBX_ROLLED
  for (u32 k = 0; k < wl; ++k)
    if (r.at(i + k) != (u8)w[k]) return false;
  return true;
}

// Mask-mode walker (documents jmask_build accepted: <= 60 bytes, no backslash,
// no byte < 0x20).  The same grammar and path semantics as the byte scanner in
// json_extract below, walked one MEMBER per iteration (key, ':', value, then the
// closers and the comma that follow it) instead of one token per iteration: the
// documents of a warp mostly share their shape, so lanes stay on the same
// instruction stream (a token loop diverges on the token kind every step).
// Whitespace is a clz over the non-space mask, a string's end a clz over the
// quote mask (no escapes); the masks' sentinels bound every scan.
template <int NP, class KM>
FBX_DI u32 json_extract_m(const u8* p, const u32 n, const u64 q, const u64 nsp,
                          const JPathSet ps, JLeaf (&leaf)[NP]) {
#define FBX_JSKIP(x) ((x) + (u32)__clzll((long long)(nsp << (x))))
  u64 kind = 0;   // bit d: the container at depth d+1 is an object
  u32 depth = 0;
  u64 live = 0;   // byte d (d < 8): paths live in the object at depth d+1
  u32 i = (u32)__clzll((long long)nsp);
  while (true) {
    // ---- one member (object) or element (array) at i, or the top-level value
    u32 leafm = 0u, descm = 0u;
    const bool obj = depth && ((kind >> (depth - 1u)) & 1ull);
    if (obj) {
      if (i >= n || p[i] != '"') return JS_MALFORMED;
      const u32 kb = i + 1u;
      const u32 ke = kb + (u32)__clzll((long long)(q << kb));
      if (ke >= n) return JS_MALFORMED;
      if (depth <= 8u) {
        const u32 lv = (u32)((live >> ((depth - 1u) * 8u)) & 0xFFull);
        if (lv) {
          const u32 sidx = depth - 1u, klen = ke - kb;
          const u64 kpre = load_prefix8(p + kb, klen);
#pragma unroll
          for (int pp = 0; pp < NP; ++pp) {
            if (!(lv & (1u << pp))) continue;
            const u32 ns = KM::nseg(pp);
            if (sidx >= ns) continue;
            bool eq = KM::eq(pp, sidx, kpre, klen);
            if (eq && klen > 8u) {
              const u32 off = ps.seg_off[pp * 8 + sidx];
              FBX_ROLLED
              for (u32 k = 8; k < klen && eq; ++k) eq = p[kb + k] == ps.seg[off + k];
            }
            if (!eq) continue;
            leaf[pp] = JLeaf{0, 0, J_MISSING, 0};  // a later duplicate key replaces the value
            if (sidx + 1u == ns) leafm |= (1u << pp); else descm |= (1u << pp);
          }
        }
      }
      i = FBX_JSKIP(ke + 1u);
      if (i >= n || p[i] != ':') return JS_MALFORMED;
      i = FBX_JSKIP(i + 1u);
    }
    // ---- the value at i
    if (i >= n) return JS_MALFORMED;
    const u32 c = p[i];
    if (c == '{' || c == '[') {
      const bool o = c == '{';
      if (o) kind |= (1ull << depth); else kind &= ~(1ull << depth);
#pragma unroll
      for (int pp = 0; pp < NP; ++pp)
        if (leafm & (1u << pp)) leaf[pp] = JLeaf{i, i, J_CONTAINER, 0};
      const u32 childlive = o ? (depth == 0u ? ((1u << NP) - 1u) : descm) : 0u;
      ++depth;
      if (depth <= 8u) {
        live &= ~(0xFFull << ((depth - 1u) * 8u));
        live |= (u64)(childlive & 0xFFu) << ((depth - 1u) * 8u);
      }
      i = FBX_JSKIP(i + 1u);
      if (i >= n) return JS_MALFORMED;
      if (p[i] != (o ? '}' : ']')) continue;  // first member / element
      --depth;  // empty container: a complete value
      i = FBX_JSKIP(i + 1u);
    } else {
      u32 vb = i, ve, vt;
      if (c == '"') {
        vb = i + 1u;
        ve = vb + (u32)__clzll((long long)(q << vb));
        if (ve >= n) return JS_MALFORMED;
        vt = J_STRING;
        i = ve + 1u;
      } else {
        // a number or literal (4300-digit limit unreachable in 60 bytes)
        u32 e;
        const u32 neg = c == '-' ? 1u : 0u;
        const u32 d = i + neg < n ? p[i + neg] : 0u;
        if (d - '0' < 10u) {
          e = i + neg + 1u;
          if (d != '0') {
            FBX_ROLLED
            while (e < n && p[e] - '0' < 10u) ++e;
          }
          vt = J_INT;
          if (e + 1u < n && p[e] == '.' && p[e + 1u] - '0' < 10u) {
            e += 2u;
            FBX_ROLLED
            while (e < n && p[e] - '0' < 10u) ++e;
            vt = J_FLOAT;
          }
          if (e < n && (p[e] | 0x20u) == 'e') {
            u32 k = e + 1u;
            if (k < n && (p[k] == '+' || p[k] == '-')) ++k;
            if (k < n && p[k] - '0' < 10u) {
              FBX_ROLLED
              while (k < n && p[k] - '0' < 10u) ++k;
              e = k;
              vt = J_FLOAT;
            }
          }
        } else {
          const u64 w = load_prefix8(p + i, n - i);
          if ((w & 0xFFFFFFFFull) == 0x65757274ull) { vt = J_TRUE; e = i + 4u; }               // true
          else if ((w & 0xFFFFFFFFFFull) == 0x65736C6166ull) { vt = J_FALSE; e = i + 5u; }     // false
          else if ((w & 0xFFFFFFFFull) == 0x6C6C756Eull) { vt = J_NULL; e = i + 4u; }          // null
          else if ((w & 0xFFFFFFull) == 0x4E614Eull) { vt = J_NAN; e = i + 3u; }               // NaN
          else if (w == 0x7974696E69666E49ull) { vt = J_POSINF; e = i + 8u; }                  // Infinity
          else if (neg && w == 0x74696E69666E492Dull && i + 8u < n && p[i + 8u] == 'y') {   // -Infinity
            vt = J_NEGINF; e = i + 9u;
          } else {
            return JS_MALFORMED;
          }
        }
        ve = e;
        i = e;
      }
#pragma unroll
      for (int pp = 0; pp < NP; ++pp)
        if (leafm & (1u << pp)) leaf[pp] = JLeaf{vb, ve, vt, 0};
      i = FBX_JSKIP(i);
    }
    // ---- after a complete value: closers, then one comma (or the end)
    while (true) {
      if (depth == 0u) return i >= n ? JS_OK : JS_MALFORMED;
      if (i >= n) return JS_MALFORMED;
      const u32 ch = p[i];
      const bool ob = (kind >> (depth - 1u)) & 1ull;
      if (ch == ',') break;
      if (ch != (ob ? '}' : ']')) return JS_MALFORMED;
      --depth;
      i = FBX_JSKIP(i + 1u);
    }
    i = FBX_JSKIP(i + 1u);
  }
#undef FBX_JSKIP
}

// Validate the whole document (CPython json.loads, strict) and extract the NP
// dot paths.  Inlined so the leaves live in registers.  Returns JS_*.
// KM: plan-generated key matcher -- KM::nseg(p) and KM::eq(p, sidx, prefix8, len)
// with the path segments as immediates (escaped keys use the generic compare).
template <int NP, class KM>
FBX_DI u32 json_extract(Str doc, const JPathSet ps, JLeaf (&leaf)[NP]) {
#pragma unroll
  for (int p = 0; p < NP; ++p) leaf[p] = JLeaf{0, 0, J_MISSING, 0};
  {
    u64 q = 0ull, nsp = 0ull;
    if (jmask_build(doc.p, doc.n, &q, &nsp)) return json_extract_m<NP, KM>(doc.p, doc.n, q, nsp, ps, leaf);
  }
  // every other document: the byte scanner (escapes, control bytes, long documents)
  JReader r;
  r.p = doc.p;
  r.n = doc.n;
  r.q = 0ull;
  r.nsp = 0ull;
  r.fast = false;
  const u32 n = doc.n;
  u64 kind_stack = 0;  // bit d: container at depth d+1 is an object
  u32 depth = 0;
  u64 live = 0;        // byte d (d < 8): paths live for the object at depth d+1
  u32 i = r.skip_ws(0);
  u32 leafm = 0, descm = (1u << NP) - 1u;
  bool top = true;
  while (true) {
    if (i >= n) return JS_MALFORMED;
    u32 c = r.at(i);
    u32 vb = i, ve, vt, vesc = 0;
    if (c == '{' || c == '[') {
      if (depth >= 64u) return JS_DEEP;
      bool obj = (c == '{');
      if (obj) kind_stack |= (1ull << depth); else kind_stack &= ~(1ull << depth);
      ++depth;
#pragma unroll
      for (int p = 0; p < NP; ++p)
        if (leafm & (1u << p)) leaf[p] = JLeaf{vb, vb, J_CONTAINER, 0};
      u32 childlive = (obj && depth <= 8u) ? (top ? ((1u << NP) - 1u) : descm) : 0u;
      if (depth <= 8u) {
        live &= ~(0xFFull << ((depth - 1) * 8));
        live |= (u64)(childlive & 0xFFu) << ((depth - 1) * 8);
      }
      i = r.skip_ws(i + 1);
      top = false;
      if (i < n && r.at(i) == (obj ? '}' : ']')) {
        ++i;
        --depth;
        goto after_value;
      }
      if (obj) goto member_key;
      leafm = 0;
      descm = 0;
      continue;  // first array element
    }
    top = false;
    if (c == '"') {
      u32 e = j_string(r, i + 1, &vesc);
      if (e == ~0u) return JS_MALFORMED;
      vb = i + 1;
      ve = e;
      vt = J_STRING;
      i = e + 1;
    } else if (c == '-' || j_digit(c)) {
      if (c == '-' && j_lit(r, i, "-Infinity", 9)) {
        vt = J_NEGINF;
        i += 9;
        ve = i;
      } else {
        u32 digits = 0;
        u32 e = j_number(r, i, &vt, &digits);
        if (e == ~0u) return JS_MALFORMED;
        if (vt == J_INT && digits > 4300u) return JS_BIGINT;
        ve = e;
        i = e;
      }
    } else if (c == 't' && j_lit(r, i, "true", 4)) {
      vt = J_TRUE; i += 4; ve = i;
    } else if (c == 'f' && j_lit(r, i, "false", 5)) {
      vt = J_FALSE; i += 5; ve = i;
    } else if (c == 'n' && j_lit(r, i, "null", 4)) {
      vt = J_NULL; i += 4; ve = i;
    } else if (c == 'N' && j_lit(r, i, "NaN", 3)) {
      vt = J_NAN; i += 3; ve = i;
    } else if (c == 'I' && j_lit(r, i, "Infinity", 8)) {
      vt = J_POSINF; i += 8; ve = i;
    } else {
      return JS_MALFORMED;
    }
#pragma unroll
    for (int p = 0; p < NP; ++p)
      if (leafm & (1u << p)) leaf[p] = JLeaf{vb, ve, vt, vesc};
  after_value:
    while (true) {
      i = r.skip_ws(i);
      if (depth == 0) return i == n ? JS_OK : JS_MALFORMED;
      if (i >= n) return JS_MALFORMED;
      bool obj = (kind_stack >> (depth - 1)) & 1ull;
      u32 ch = r.at(i);
      if (ch == ',') {
        i = r.skip_ws(i + 1);
        if (obj) goto member_key;
        leafm = 0;
        descm = 0;
        goto next_value;
      }
      if (ch == (obj ? '}' : ']')) {
        ++i;
        --depth;
        continue;
      }
      return JS_MALFORMED;
    }
  member_key : {
    if (i >= n || r.at(i) != '"') return JS_MALFORMED;
    u32 kesc = 0;
    u32 ke = j_string(r, i + 1, &kesc);
    if (ke == ~0u) return JS_MALFORMED;
    u32 kb = i + 1;
    i = r.skip_ws(ke + 1);
    if (i >= n || r.at(i) != ':') return JS_MALFORMED;
    i = r.skip_ws(i + 1);
    leafm = 0;
    descm = 0;
    if (depth <= 8u) {
      u32 lv = (u32)((live >> ((depth - 1) * 8)) & 0xFFull);
      u32 sidx = depth - 1;
      if (lv) {
        const u32 klen = ke - kb;
        const u64 kpre = kesc ? 0ull : load_prefix8(doc.p + kb, klen);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          if (!(lv & (1u << p))) continue;
          const u32 ns = KM::nseg(p);
          if (sidx >= ns) continue;
          bool eq;
          if (!kesc) {
            eq = KM::eq(p, sidx, kpre, klen);
            if (eq && klen > 8u) {
              u32 off = ps.seg_off[p * 8 + sidx];
              FBX_ROLLED
              for (u32 k = 8; k < klen && eq; ++k) eq = r.at(kb + k) == ps.seg[off + k];
            }
          } else {
            u32 off = ps.seg_off[p * 8 + sidx], sl = ps.seg_len[p * 8 + sidx];
            eq = j_key_eq(r, doc.p, kb, ke, kesc, ps.seg + off, sl);
          }
          if (!eq) continue;
          leaf[p] = JLeaf{0, 0, J_MISSING, 0};  // a later duplicate key replaces the value
          if (sidx + 1 == ns) leafm |= (1u << p); else descm |= (1u << p);
        }
      }
    }
    continue;
  }
  next_value:
    continue;
  }
}

}  // namespace fbx
#include "fbx_pow10.cuh"
namespace fbx {

// 192-bit product (p2:p1:p0) times 2^-s rounded to nearest-even binary64.
// Returns the bits, or ~0ull on overflow (inf).  P > 0.
FBX_DI u64 round_p192(u64 p2, u64 p1, u64 p0, int s) {
  int msb = p2 ? 191 - __clzll((long long)p2) : (p1 ? 127 - __clzll((long long)p1) : 63 - __clzll((long long)p0));
  const int exp = msb - s;
  if (exp > 1023) return ~0ull;
  int shift = exp >= -1022 ? msb - 52 : s - 1074;  // right shift to the 53-bit (or subnormal) quantum
  if (shift > 191) return 0ull;                      // far below half the smallest subnormal
  // m = P >> shift (fits 64 bits), guard bit and sticky
  u64 m, guard, sticky;
  {
    const int w = shift >> 6, b = shift & 63;
    const u64 words[4] = {p0, p1, p2, 0ull};
    m = b ? (words[w] >> b) | (words[w + 1] << (64 - b)) : words[w];
    if (w + 1 < 3 && b == 0) m = words[w];
    const int gs = shift - 1;
    if (gs < 0) {
      guard = 0; sticky = 0;
    } else {
      const int gw = gs >> 6, gb = gs & 63;
      guard = (words[gw] >> gb) & 1ull;
      u64 st = words[gw] & ((1ull << gb) - 1ull);
      for (int k = 0; k < gw; ++k) st |= words[k];
      sticky = st != 0ull;
    }
  }
  if (guard && (sticky || (m & 1ull))) ++m;
  int qexp = shift - s;  // value = m * 2^qexp
  if (m == 0) return 0ull;
  if (m >> 53) { m >>= 1; ++qexp; }
  if (m >> 52) {
    const int be = qexp + 1075;
    if (be >= 2047) return ~0ull;
    return ((u64)be << 52) | (m & ((1ull << 52) - 1ull));
  }
  return m;  // subnormal
}

// Exact decision between two adjacent doubles for an exact decimal w * 10^q (the
// bracketing Eisel-Lemire could not: the value is within 2^-64 of their midpoint,
// e.g. an exact tie like 7283009533423449.5).  Big integers of 48 x 32-bit limbs:
// w * 5^|q| * 2^x against (2m + 1) * 2^y.  Rare path: not inlined.
__device__ __noinline__ void big_mul_small(u32* l, int& nl, u32 mul) {
  u64 carry = 0;
  for (int i = 0; i < nl; ++i) {
    const u64 cur = (u64)l[i] * mul + carry;
    l[i] = (u32)cur;
    carry = cur >> 32;
  }
  if (carry && nl < 48) l[nl++] = (u32)carry;
}
// place v << sh into a zeroed 48-limb array
__device__ __noinline__ void big_set_shifted(u32* out, const u32* v, int nv, int sh) {
  for (int i = 0; i < 48; ++i) out[i] = 0u;
  const int ws = sh >> 5, bs = sh & 31;
  for (int i = 0; i < nv; ++i) {
    const u64 x = (u64)v[i] << bs;
    if (i + ws < 48) out[i + ws] |= (u32)x;
    if (i + ws + 1 < 48) out[i + ws + 1] |= (u32)(x >> 32);
  }
}
__device__ __noinline__ u64 dec_to_double_tie(u64 w, int q, u64 a_bits) {
  const u32 ea_b = (u32)(a_bits >> 52) & 0x7FFu;
  const u64 ma = ea_b ? ((a_bits & ((1ull << 52) - 1ull)) | (1ull << 52)) : (a_bits & ((1ull << 52) - 1ull));
  const int ea = ea_b ? (int)ea_b - 1075 : -1074;
  const u64 y = 2ull * ma + 1ull;  // midpoint = y * 2^(ea - 1)
  u32 X[48], Y[48], A[48], B[48];
  int nx = 2, ny = 2;
  X[0] = (u32)w; X[1] = (u32)(w >> 32);
  Y[0] = (u32)y; Y[1] = (u32)(y >> 32);
  int xs, ys;  // compare X * 2^xs with Y * 2^ys
  if (q >= 0) {
    for (int k = q; k > 0;) { const int d = k < 13 ? k : 13; u32 m = 1; for (int i = 0; i < d; ++i) m *= 5u; big_mul_small(X, nx, m); k -= d; }
    xs = q; ys = ea - 1;
  } else {
    for (int k = -q; k > 0;) { const int d = k < 13 ? k : 13; u32 m = 1; for (int i = 0; i < d; ++i) m *= 5u; big_mul_small(Y, ny, m); k -= d; }
    xs = 0; ys = ea - 1 - q;
  }
  const int mn = xs < ys ? xs : ys;
  big_set_shifted(A, X, nx, xs - mn);
  big_set_shifted(B, Y, ny, ys - mn);
  int c = 0;
  for (int i = 47; i >= 0 && c == 0; --i) c = A[i] < B[i] ? -1 : (A[i] > B[i] ? 1 : 0);
  if (c < 0) return a_bits;
  if (c > 0) return a_bits + 1ull;
  return (ma & 1ull) ? a_bits + 1ull : a_bits;  // exact tie: even mantissa
}

// Correctly rounded w * 10^q (exact=false: the value lies in [w, w+1) * 10^q,
// i.e. nonzero digits were dropped past the 19th).  Bracketing Eisel-Lemire with
// an exact big-integer decision when the bracket straddles a midpoint; the exact
// model is decimal_tables.to_double.  Returns 0 ok, 1 needs all the digits (an
// inexact decimal that close to a midpoint), 2 overflow (*bits = +inf).
FBX_DI u32 dec_to_double(u64 w, int q, bool exact, u64* bits) {
  if (w == 0 || q < P10_QMIN) { *bits = 0ull; return 0; }
  if (q > P10_QMAX) { *bits = 0x7FF0000000000000ull; return 2; }
  const int k = q - P10_QMIN;
  const u64 th = __ldg(P10_HI + k), tl = __ldg(P10_LO + k);
  const int s = __ldg(P10_S + k);
  const bool tex = __ldg(P10_EXACT + k) != 0;
  // lo = w * T
  u64 a0 = w * tl, a1 = __umul64hi(w, tl);
  u64 b0 = w * th, b1 = __umul64hi(w, th);
  u64 p0 = a0, p1 = a1 + b0, p2 = b1 + (p1 < a1 ? 1ull : 0ull);
  const u64 lo_bits = round_p192(p2, p1, p0, s);
  if (!(exact && tex)) {
    // hi = (w + !exact) * (T + !tex) - 1
    const u64 w2 = w + (exact ? 0ull : 1ull);
    const u64 t2l = tl + (tex ? 0ull : 1ull), t2h = th + (t2l < tl ? 1ull : 0ull);
    u64 c0 = w2 * t2l, c1 = __umul64hi(w2, t2l);
    u64 d0 = w2 * t2h, d1 = __umul64hi(w2, t2h);
    u64 q0 = c0, q1 = c1 + d0, q2 = d1 + (q1 < c1 ? 1ull : 0ull);
    // minus one
    const u64 borrow0 = q0 == 0ull;
    q0 -= 1ull;
    if (borrow0) { const u64 borrow1 = q1 == 0ull; q1 -= 1ull; if (borrow1) q2 -= 1ull; }
    const u64 hi_bits = round_p192(q2, q1, q0, s);
    if (hi_bits != lo_bits) {
      if (!exact || lo_bits == ~0ull) return 1;  // digits beyond the 19th: needs them all
      const u64 r = dec_to_double_tie(w, q, lo_bits);
      if ((r & 0x7FFFFFFFFFFFFFFFull) >= 0x7FF0000000000000ull) { *bits = 0x7FF0000000000000ull; return 2; }
      *bits = r;
      return 0;
    }
  }
  if (lo_bits == ~0ull) { *bits = 0x7FF0000000000000ull; return 2; }
  *bits = lo_bits;
  return 0;
}

// JSON leaf -> Float32 bits (viewpipe.py:278-279: canon_f32(float(value))).
// 0 = ok, 1 = not a number (-> null), 2 = OverflowError (float(int) or
// struct.pack 'f'), 3 = needs a bignum decimal conversion (not on device).
FBX_DI u32 j_to_f32(const u8* s, JLeaf lf, u32* bits) {
  if (lf.type == J_NAN) { *bits = 0x7FC00000u; return 0; }
  if (lf.type == J_POSINF) { *bits = 0x7F800000u; return 0; }
  if (lf.type == J_NEGINF) { *bits = 0xFF800000u; return 0; }
  if (lf.type != J_INT && lf.type != J_FLOAT) return 1;
  u32 i = lf.beg;
  const bool neg = s[i] == '-';
  if (neg) ++i;
  u64 w = 0;
  u32 sig = 0;
  int e10 = 0;
  bool exact = true, frac = false;
  for (; i < lf.end; ++i) {
    const u32 c = s[i];
    if (c == '.') { frac = true; continue; }
    if (c == 'e' || c == 'E') break;
    const u32 d = c - '0';
    if (frac) --e10;
    if (sig == 0 && d == 0) continue;
    if (sig < 19) { w = w * 10u + d; ++sig; }
    else { ++e10; if (d) exact = false; }
  }
  if (i < lf.end) {  // exponent
    ++i;
    bool eneg = false;
    if (s[i] == '+' || s[i] == '-') { eneg = s[i] == '-'; ++i; }
    int ev = 0;
    for (; i < lf.end; ++i)
      if (ev < 100000) ev = ev * 10 + (int)(s[i] - '0');
    e10 += eneg ? -ev : ev;
  }
  u64 db;
  const u32 st = dec_to_double(w, e10, exact, &db);
  if (st == 1) return 3;
  if (st == 2 && lf.type == J_INT) return 2;  // float(int): "int too large to convert to float"
  if (lf.type == J_INT && w == 0) db = 0ull;  // int -0 is 0
  else if (neg) db |= 0x8000000000000000ull;
  const double d = __longlong_as_double((long long)db);
  const float f = __double2float_rn(d);
  *bits = __float_as_uint(f);
  if (isinf(f) && !isinf(d)) return 2;
  return 0;
}

// JSON int literal -> int64 with range check (viewpipe.py:271-274)
FBX_DI bool j_to_i64(const u8* s, u32 b, u32 e, i64* out) {
  bool neg = s[b] == '-';
  u32 i = b + (neg ? 1u : 0u);
  u64 v = 0;
  const u64 lim = neg ? (1ull << 63) : ((1ull << 63) - 1ull);
  for (; i < e; ++i) {
    u32 d = s[i] - '0';
    if (v > (lim - d) / 10ull) return false;
    v = v * 10ull + d;
  }
  *out = neg ? (i64)(0ull - v) : (i64)v;
  return true;
}

// ---------------------------------------------------------------------------
// str() of a Float32 value (featureops.py:298-299 lower/trim, :318 token, :336
// lookup, concat): CPython's repr -- the shortest digits that round-trip the
// value widened to binary64, laid out by format_float_short.  Exact integer
// algorithm; decimal_tables.f32_repr is its Python model (checked against
// repr() on CPU, tests/test_host.py).
// ---------------------------------------------------------------------------
// floor(x * 2^t / 10^k) (< 10^19 by the choice of k) and whether it is inexact
FBX_DI u64 repr_window(u64 x, int t, int k, bool* sticky) {
  if (k >= 0) {
    if (t < 0) {
      const u64 ip = -t >= 64 ? 0ull : x >> -t;
      const bool fr = -t >= 64 ? x != 0ull : (x & ((1ull << -t) - 1ull)) != 0ull;
      u64 p = 1;
      for (int i = 0; i < k; ++i) p *= 10u;
      *sticky = fr || (ip % p) != 0ull;
      return ip / p;
    }
    u32 l[4];  // x << t < 2^128 (x < 2^55, t <= 73)
    const u64 lo = t >= 64 ? 0ull : x << t;
    const u64 hi = t == 0 ? 0ull : (t >= 64 ? x << (t - 64) : x >> (64 - t));
    l[0] = (u32)lo; l[1] = (u32)(lo >> 32); l[2] = (u32)hi; l[3] = (u32)(hi >> 32);
    bool st = false;
    for (int kk = k; kk > 0;) {
      const int d = kk < 9 ? kk : 9;
      u32 div = 1;
      for (int i = 0; i < d; ++i) div *= 10u;
      u64 rem = 0;
#pragma unroll
      for (int i = 3; i >= 0; --i) {
        const u64 cur = (rem << 32) | l[i];
        l[i] = (u32)(cur / div);
        rem = cur % div;
      }
      st |= rem != 0ull;
      kk -= d;
    }
    *sticky = st;
    return ((u64)l[1] << 32) | l[0];
  }
  // x * 10^-k * 2^t = (x * 5^-k) * 2^(t - k); x * 5^62 < 2^199
  u32 l[8] = {(u32)x, (u32)(x >> 32), 0u, 0u, 0u, 0u, 0u, 0u};
  for (int kk = -k; kk > 0;) {
    const int d = kk < 13 ? kk : 13;
    u32 mul = 1;
    for (int i = 0; i < d; ++i) mul *= 5u;
    u64 carry = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const u64 cur = (u64)l[i] * mul + carry;
      l[i] = (u32)cur;
      carry = cur >> 32;
    }
    kk -= d;
  }
  const int sh = t - k;
  if (sh >= 0) {
    *sticky = false;
    return (((u64)l[1] << 32) | l[0]) << sh;
  }
  const int r = -sh, ws = r >> 5, bs = r & 31;
  bool st = (l[ws] & ((1u << bs) - 1u)) != 0u;
  for (int i = 0; i < ws; ++i) st |= l[i] != 0u;
  *sticky = st;
  const u32 a = l[ws], b = ws + 1 < 8 ? l[ws + 1] : 0u, c = ws + 2 < 8 ? l[ws + 2] : 0u;
  return ((u64)__funnelshift_r(b, c, bs) << 32) | __funnelshift_r(a, b, bs);
}

// writes repr(float) of the float32 bits; returns the length (<= 24).  Not
// inlined: one body per kernel however many operators stringify a Float32.
__device__ __noinline__ u32 f32_repr(u8* dst, u32 bits) {
  const u32 sgn = bits >> 31, ex = (bits >> 23) & 0xFFu, m = bits & 0x7FFFFFu;
  u32 n = 0;
  if (ex == 255u && m) { dst[0] = 'n'; dst[1] = 'a'; dst[2] = 'n'; return 3u; }
  if (sgn) dst[n++] = '-';
  if (ex == 255u) { dst[n] = 'i'; dst[n + 1] = 'n'; dst[n + 2] = 'f'; return n + 3u; }
  if (ex == 0u && m == 0u) { dst[n] = '0'; dst[n + 1] = '.'; dst[n + 2] = '0'; return n + 3u; }
  // widened: f * 2^e, f in [2^52, 2^53) and even -> closed rounding interval
  const u32 mant = ex ? (m | 0x800000u) : m;
  const int bl = 32 - __clz(mant);
  const u64 f = (u64)mant << (53 - bl);
  const int t = (ex ? (int)ex - 150 : -149) - (53 - bl) - 2;  // units of 2^t
  const u64 v4 = 4ull * f, lo4 = v4 - (f == (1ull << 52) ? 1ull : 2ull), hi4 = v4 + 2ull;
  const int k = (((54 + t) * 78913) >> 18) - 17;  // floor(log10 hi) - 17
  bool sl, sv, shh;
  const u64 wl = repr_window(lo4, t, k, &sl), wv = repr_window(v4, t, k, &sv);
  const u64 wh = repr_window(hi4, t, k, &shh);
  // largest p with a multiple of 10^(k+p) in [lo, hi]: monotone, p = 1 always holds
  int p = 1;
  u64 p10 = 10u, bot = wl / 10u + ((wl % 10u) != 0u || sl), top = wh / 10u;
  while (p < 18) {
    const u64 q10 = p10 * 10u;
    const u64 nb = wl / q10 + ((wl % q10) != 0u || sl), nt = wh / q10;
    if (nb > nt) break;
    p10 = q10; ++p; bot = nb; top = nt;
  }
  u64 w = wv / p10;
  const u64 r = wv % p10, half = p10 >> 1;
  if (r > half || (r == half && (sv || (w & 1u)))) ++w;
  w = w < bot ? bot : (w > top ? top : w);
  u8 dg[20];
  const u32 nd = u64_dec_len(w);
  u64_dec(dg, w, nd);
  const int decpt = (int)nd + k + p;
  if (decpt <= -4 || decpt > 16) {
    dst[n++] = dg[0];
    if (nd > 1u) {
      dst[n++] = '.';
      for (u32 i = 1; i < nd; ++i) dst[n++] = dg[i];
    }
    int x = decpt - 1;
    dst[n++] = 'e';
    dst[n++] = x < 0 ? '-' : '+';
    x = x < 0 ? -x : x;
    if (x >= 100) dst[n++] = (u8)('0' + x / 100);
    dst[n++] = (u8)('0' + (x / 10) % 10);
    dst[n++] = (u8)('0' + x % 10);
  } else if (decpt <= 0) {
    dst[n++] = '0';
    dst[n++] = '.';
    for (int i = 0; i < -decpt; ++i) dst[n++] = '0';
    for (u32 i = 0; i < nd; ++i) dst[n++] = dg[i];
  } else if ((u32)decpt < nd) {
    for (u32 i = 0; i < nd; ++i) {
      if (i == (u32)decpt) dst[n++] = '.';
      dst[n++] = dg[i];
    }
  } else {
    for (u32 i = 0; i < nd; ++i) dst[n++] = dg[i];
    for (u32 i = nd; i < (u32)decpt; ++i) dst[n++] = '0';
    dst[n++] = '.';
    dst[n++] = '0';
  }
  return n;
}

}  // namespace fbx

namespace fbx {

// ---------------------------------------------------------------------------
// repr() of a binary64 value (json.dumps of Float leaves, Json-kind extraction,
// viewpipe.py:268): the f32_repr scheme with big-integer windows -- x << t up to
// 2^1030 and x * 5^341 < 2^850 fit 36 x 32-bit limbs -- subnormals at their fixed
// spacing and the rounding interval closed only for an even mantissa.  Python
// model: decimal_tables.f64_repr (checked against repr(), tests/test_host.py).
// Rare path: not inlined, limbs in local memory.
// ---------------------------------------------------------------------------
__device__ __noinline__ u64 repr_window_big(u64 x, int t, int k, bool* sticky) {
  u32 l[36];
  int nl;
  if (k >= 0 && t < 0) {
    const u64 ip = -t >= 64 ? 0ull : x >> -t;
    const bool fr = -t >= 64 ? x != 0ull : (x & ((1ull << -t) - 1ull)) != 0ull;
    u64 p = 1;
    for (int i = 0; i < k; ++i) p *= 10u;
    *sticky = fr || (ip % p) != 0ull;
    return ip / p;
  }
  if (k >= 0) {  // (x << t) / 10^k
    for (int i = 0; i < 36; ++i) l[i] = 0u;
    const int ws = t >> 5, bs = t & 31;
    const u64 xs0 = (u64)(u32)x << bs, xs1 = (u64)(u32)(x >> 32) << bs;
    // x << bs spans up to 3 limbs
    const u32 a0 = (u32)xs0, a1 = (u32)(xs0 >> 32) | (u32)xs1, a2 = (u32)(xs1 >> 32);
    l[ws] = a0;
    if (ws + 1 < 36) l[ws + 1] = a1;
    if (ws + 2 < 36) l[ws + 2] = a2;
    nl = ws + 3 < 36 ? ws + 3 : 36;
    bool st = false;
    for (int kk = k; kk > 0;) {
      const int d = kk < 9 ? kk : 9;
      u32 div = 1;
      for (int i = 0; i < d; ++i) div *= 10u;
      u64 rem = 0;
      for (int i = nl - 1; i >= 0; --i) {
        const u64 cur = (rem << 32) | l[i];
        l[i] = (u32)(cur / div);
        rem = cur % div;
      }
      while (nl > 2 && l[nl - 1] == 0u) --nl;
      st |= rem != 0ull;
      kk -= d;
    }
    *sticky = st;
    return ((u64)l[1] << 32) | l[0];
  }
  // x * 10^-k * 2^t = (x * 5^-k) * 2^(t - k)
  for (int i = 0; i < 36; ++i) l[i] = 0u;
  l[0] = (u32)x;
  l[1] = (u32)(x >> 32);
  nl = 2;
  for (int kk = -k; kk > 0;) {
    const int d = kk < 13 ? kk : 13;
    u32 mul = 1;
    for (int i = 0; i < d; ++i) mul *= 5u;
    u64 carry = 0;
    for (int i = 0; i < nl; ++i) {
      const u64 cur = (u64)l[i] * mul + carry;
      l[i] = (u32)cur;
      carry = cur >> 32;
    }
    if (carry && nl < 36) l[nl++] = (u32)carry;
    kk -= d;
  }
  const int sh = t - k;
  if (sh >= 0) {
    *sticky = false;
    return (((u64)l[1] << 32) | l[0]) << sh;
  }
  const int r = -sh, ws = r >> 5, bs = r & 31;
  if (ws >= 36) { *sticky = true; return 0ull; }
  bool st = (l[ws] & ((1u << bs) - 1u)) != 0u;
  for (int i = 0; i < ws; ++i) st |= l[i] != 0u;
  *sticky = st;
  const u32 a = l[ws], b = ws + 1 < 36 ? l[ws + 1] : 0u, c = ws + 2 < 36 ? l[ws + 2] : 0u;
  return ((u64)__funnelshift_r(b, c, bs) << 32) | __funnelshift_r(a, b, bs);
}

// writes repr(float) of the binary64 bits (finite); returns the length (<= 24)
__device__ __noinline__ u32 f64_repr(u8* dst, u64 bits) {
  const u32 sgn = (u32)(bits >> 63), ex = (u32)(bits >> 52) & 0x7FFu;
  const u64 m = bits & ((1ull << 52) - 1ull);
  u32 n = 0;
  if (sgn) dst[n++] = '-';
  if (ex == 0u && m == 0ull) { dst[n] = '0'; dst[n + 1] = '.'; dst[n + 2] = '0'; return n + 3u; }
  const u64 f = ex ? (m | (1ull << 52)) : m;
  const int e = ex ? (int)ex - 1075 : -1074;
  const bool closed = (f & 1ull) == 0ull;
  const u64 v4 = 4ull * f, lo4 = v4 - ((m == 0ull && ex > 1u) ? 1ull : 2ull), hi4 = v4 + 2ull;
  const int t = e - 2;
  const int hb = 63 - __clzll((long long)hi4);
  const int k = (((hb + t) * 78913) >> 18) - 17;  // floor(log10 hi) - 17
  bool sl, sv, shh;
  const u64 wl = repr_window_big(lo4, t, k, &sl), wv = repr_window_big(v4, t, k, &sv);
  const u64 wh = repr_window_big(hi4, t, k, &shh);
  // largest p with a multiple of 10^(k+p) in the interval (monotone in p)
  int p = 0;
  u64 p10 = 1, bot = 0, top = 0;
  while (p < 19) {
    const u64 q10 = p10 * 10u;
    u64 nb, nt;
    if (closed) {
      nb = wl / q10 + ((wl % q10) != 0u || sl);
      nt = wh / q10;
    } else {
      nb = wl / q10 + 1u;
      nt = wh / q10 - (((wh % q10) == 0u && !shh) ? 1u : 0u);
    }
    if (nb > nt) break;
    p10 = q10; ++p; bot = nb; top = nt;
  }
  u64 w = wv / p10;
  const u64 r = wv % p10, half = p10 >> 1;
  if (p > 0 && (r > half || (r == half && (sv || (w & 1u))))) ++w;
  if (p > 0) w = w < bot ? bot : (w > top ? top : w);
  u8 dg[20];
  const u32 nd = u64_dec_len(w);
  u64_dec(dg, w, nd);
  const int decpt = (int)nd + k + p;
  if (decpt <= -4 || decpt > 16) {
    dst[n++] = dg[0];
    if (nd > 1u) {
      dst[n++] = '.';
      for (u32 i = 1; i < nd; ++i) dst[n++] = dg[i];
    }
    int x = decpt - 1;
    dst[n++] = 'e';
    dst[n++] = x < 0 ? '-' : '+';
    x = x < 0 ? -x : x;
    if (x >= 100) dst[n++] = (u8)('0' + x / 100);
    dst[n++] = (u8)('0' + (x / 10) % 10);
    dst[n++] = (u8)('0' + x % 10);
  } else if (decpt <= 0) {
    dst[n++] = '0';
    dst[n++] = '.';
    for (int i = 0; i < -decpt; ++i) dst[n++] = '0';
    for (u32 i = 0; i < nd; ++i) dst[n++] = dg[i];
  } else if ((u32)decpt < nd) {
    for (u32 i = 0; i < nd; ++i) {
      if (i == (u32)decpt) dst[n++] = '.';
      dst[n++] = dg[i];
    }
  } else {
    for (u32 i = 0; i < nd; ++i) dst[n++] = dg[i];
    for (u32 i = nd; i < (u32)decpt; ++i) dst[n++] = '0';
    dst[n++] = '.';
    dst[n++] = '0';
  }
  return n;
}

}  // namespace fbx

namespace fbx {

// ---------------------------------------------------------------------------
// Json-kind extraction (viewpipe.py:266-267): json.dumps(value, sort_keys=True,
// separators=(",", ":")) -- ensure_ascii escaping, ints canonical ("-0" -> "0"),
// floats as repr() of the correctly rounded double ("Infinity" on overflow),
// objects re-emitted in code-point key order with the LAST duplicate winning.
// The document was validated by json_extract.  Objects are emitted by
// selection (each step scans the members for the smallest key above the last
// one emitted), containers through an explicit stack: no member storage.
// dst == nullptr measures.  Returns ~0u when a float needs the bignum parse.
// Python model: decimal_tables.json_canon (checked against json.dumps).
// ---------------------------------------------------------------------------
FBX_DI u32 jc_ws(const u8* s, u32 n, u32 i) {
  while (i < n && (s[i] == ' ' || s[i] == '\t' || s[i] == '\n' || s[i] == '\r')) ++i;
  return i;
}
FBX_DI u32 jc_str_end(const u8* s, u32 i) {  // i after the opening quote
  while (s[i] != '"') i += (s[i] == '\\') ? 2u : 1u;
  return i;
}
FBX_DI u32 jc_value_end(const u8* s, u32 n, u32 i) {
  u32 c = s[i];
  if (c == '"') return jc_str_end(s, i + 1) + 1;
  if (c == '{' || c == '[') {
    int depth = 0;
    while (true) {
      c = s[i];
      if (c == '"') { i = jc_str_end(s, i + 1) + 1; continue; }
      if (c == '{' || c == '[') ++depth;
      else if ((c == '}' || c == ']') && --depth == 0) return i + 1;
      ++i;
    }
  }
  while (i < n) {
    c = s[i];
    if (c == ',' || c == '}' || c == ']' || c == ' ' || c == '\t' || c == '\n' || c == '\r') break;
    ++i;
  }
  return i;
}
FBX_DI u32 jc_hex4(const u8* p) {
  return (j_hexval(p[0]) << 12) | (j_hexval(p[1]) << 8) | (j_hexval(p[2]) << 4) | j_hexval(p[3]);
}
// next code point of a string body (escapes decoded, surrogate pairs joined)
FBX_DI u32 jc_next_cp(const u8* s, u32& i) {
  const u32 c = s[i];
  if (c != '\\') {
    if (c < 0x80u) { ++i; return c; }
    if (c < 0xE0u) { const u32 cp = ((c & 0x1Fu) << 6) | (s[i + 1] & 0x3Fu); i += 2; return cp; }
    if (c < 0xF0u) {
      const u32 cp = ((c & 0x0Fu) << 12) | ((s[i + 1] & 0x3Fu) << 6) | (s[i + 2] & 0x3Fu);
      i += 3;
      return cp;
    }
    const u32 cp = ((c & 0x07u) << 18) | ((s[i + 1] & 0x3Fu) << 12) | ((s[i + 2] & 0x3Fu) << 6) |
                   (s[i + 3] & 0x3Fu);
    i += 4;
    return cp;
  }
  const u32 x = s[i + 1];
  if (x != 'u') {
    i += 2;
    return x == 'b' ? 8u : x == 'f' ? 12u : x == 'n' ? 10u : x == 'r' ? 13u : x == 't' ? 9u : x;
  }
  u32 cp = jc_hex4(s + i + 2);
  i += 6;
  if (cp >= 0xD800u && cp <= 0xDBFFu && s[i] == '\\' && s[i + 1] == 'u') {
    const u32 lo = jc_hex4(s + i + 2);
    if (lo >= 0xDC00u && lo <= 0xDFFFu) {
      cp = 0x10000u + ((cp - 0xD800u) << 10) + (lo - 0xDC00u);
      i += 6;
    }
  }
  return cp;
}
// code-point order of two string bodies [ab, ae) and [bb, be)
FBX_DI int jc_key_cmp(const u8* s, u32 ab, u32 ae, u32 bb, u32 be) {
  while (ab < ae && bb < be) {
    const u32 x = jc_next_cp(s, ab), y = jc_next_cp(s, bb);
    if (x != y) return x < y ? -1 : 1;
  }
  return (ab < ae) ? 1 : ((bb < be) ? -1 : 0);
}
FBX_DI void jc_put(u8* dst, u32& o, u32 c) { if (dst) dst[o] = (u8)c; ++o; }
FBX_DI void jc_put_u(u8* dst, u32& o, u32 v) {
  const char* hx = "0123456789abcdef";
  jc_put(dst, o, '\\'); jc_put(dst, o, 'u');
  jc_put(dst, o, hx[(v >> 12) & 15u]); jc_put(dst, o, hx[(v >> 8) & 15u]);
  jc_put(dst, o, hx[(v >> 4) & 15u]); jc_put(dst, o, hx[v & 15u]);
}
FBX_DI void jc_put_str(const u8* s, u32 b, u32 e, u8* dst, u32& o) {
  jc_put(dst, o, '"');
  for (u32 i = b; i < e;) {
    const u32 cp = jc_next_cp(s, i);
    if (cp == '"' || cp == '\\') { jc_put(dst, o, '\\'); jc_put(dst, o, cp); }
    else if (cp >= 0x20u && cp <= 0x7Eu) jc_put(dst, o, cp);
    else if (cp == 8u) { jc_put(dst, o, '\\'); jc_put(dst, o, 'b'); }
    else if (cp == 12u) { jc_put(dst, o, '\\'); jc_put(dst, o, 'f'); }
    else if (cp == 10u) { jc_put(dst, o, '\\'); jc_put(dst, o, 'n'); }
    else if (cp == 13u) { jc_put(dst, o, '\\'); jc_put(dst, o, 'r'); }
    else if (cp == 9u) { jc_put(dst, o, '\\'); jc_put(dst, o, 't'); }
    else if (cp < 0x10000u) jc_put_u(dst, o, cp);
    else {
      const u32 v = cp - 0x10000u;
      jc_put_u(dst, o, 0xD800u | (v >> 10));
      jc_put_u(dst, o, 0xDC00u | (v & 0x3FFu));
    }
  }
  jc_put(dst, o, '"');
}
// a scalar at [b, e): string (quotes included), number or literal
FBX_DI bool jc_put_scalar(const u8* s, u32 b, u32 e, u8* dst, u32& o) {
  const u32 c = s[b];
  if (c == '"') { jc_put_str(s, b + 1, e - 1, dst, o); return true; }
  if (c == '-' && s[b + 1] == 'I') { for (u32 i = b; i < e; ++i) jc_put(dst, o, s[i]); return true; }
  if (c != '-' && (c - '0') >= 10u) { for (u32 i = b; i < e; ++i) jc_put(dst, o, s[i]); return true; }
  bool flt = false;
  for (u32 i = b; i < e; ++i) flt |= (s[i] == '.' || s[i] == 'e' || s[i] == 'E');
  if (!flt) {  // Python int: digits as written, except -0
    if (c == '-' && e - b == 2u && s[b + 1] == '0') { jc_put(dst, o, '0'); return true; }
    for (u32 i = b; i < e; ++i) jc_put(dst, o, s[i]);
    return true;
  }
  JLeaf lf{b, e, J_FLOAT, 0u};
  u64 db;
  {
    u32 i = lf.beg;
    const bool neg = s[i] == '-';
    if (neg) ++i;
    u64 w = 0;
    u32 sig = 0;
    int e10 = 0;
    bool exact = true, frac = false;
    for (; i < lf.end; ++i) {
      const u32 ch = s[i];
      if (ch == '.') { frac = true; continue; }
      if (ch == 'e' || ch == 'E') break;
      const u32 d = ch - '0';
      if (frac) --e10;
      if (sig == 0 && d == 0) continue;
      if (sig < 19) { w = w * 10u + d; ++sig; }
      else { ++e10; if (d) exact = false; }
    }
    if (i < lf.end) {
      ++i;
      bool eneg = false;
      if (s[i] == '+' || s[i] == '-') { eneg = s[i] == '-'; ++i; }
      int ev = 0;
      for (; i < lf.end; ++i)
        if (ev < 100000) ev = ev * 10 + (int)(s[i] - '0');
      e10 += eneg ? -ev : ev;
    }
    const u32 st = dec_to_double(w, e10, exact, &db);
    if (st == 1u) return false;
    if (neg) db |= 0x8000000000000000ull;
  }
  if ((db & 0x7FFFFFFFFFFFFFFFull) == 0x7FF0000000000000ull) {
    if (db >> 63) jc_put(dst, o, '-');
    const char* w = "Infinity";
    for (int i = 0; i < 8; ++i) jc_put(dst, o, (u8)w[i]);
    return true;
  }
  u8 buf[32];
  const u32 L = f64_repr(buf, db);
  for (u32 i = 0; i < L; ++i) jc_put(dst, o, buf[i]);
  return true;
}

constexpr int JC_MAXD = 64;
struct JcFrame {
  u32 obj, pos, lkb, lke, first;
};

// json.dumps(..., sort_keys=True, separators=(",", ":")) of the leaf; ~0u: unsupported
__device__ __noinline__ u32 json_canon(const u8* s, u32 n, JLeaf lf, u8* dst) {
  u32 o = 0;
  if (lf.type != J_CONTAINER) {
    if (lf.type == J_STRING) { jc_put_str(s, lf.beg, lf.end, dst, o); return o; }
    u32 b = lf.beg, e = lf.end;
    if (!jc_put_scalar(s, b, e, dst, o)) return ~0u;
    return o;
  }
  JcFrame st[JC_MAXD];
  int d = 0;
  u32 i0 = lf.beg;
  st[0] = JcFrame{s[i0] == '{' ? 1u : 0u, jc_ws(s, n, i0 + 1), 0u, 0u, 1u};
  jc_put(dst, o, s[i0]);
  d = 1;
  while (d > 0) {
    JcFrame& f = st[d - 1];
    u32 vb, ve;
    if (!f.obj) {
      const u32 i = f.pos;
      if (s[i] == ']') { jc_put(dst, o, ']'); --d; continue; }
      if (!f.first) jc_put(dst, o, ',');
      f.first = 0u;
      vb = i;
      ve = jc_value_end(s, n, i);
      u32 nx = jc_ws(s, n, ve);
      if (s[nx] == ',') nx = jc_ws(s, n, nx + 1);
      f.pos = nx;
    } else {
      u32 bkb = 0, bke = 0, bv = 0;
      bool have = false;
      u32 i = f.pos;
      while (s[i] != '}') {
        const u32 kb = i + 1, ke = jc_str_end(s, kb);
        u32 vi = jc_ws(s, n, ke + 1);
        vi = jc_ws(s, n, vi + 1);
        const u32 vend = jc_value_end(s, n, vi);
        if (f.first || jc_key_cmp(s, kb, ke, f.lkb, f.lke) > 0) {
          if (!have || jc_key_cmp(s, kb, ke, bkb, bke) <= 0) {  // equal: the later one wins
            bkb = kb; bke = ke; bv = vi; have = true;
          }
        }
        i = jc_ws(s, n, vend);
        if (s[i] == ',') i = jc_ws(s, n, i + 1);
      }
      if (!have) { jc_put(dst, o, '}'); --d; continue; }
      if (!f.first) jc_put(dst, o, ',');
      f.first = 0u;
      f.lkb = bkb;
      f.lke = bke;
      jc_put_str(s, bkb, bke, dst, o);
      jc_put(dst, o, ':');
      vb = bv;
      ve = jc_value_end(s, n, bv);
    }
    if (s[vb] == '{' || s[vb] == '[') {
      if (d >= JC_MAXD) return ~0u;
      st[d] = JcFrame{s[vb] == '{' ? 1u : 0u, jc_ws(s, n, vb + 1), 0u, 0u, 1u};
      jc_put(dst, o, s[vb]);
      ++d;
    } else if (!jc_put_scalar(s, vb, ve, dst, o)) {
      return ~0u;
    }
  }
  return o;
}

}  // namespace fbx
