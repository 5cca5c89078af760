// posit32.cuh -- Posit(32,2) scalar arithmetic for sm_100a device code.
//
// Product path (shares nothing with oracle/).  Every operation returns the
// correctly rounded result of the exact value: round-to-nearest-even on the
// encoding, saturation at +-maxpos / +-minpos, NaR absorbing
// (Eq.1 P:123-138 for the format; P:146-151 for decode ->
// operate -> encode; readings Q1-Q5).
//
// Design (B200-first, not the paper's SoftPosit loop): the regime run is
// found with one __clz on x ^ (x >> 31) instead of the sequential bit loop
// whose magnitude-dependent cost the paper measures (Table
// tabprof).  Decoded values are (sign, scale E, significand M with the hidden
// bit at bit 31).  Exact intermediate results are formed in 64-bit integers
// with a sticky bit jammed into bit 0, and rounded once by writing the posit
// bit string regime || e || fraction and applying RNE to its first 31 bits.
#pragma once
#include <stdint.h>

namespace p32 {

constexpr uint32_t NAR = 0x80000000u;
constexpr uint32_t ONE = 0x40000000u;
constexpr uint32_t MONE = 0xC0000000u;
constexpr uint32_t MAXPOS = 0x7FFFFFFFu;

struct Dec {
  int32_t E;      // scale: value = (-1)^neg * M * 2^(E - 31)
  uint32_t M;     // significand, hidden bit at 31 (0 for zero)
  uint32_t neg;   // 0 or 1
  uint32_t kind;  // 0 zero, 1 NaR, 2 number
};

// Decode with one count-leading-zeros (branch-free for numbers).
__device__ __forceinline__ Dec decode(uint32_t x) {
  Dec d;
  d.neg = x >> 31;
  const uint32_t a = d.neg ? (0u - x) : x;          // two's complement magnitude (reading Q4)
  const uint32_t y = a << 1;                         // regime starts at bit 31
  const uint32_t t = (uint32_t)((int32_t)y >> 31);   // all ones iff the run is of 1s
  const int m = __clz((int)(y ^ t));                 // run length (1..31 for numbers)
  const int k = t ? (m - 1) : -m;
  const uint32_t rest = (y << (m & 31)) << 1;        // bits after the terminator
  const int e = (int)(rest >> 30);                   // missing exponent bits read as 0
  d.E = 4 * k + e;
  d.M = 0x80000000u | ((rest << 2) >> 1);            // 1.f, fraction left-aligned below bit 31
  d.kind = (x == 0u) ? 0u : ((x == NAR) ? 1u : 2u);
  if (x == 0u) d.M = 0u;
  return d;
}

// Round the exact nonzero value (-1)^neg * S * 2^(E - 63) to a pattern.
// S has its leading one at bit 63; a sticky for discarded bits must already be
// OR-ed into S's bit 0 (bit 0 is far below any rounding position).
__device__ __forceinline__ uint32_t round_encode(uint32_t neg, int32_t E, uint64_t S) {
  uint32_t p;
  if (E >= 120) {
    p = MAXPOS;                                      // |x| >= maxpos (reading Q2)
  } else if (E < -120) {
    p = 1u;                                          // |x| < minpos -> minpos
  } else {
    const int k = E >> 2;                            // floor(E / 4)
    const uint32_t e = (uint32_t)(E & 3);
    // regime: k >= 0 -> (k+1) ones then 0 ; k < 0 -> (-k) zeros then 1
    const int rl = (k >= 0) ? (k + 2) : (1 - k);     // regime length incl. terminator, 2..31
    const uint64_t reg = (k >= 0) ? ((((uint64_t)1 << (k + 1)) - 1) << 1) : (uint64_t)1;
    const uint64_t frac = S << 1;                    // fraction left-aligned, hidden bit dropped
    uint64_t v = (reg << (64 - rl)) | ((uint64_t)e << (62 - rl)) | (frac >> (rl + 2));
    const uint64_t lost = frac << (62 - rl);         // bits of frac shifted out above (rl+2 <= 33)
    p = (uint32_t)(v >> 33);                         // first 31 bits of the string
    const uint32_t guard = (uint32_t)(v >> 32) & 1u;
    const uint32_t sticky = ((uint32_t)v != 0u) | (lost != 0);
    p += guard & (sticky | (p & 1u));                // RNE on the encoding (reading Q1)
    if (p == 0u) p = 1u;                             // never round a nonzero to 0 (E == -120 edge)
  }
  return neg ? (0u - p) : p;
}

__device__ __forceinline__ uint32_t neg(uint32_t a) { return 0u - a; }

__device__ __forceinline__ uint32_t mul(uint32_t a, uint32_t b) {
  if (a == NAR || b == NAR) return NAR;
  if (a == 0u || b == 0u) return 0u;
  const Dec x = decode(a), y = decode(b);
  uint64_t S = (uint64_t)x.M * (uint64_t)y.M;        // exact 56-bit product, leading one at 62 or 63
  int32_t E = x.E + y.E;
  if (S >> 63) E += 1; else S <<= 1;
  return round_encode(x.neg ^ y.neg, E, S);
}

__device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b) {
  if (a == NAR || b == NAR) return NAR;
  if (a == 0u) return b;
  if (b == 0u) return a;
  Dec x = decode(a), y = decode(b);
  // order by magnitude: patterns' magnitudes compare as integers (P:37 of SPEC: order = int order)
  const uint32_t ma = x.neg ? (0u - a) : a, mb = y.neg ? (0u - b) : b;
  if (mb > ma) { const Dec t = x; x = y; y = t; }
  const uint32_t d = (uint32_t)(x.E - y.E);
  const uint64_t X = (uint64_t)x.M << 31;            // leading one at bit 62
  const uint64_t Yf = (uint64_t)y.M << 31;
  uint64_t Y;
  if (d == 0u) Y = Yf;
  else if (d >= 63u) Y = 1u;                         // entirely below: sticky only
  else Y = (Yf >> d) | (uint64_t)((Yf << (64 - d)) != 0);   // jam the sticky into bit 0
  const uint64_t S = (x.neg == y.neg) ? (X + Y) : (X - Y);
  if (S == 0) return 0u;                             // exact cancellation
  const int lz = __clzll((long long)S);
  return round_encode(x.neg, x.E + 1 - lz, S << lz);
}

__device__ __forceinline__ uint32_t sub(uint32_t a, uint32_t b) { return add(a, neg(b)); }

__device__ __forceinline__ uint32_t div(uint32_t a, uint32_t b) {
  if (a == NAR || b == NAR || b == 0u) return NAR;  // reading Q3
  if (a == 0u) return 0u;
  const Dec x = decode(a), y = decode(b);
  // q = floor(Mx 2^32 / My), r = remainder: estimate with one correctly rounded
  // binary64 division (both operands exact in binary64; |estimate - quotient|
  // < 1), then fix q by the sign / size of the exact 64-bit remainder.
  const uint64_t num = (uint64_t)x.M << 32;
  uint64_t q = (uint64_t)__ddiv_rn((double)x.M * 4294967296.0, (double)y.M);
  int64_t r = (int64_t)(num - q * (uint64_t)y.M);
  if (r < 0) { q -= 1u; r += (int64_t)y.M; }
  else if (r >= (int64_t)y.M) { q += 1u; r -= (int64_t)y.M; }
  int32_t E = x.E - y.E;
  int lz = __clzll((long long)q);                    // 31 (q >= 2^32) or 32
  E += 31 - lz;                                      // leading one at bit 32 -> E, at 31 -> E-1
  uint64_t S = (q << lz) | (uint64_t)(r != 0);       // q occupies <= 33 bits; bit 0 free for the sticky
  return round_encode(x.neg ^ y.neg, E, S);
}

__device__ __forceinline__ uint32_t sqrt(uint32_t a) {
  if (a == NAR || (int32_t)a < 0) return NAR;        // reading Q3
  if (a == 0u) return 0u;
  const Dec x = decode(a);
  const int odd = x.E & 1;
  // value = M * 2^(E-31) = N * 2^(E - odd - 62) with N = (M << odd) << 31 in [2^62, 2^64)
  const uint64_t N = ((uint64_t)x.M << odd) << 31;
  uint64_t r = (uint64_t)__dsqrt_rn((double)N);      // estimate, then make exact
  if (r > 0xFFFFFFFFull) r = 0xFFFFFFFFull;
  while (r * r > N) r--;
  while (r < 0xFFFFFFFFull && (r + 1) * (r + 1) <= N) r++;
  const uint64_t S = (r << 32) | (uint64_t)(r * r != N);   // leading one at 63
  return round_encode(0u, (x.E - odd) / 2, S);
}

__device__ __forceinline__ uint32_t from_f64(double v) {
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  const uint32_t s = (uint32_t)(b >> 63);
  const int ex = (int)((b >> 52) & 0x7FF);
  const uint64_t man = b & 0xFFFFFFFFFFFFFull;
  if (ex == 0x7FF) return NAR;                       // NaN, Inf
  if (ex == 0) return man ? (s ? (0u - 1u) : 1u) : 0u;   // subnormal -> minpos; +-0 -> 0
  const uint64_t S = ((uint64_t)1 << 63) | (man << 11);
  return round_encode(s, ex - 1023, S);
}

__device__ __forceinline__ double to_f64(uint32_t a) {
  if (a == 0u) return 0.0;
  if (a == NAR) return __longlong_as_double(0x7FF8000000000000ll);
  const Dec x = decode(a);
  const uint64_t b = ((uint64_t)x.neg << 63) | ((uint64_t)(x.E + 1023) << 52) | ((uint64_t)(x.M & 0x7FFFFFFFu) << 21);
  return __longlong_as_double((long long)b);
}

}  // namespace p32
