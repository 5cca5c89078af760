// gemm_d.cuh -- the posit MAC on the binary64 pipe ("D-MAC").
//
// Same contract as gemm.cuh's integer MAC (reading Q6): for every
// output, c <- c (+) (a (x) b) in ascending k, each (x) and (+) one correctly
// rounded Posit(32,2) operation (Eq.2; trailing update
// P:438-442).  Only the machinery differs: posit values inside the fast range
// are exact binary64 numbers (<= 28 significant bits, |scale| <= 107), so
//
//   * the rounding of a value x of binade E onto the posit lattice -- the
//     multiples of q(E) = 2^(E - f_s(E)), f_s(E) = 27 - t(E),
//     t(E) = (E ^ (E >> 31)) >> 2 -- is ONE binary64 round-to-nearest-even
//     addition of the constant M(E) = 1.5 * 2^(E - f_s(E) + 52): x + M(E) lies
//     in M's binade, whose ulp is exactly q(E), and M(E) / q(E) is even, so
//     the parity that breaks ties is the parity of the posit's last fraction
//     bit (RNE on the encoding where no exponent bit is cut, reading Q1);
//     subtracting M(E) again is exact;
//   * the product:  P = fma(a, b, M) - M  rounds the EXACT 56-bit product once
//     (the fma rounds a*b + M in one step).  M is looked up from the binade of
//     RN(a*b) (one DMUL); when that rounding carries into the next binade the
//     exact product is within 2^-53 relative of the power of two, which is a
//     lattice point of both binades, so either constant gives it;
//   * the sum:  c + P is exact in binary64 unless the exponent gap exceeds
//     25.  Rounding its RN value again would double-round, so the sum is
//     first rounded to ODD at 53 bits -- y = the odd one of RD(c + P) and
//     RU(c + P) (equal when exact) -- and then onto the lattice with M: a
//     round-to-odd result at p + 2 or more bits rounds to nearest at p bits
//     exactly as the exact value does (every lattice midpoint is an even
//     53-bit number, and y lies strictly between the same two such numbers
//     as the exact sum).  M comes from the binade of RD(c + P) (the same
//     argument as for the product covers a carry to the next binade).
//
// Per MAC: DMUL, DFMA, 5 DADD (all on the binary64 pipe), two table lookups
// (SHF + address + LDS.64 each), LOP3 + SEL + IMNMX for the odd pick -- about
// 16 issue slots against the integer MAC's 42, and the binary64 pipe is
// otherwise idle.  The fast range is the integer MAC's: operands of a k-slab
// |E| <= 37 (nonzero, not NaR), the accumulator |E| <= 91 at a slab start;
// everything else takes the generic per-operation path (same bits).
#pragma once
#include <stdint.h>
#include <type_traits>
#include "posit32.cuh"

namespace pgd {

// Table entries are indexed by the biased exponent (hi word >> 20, sign masked
// off): one entry per binade for both signs, so a warp whose lanes hold values
// of either sign reads one address per binade (with the sign in the index the
// two copies sat 16 KB apart, in the same banks: r2f ncu, 8.8e9 bank conflicts
// and MIO throttle 7.1 per issue).  PGD_TAB32: 4-byte entries (M's hi word; its
// lo word is 0) -- half the shared-memory wavefronts per lookup.
#ifndef PGD_TAB32
#define PGD_TAB32 1
#endif
constexpr int DT_SIZE = 2048;

// M(E) for the binade of a binary64 whose hi word >> 20 is i.  Entries outside
// |E| <= 110 (and zero, i = 0 / 2048) are never used to round a nonzero value
// in the fast path; they hold M(0) so that 0 + M - M = 0.
__device__ __forceinline__ double dtab_entry(int i) {
  const int e = i & 0x7FF;
  int E = e - 1023;
  if (e == 0 || E < -110 || E > 110) E = 0;
  const int t = (E ^ (E >> 31)) >> 2;
  const int fs = 27 - t;                                   // posit fraction bits at scale E (>= 0 here)
  const uint32_t hi = ((uint32_t)(E - fs + 52 + 1023) << 20) | 0x80000u;   // 1.5 * 2^(E - fs + 52)
  return __hiloint2double((int)hi, 0);
}

__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// The table's element type, T64 = 8-byte entries (M itself, one LDS.64 into
// the register pair) or 4-byte entries (M's hi word; the lo word is then
// assembled, costing an IMAD.MOV per lookup, 1.31 per MAC in k_gemm_d's loop).
// r2g A/B on C2: 8-byte 2810 vs 4-byte 2753 / 2743 Gflop/s, so the GEMM uses
// T64 (PGD_GEMM_TAB64); the panel kernels keep 4-byte entries (PGD_TAB32) to
// keep their shared-memory footprint (three Cholesky TRSM CTAs per SM).
#ifndef PGD_GEMM_TAB64
#define PGD_GEMM_TAB64 1
#endif
constexpr bool T64_PANEL = PGD_TAB32 == 0;
constexpr bool T64_GEMM = PGD_GEMM_TAB64 != 0;
template <bool T64>
using dtab_tt = std::conditional_t<T64, double, uint32_t>;
using dtab_t = dtab_tt<T64_PANEL>;

// the table's fill value for entry i
template <bool T64 = T64_PANEL>
__device__ __forceinline__ dtab_tt<T64> dtab_fill(int i) {
  if constexpr (T64) return dtab_entry(i);
  else return (uint32_t)__double2hiint(dtab_entry(i));
}

// table entry for a binary64 hi word h (tab0: shared-memory byte address of entry 0)
template <bool T64 = T64_PANEL>
__device__ __forceinline__ double mtab_h(uint32_t h, uint32_t tab0) {
  if constexpr (!T64) {
    // lo word = the entry's byte offset: any lo word with an even last bit keeps
    // M / q even and M inside its binade, and the offset register is live anyway
    const uint32_t off = ((h >> 20) & 0x7FFu) << 2;
    return __hiloint2double((int)lds_u32(tab0 + off), (int)off);
  } else {
    return lds_f64(tab0 + (((h >> 20) & 0x7FFu) << 3));
  }
}

// table entry of the binade of x
template <bool T64 = T64_PANEL>
__device__ __forceinline__ double mtab(double x, uint32_t tab0) { return mtab_h<T64>((uint32_t)__double2hiint(x), tab0); }

// M(E) computed in registers: biased exponent eb + 25 + t(E), E = eb - 1023
// (zero, eb = 0, gets a tiny normal M, which leaves 0 at 0)
__device__ __forceinline__ double m_reg(double x) {
  const uint32_t h = (uint32_t)__double2hiint(x);
  const int32_t eb = (int32_t)((h >> 20) & 0x7FFu);
  const int32_t E = eb - 1023;
  const int32_t t = (E ^ (E >> 31)) >> 2;
  return __hiloint2double((int)((((uint32_t)(eb + 25 + t)) << 20) | 0x80000u), 0);
}

#ifndef PGD_PROD_REG                 // 1: the product's M from registers (one table lookup per MAC instead of two)
#define PGD_PROD_REG 0
#endif

// the odd one of two adjacent binary64 patterns' low words: d's if d is odd, else u's
// (LOP3 a & b, LUT 0xC0, with a predicate output + SEL)
__device__ __forceinline__ uint32_t odd_lo(uint32_t dlo, uint32_t ulo) {
  uint32_t y, t;
  asm("{\n\t.reg .pred p;\n\tlop3.or.b32 %1|p, %2, 1, 0, 0xC0, 0;\n\tselp.b32 %0, %2, %3, p;\n\t}"
      : "=r"(y), "=r"(t) : "r"(dlo), "r"(ulo));
  return y;
}

// c (+) (a (x) b): a, b, c exact posit values in binary64, inside the fast range
template <bool T64 = T64_PANEL>
__device__ __forceinline__ double dmac(double c, double a, double b, uint32_t tab0) {
  const double Mp = PGD_PROD_REG ? m_reg(__dmul_rn(a, b)) : mtab<T64>(__dmul_rn(a, b), tab0);
  const double P = __dsub_rn(__fma_rn(a, b, Mp), Mp);     // a (x) b
  const double d = __dadd_rd(c, P), u = __dadd_ru(c, P);
  const uint32_t dlo = (uint32_t)__double2loint(d), dhi = (uint32_t)__double2hiint(d);
  const uint32_t ulo = (uint32_t)__double2loint(u), uhi = (uint32_t)__double2hiint(u);
  // round to odd: the odd one of the two neighbours; their bit patterns are p and p + 1,
  // and the hi word of the odd one is the smaller hi word (a carry only leaves an odd p)
  const uint32_t ylo = odd_lo(dlo, ulo);
  const uint32_t yhi = umin(dhi, uhi);
  const double Mc = mtab_h<T64>(dhi, tab0);
  return __dsub_rn(__dadd_rn(__hiloint2double((int)yhi, (int)ylo), Mc), Mc);   // c (+) P
}

// c (+) P for an already rounded product P (the sum half of dmac)
template <bool T64 = T64_PANEL>
__device__ __forceinline__ double dadd_pos(double c, double P, uint32_t tab0) {
  const double d = __dadd_rd(c, P), u = __dadd_ru(c, P);
  const uint32_t dlo = (uint32_t)__double2loint(d), dhi = (uint32_t)__double2hiint(d);
  const uint32_t ulo = (uint32_t)__double2loint(u), uhi = (uint32_t)__double2hiint(u);
  const uint32_t ylo = odd_lo(dlo, ulo);
  const uint32_t yhi = umin(dhi, uhi);
  const double Mc = mtab_h<T64>(dhi, tab0);
  return __dsub_rn(__dadd_rn(__hiloint2double((int)yhi, (int)ylo), Mc), Mc);
}

// a (x) b (the product half of dmac)
template <bool T64 = T64_PANEL>
__device__ __forceinline__ double dmul_pos(double a, double b, uint32_t tab0) {
  const double Mp = mtab<T64>(__dmul_rn(a, b), tab0);
  return __dsub_rn(__fma_rn(a, b, Mp), Mp);
}

// ---- conversions ------------------------------------------------------------
// posit pattern -> its exact binary64 value (sign flipped by `flip`); `special`
// collects zero, NaR and |E| > EMAX (outside the fast range; the value is then
// not used).
template <int EMAX = 37>
__device__ __forceinline__ double stage_decode_d(uint32_t x, uint32_t flip, uint32_t& special) {
  const uint32_t s = (x >> 31) ^ flip;
  const uint32_t a = (x >> 31) ? (0u - x) : x;
  const uint32_t y = a << 1;
  const uint32_t t = (uint32_t)((int32_t)y >> 31);
  const int m = __clz((int)(y ^ t));
  const int k = t ? (m - 1) : -m;
  const uint32_t rest = (y << (m & 31)) << 1;
  const int E = 4 * k + (int)(rest >> 30);
  const uint32_t f = rest << 2;                                  // fraction, left-aligned
  special |= (uint32_t)((x << 1) == 0u) | (uint32_t)(E > EMAX) | (uint32_t)(E < -EMAX);
  const uint32_t hi = (s << 31) | ((uint32_t)(E + 1023) << 20) | (f >> 12);
  return __hiloint2double((int)hi, (int)(f << 20));
}

// exact value of a posit that is 0 or has |E| <= 107 (else returns false: NaR
// or outside the exact range of the fast accumulator)
__device__ __forceinline__ bool d_decode(uint32_t x, double& v) {
  if (x == 0u) { v = 0.0; return true; }
  const p32::Dec dd = p32::decode(x);
  const uint32_t f = dd.M << 1;                                  // hidden bit dropped, fraction left-aligned
  const uint32_t hi = (dd.neg << 31) | ((uint32_t)(dd.E + 1023) << 20) | (f >> 12);
  v = __hiloint2double((int)hi, (int)(f << 20));
  return x != p32::NAR && dd.E <= 107 && dd.E >= -107;
}

// pattern of a binary64 value ON the posit lattice (every D-MAC result is):
// regime, exponent and fraction assembled without rounding for |E| <= 107,
// the generic rounding encoder beyond
__device__ __forceinline__ uint32_t d_encode(double v) {
  const uint32_t hi = (uint32_t)__double2hiint(v), lo = (uint32_t)__double2loint(v);
  const uint32_t eb = (hi >> 20) & 0x7FFu;
  if (eb == 0u) return 0u;                                       // zero (no subnormal is ever formed)
  const int32_t E = (int32_t)eb - 1023;
  const uint32_t f = (hi << 12) | (lo >> 20);                    // top 32 fraction bits
  if (E <= 107 && E >= -107) {
    const int32_t k = E >> 2;
    const uint32_t e = (uint32_t)E & 3u;
    const int32_t rl = k >= 0 ? k + 2 : 1 - k;
    const uint32_t reg = k >= 0 ? (0x7FFFFFFFu ^ (0x7FFFFFFFu >> (k + 1))) : (1u << (30 + k));
    const uint32_t body = reg | (e << (29 - rl)) | (f >> (rl + 3));
    return (hi >> 31) ? 0u - body : body;
  }
  const uint64_t S = (1ull << 63) | ((uint64_t)f << 31) | ((uint64_t)(lo & 0xFFFFFu) << 11);
  return p32::round_encode(hi >> 31, E, S);
}

// binary64 hi word -> the accumulator is above the slab-start limit
__device__ __forceinline__ bool d_above(double v, int limit) {
  return (int)(((uint32_t)__double2hiint(v) >> 20) & 0x7FFu) > 1023 + limit;
}

}  // namespace pgd
