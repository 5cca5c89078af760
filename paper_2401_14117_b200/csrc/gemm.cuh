// gemm.cuh -- the hot path: Posit(32,2) GEMM / SYRK trailing update on sm_100a.
//
// Computes, for every output element, exactly the order contract of
// DESIGN.md (reading Q6):
//     c <- (beta == 0 ? 0 : C_ij);  for l = 0..K-1:  c <- c (+/-) (a_il (x) b_lj)
// where (x) and (+) are correctly rounded Posit(32,2) mul / add (PAPER.md
// Eq.2; trailing update P:438-442).  No split-K: each output's
// chain runs in one thread, ascending l.
//
// B200 design (not the paper's SoftPosit port):
//  * operands are decoded ONCE per staged element into shared memory as
//    (significand, (scale << 8) | sign) pairs -- the paper's per-operation
//    "pre-processing" loop (Table tabprof) disappears from the
//    inner loop;
//  * the accumulator stays decoded in registers for the whole K loop and is
//    kept ON the posit lattice: every mul and every add is rounded at the
//    posit fraction width f_s(E) = 27 - t(E), t(E) = (E ^ (E >> 31)) >> 2,
//    directly in the decoded domain (valid while f_s >= 1, |E| <= 107);
//  * rounding is RNE via two carry-chained adds (no masks, no branches);
//  * a k-tile that contains a zero, NaR or |scale| > 53 operand is run by the
//    generic per-operation path (uniform branch for the whole CTA); an
//    accumulator whose sum leaves |E| <= 107 marks the thread, which then
//    recomputes its outputs with the generic path.  An exact cancellation
//    (c (+) p == 0) stays in the fast path: the zero accumulator gets a scale
//    far below any product.  Both
//    are bit-identical by construction (same contract), and rare on the
//    paper's workloads (N(0,1) / U[-1,1) data).
#pragma once
#include <stdint.h>
#include "posit32.cuh"

namespace pg {

constexpr int E_STAGE_MAX = 53;    // |Ea|,|Eb| <= 53  ->  |Ea+Eb+1| <= 107
constexpr int T_FAST_MAX = 26;     // f_s >= 1  <=>  t <= 26
constexpr int E_ZERO = -2048;      // scale used for a zero accumulator

struct Params {
  int64_t m, n, k;
  const uint32_t* A; int64_t lda;
  const uint32_t* B; int64_t ldb;
  uint32_t* C; int64_t ldc;
  int neg;        // alpha = -1
  int beta;       // 0 or 1
  const int32_t* stop;   // optional device flag: nonzero -> the kernel is a no-op (potrf after a failure)
  int one = 1;           // the constant 1, passed at run time (keeps IMADs on the FMA pipe)
};

// ---- staging decode --------------------------------------------------------
// A side: significand hidden bit at 31.  B side: hidden bit at 30.
// w = (E << 8) | sign.  Returns "special" (zero, NaR, |E| > 53).
template <int HID>
__device__ __forceinline__ uint2 stage_decode(uint32_t x, uint32_t flip, uint32_t& special) {
  const uint32_t s = (x >> 31) ^ flip;
  const uint32_t a = (x >> 31) ? (0u - x) : x;
  const uint32_t y = a << 1;
  const uint32_t t = (uint32_t)((int32_t)y >> 31);
  const int m = __clz((int)(y ^ t));
  const int k = t ? (m - 1) : -m;
  const uint32_t rest = (y << (m & 31)) << 1;
  const int E = 4 * k + (int)(rest >> 30);
  const uint32_t M = (0x80000000u | ((rest << 2) >> 1)) >> (31 - HID);
  special |= (uint32_t)((x << 1) == 0u) | (uint32_t)(E > E_STAGE_MAX) | (uint32_t)(E < -E_STAGE_MAX);
  return make_uint2(M, ((uint32_t)E << 8) | s);
}

// ---- accumulator <-> pattern (exact: the accumulator is on the lattice) ----
struct Acc { uint32_t M; int32_t E; uint32_t s; };

__device__ __forceinline__ uint32_t acc_encode(const Acc& c) {
  if (c.M == 0u || c.E < -1000) return 0u;          // exact zero (see mac: scale far below range)
  // M hidden at 30 -> S hidden at 63; the sign is bit 0 of c.s
  return p32::round_encode(c.s & 1u, c.E, (uint64_t)c.M << 33);
}

// returns false if the value cannot live in the fast accumulator (NaR, |E| > 107)
__device__ __forceinline__ bool acc_decode(uint32_t x, Acc& c) {
  if (x == 0u) { c.M = 0u; c.E = E_ZERO; c.s = 0u; return true; }   // zero: far below any product
  const p32::Dec d = p32::decode(x);
  c.M = d.M >> 1; c.E = d.E; c.s = d.neg;
  return x != p32::NAR && d.E <= 107 && d.E >= -107;
}

// ---- rounding-position tables ---------------------------------------------
// For a scale E the posit fraction width is f_s(E) = 27 - t(E) with
// t(E) = (E ^ (E >> 31)) >> 2 (valid for |E| <= 107, f_s >= 1).  The shift
// amounts the MAC needs are read from two small shared-memory tables indexed
// by E (one LDS each) instead of being recomputed with ALU ops:
//   product: Tp[E] = { t + 2 (bits of hi below the kept fraction, + n), t + 3 }
//   sum:     Tx[E] = { t + 5 (+ BAD_FLAG if t > 26), t + 3, 2^(27 - t), 0 }
// (the sum rounds the 32 fraction bits only, keeping f_s = 27 - t of them;
//  the hidden bit 2^(27-t) in units of the kept fraction lsb is added
//  back inside the rounding carry chain).
constexpr int TBIAS = 192;               // table index = E + TBIAS, E in [-192, 191]
constexpr int TSIZE = 384;
constexpr uint32_t BAD_FLAG = 1u << 23;  // accumulated with IMAD; checked once per k-slab
constexpr int E_CLAMP = 150;             // accumulator scales are clamped per k-slab (table bounds)
constexpr int E_ZERO_LIMIT = -1000;      // scales below this encode an exact zero accumulator

__device__ __forceinline__ void fill_tables(uint2* tp, uint4* tx, int tid, int nthr) {
  for (int i = tid; i < TSIZE; i += nthr) {
    const int E = i - TBIAS;
    const uint32_t t = (uint32_t)(E ^ (E >> 31)) >> 2;
    tp[i] = make_uint2(t + 2u, t + 3u);
    const bool fast = t <= (uint32_t)T_FAST_MAX;
    tx[i] = make_uint4(t + 5u + (fast ? 0u : BAD_FLAG), t + 3u, fast ? (1u << (27 - t)) : 0u, 0u);
  }
}

// integer multiply-add forced onto the FMA pipe (the ALU pipe is the bottleneck):
// the multiplier comes from a kernel parameter, so ptxas cannot strength-reduce it.
__device__ __forceinline__ uint32_t fmad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

struct MacConst {
  uint32_t one, two, eight, sixteen;   // = 1, 2, 8, 16 at run time (opaque to ptxas)
  uint32_t tp0, tx0;                   // shared-memory byte addresses of table entry E = 0
};

// ---- the decoded-domain MAC -------------------------------------------------
// c <- c (+) (a (x) b), a = (Ma hidden@31, wa), b = (Mb hidden@30, wb).
// badacc accumulates BAD_FLAG when the sum leaves the fast range (the caller
// checks it once per k-slab).
__device__ __forceinline__ void mac(Acc& c, uint32_t Ma, uint32_t wa, uint32_t Mb, uint32_t wb, const MacConst& K,
                                    uint32_t& badacc) {
  // -- product: exact 56-bit product, rounded once at f_s(Ep) -------------
  const uint32_t wab = fmad(wa, K.one, wb);           // (Ea+Eb) << 8 | (sa + sb)
  const uint32_t hi = __umulhi(Ma, Mb);               // [2^29, 2^31)
  const uint32_t lo = Ma * Mb;                        // sticky source
  const uint32_t n = hi >> 30;
  const int32_t Ep = ((int32_t)wab >> 8) + (int32_t)n;
  const uint2 T = lds64(fmad((uint32_t)Ep, K.eight, K.tp0));
  const uint32_t Dp = fmad(n, K.one, T.x);            // bits of hi below the kept fraction
  const uint32_t qp = hi >> Dp;
  const uint32_t yp = __funnelshift_r(0u, hi, Dp) | (qp & 1u);   // dropped bits at top, lsb at bit 0
  uint32_t rp;
  asm("{\n\t.reg .u32 t;\n\t"
      "add.cc.u32 t, %1, 0xFFFFFFFF;\n\t"             // CF = (lo != 0)         (sticky)
      "addc.cc.u32 t, %2, 0x7FFFFFFF;\n\t"            // CF = round up (RNE)
      "addc.u32 %0, %3, 0;\n\t}"
      : "=r"(rp) : "r"(lo), "r"(yp), "r"(qp));
  const uint32_t Mp = rp << T.y;                      // hidden@30 (2^31 if rounding carried)
  // sign of the product = bit 0 of wab (sa + sb); c.s keeps its sign in bit 0 too

  // -- sum: exact aligned add with jammed sticky, rounded once at f_s(Ex) --
  // lexicographic (E, M) compare as one 64-bit signed compare: branch-free
  const long long kp = (long long)(((unsigned long long)(uint32_t)Ep << 32) | Mp);
  const long long kc = (long long)(((unsigned long long)(uint32_t)c.E << 32) | c.M);
  const bool pbig = kp > kc;
  const uint32_t Mbg = pbig ? Mp : c.M;
  const uint32_t Msm = fmad(Mbg, 0u - K.one, fmad(Mp, K.one, c.M));        // the other one
  const uint32_t sbg = pbig ? wab : c.s;
  const int32_t Ebg = max(Ep, c.E);
  const uint32_t ad = fmad((uint32_t)Ebg, K.two, 0u - fmad((uint32_t)Ep, K.one, (uint32_t)c.E));  // |Ep - Ec|
  const uint32_t sh = __funnelshift_rc(Msm, 0u, ad);          // Msm >> min(ad, 32)
  const uint32_t lost = __funnelshift_rc(0u, Msm, ad);        // bits shifted out (nonzero iff any)
  uint32_t jam;
  asm("min.u32 %0, %1, 1;" : "=r"(jam) : "r"(lost));          // sticky of the shifted-out bits
  const uint32_t Msj = sh | jam;                              // jam sticky into bit 0
  const uint32_t eff = (wab ^ c.s) & 1u;                      // effective subtraction
  const uint32_t x = Mbg + (Msj ^ (0u - eff)) + eff;          // |big| +/- |small|, >= 0
  uint32_t flo;
  asm("bfind.u32 %0, %1;" : "=r"(flo) : "r"(x));             // leading one (0xFFFFFFFF if x == 0)
  const uint32_t xf = __funnelshift_r(0u, x, flo);            // fraction bits left-aligned (hidden dropped)
  const uint32_t Exi = fmad(flo, K.one, (uint32_t)Ebg);       // Ex + 30
  const uint4 U = lds128(fmad(Exi, K.sixteen, K.tx0));
  const uint32_t qx = __funnelshift_r(xf, 0u, U.x);          // xf >> (U.x & 31)
  const uint32_t yx = __funnelshift_r(0u, xf, U.x) | (qx & 1u);
  uint32_t rx;
  asm("{\n\t.reg .u32 t;\n\t"
      "add.cc.u32 t, %1, 0x7FFFFFFF;\n\t"
      "addc.u32 %0, %2, %3;\n\t}"                      // + hidden bit + round up
      : "=r"(rx) : "r"(yx), "r"(qx), "r"(U.z));
  const uint32_t Mn = rx << U.y;                              // hidden@30, or 2^31 on carry
  const uint32_t cy = Mn >> 31;
  c.M = Mn >> cy;
  // exact cancellation (x == 0, flo = -1): scale pushed far below any product,
  // so the (zero) accumulator is the small operand of every later add
  const int32_t E1 = (int32_t)Exi + (int32_t)cy - 30;
  c.E = (int32_t)fmad((uint32_t)((int32_t)flo >> 31), 4096u, (uint32_t)E1);
  c.s = sbg;
  badacc = fmad(U.x, K.one, badacc);                          // BAD_FLAG bits accumulate
}

}  // namespace pg
