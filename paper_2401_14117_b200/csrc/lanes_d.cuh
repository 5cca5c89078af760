// lanes_d.cuh -- the binary64-pipe MAC (gemm_d.cuh) for the panel-side
// kernels: lane values kept as exact binary64 numbers, and the per-binade
// rounding constant M(E) computed in registers instead of read from a
// shared-memory table (these kernels are latency-bound, and their shared
// memory holds their tiles).
//
// Contract as lanes.cuh (reading Q6): every update c <- c (-) a (x) b
// is one rounded product and one rounded difference; values and operands
// outside the D-MAC's exact range (zero / NaR operands, |E| > 37 operands,
// |E| > 75 values) take the generic pattern path; both give the same bits.
#pragma once
#include <stdint.h>
#include "posit32.cuh"
#include "gemm_d.cuh"

namespace pld {

// M(E) in registers (gemm_d.cuh's table, computed)
__device__ __forceinline__ double m_of(double x) { return pgd::m_reg(x); }

// a (x) b and c (+) p on exact posit values inside the fast range
__device__ __forceinline__ double mul_r(double a, double b) {
  const double M = m_of(__dmul_rn(a, b));
  return __dsub_rn(__fma_rn(a, b, M), M);
}
__device__ __forceinline__ double add_r(double c, double p) {
  const double d = __dadd_rd(c, p), u = __dadd_ru(c, p);
  const uint32_t dlo = (uint32_t)__double2loint(d), dhi = (uint32_t)__double2hiint(d);
  const uint32_t ulo = (uint32_t)__double2loint(u), uhi = (uint32_t)__double2hiint(u);
  const double y = __hiloint2double((int)umin(dhi, uhi), (int)pgd::odd_lo(dlo, ulo));
  const double M = m_of(d);
  return __dsub_rn(__dadd_rn(y, M), M);
}

// |E| of a binary64 value's binade (zero: a large negative number)
__device__ __forceinline__ int32_t ebin(double x) {
  return (int32_t)(((uint32_t)__double2hiint(x) >> 20) & 0x7FFu) - 1023;
}

// a lane value: exact binary64 (dec) or a pattern outside the fast range
struct LD {
  double v;
  uint32_t pat;
  bool dec;
};

// value range of a fast lane: 0 or |E| <= 75
__device__ __forceinline__ bool in_lane_range(double v) {
  const int32_t e = ebin(v);
  return e <= 75 && (e >= -75 || e == -1023);
}

__device__ __forceinline__ void ld_load(LD& c, uint32_t x) {
  c.pat = x;
  double v;
  c.dec = pgd::d_decode(x, v) && in_lane_range(v);
  c.v = v;
}

__device__ __forceinline__ uint32_t ld_pattern(const LD& c) { return c.dec ? pgd::d_encode(c.v) : c.pat; }

// operand view: nonzero and |E| <= 37
__device__ __forceinline__ bool op_fast(double v) {
  const int32_t e = ebin(v);
  return e <= 37 && e >= -37;
}

// c <- c (-) a (x) b: a, b exact values (afast / bfast: inside the operand
// range), ap / bp their patterns for the generic path
__device__ __forceinline__ void ld_fms(LD& c, double a, bool afast, uint32_t ap, double b, bool bfast, uint32_t bp) {
  if (afast && bfast && c.dec) {
    c.v = add_r(c.v, -mul_r(a, b));
    c.dec = in_lane_range(c.v);
    if (!c.dec) c.pat = pgd::d_encode(c.v);
  } else {
    ld_load(c, p32::sub(ld_pattern(c), p32::mul(ap, bp)));
  }
}

// q = b (/) d for exact posit values b (|E| <= 91) and d (fast operand) with
// r = RN(1 / d): q1 = RN(b / d) refined once (faithful), e1 = b - q1 d exact
// (fma; q1 within one ulp), so the exact quotient is q1 + e1 / d; y = the odd
// one of q1 and its neighbour on that side (round to odd at 53 bits), then
// RN(y + M) - M rounds it onto the posit lattice exactly as the exact quotient
// (gemm_d.cuh, the sum's argument).  false: the quotient is not a fast operand.
__device__ __forceinline__ bool div_r(double b, double d, double r, double& x) {
  const double q0 = __dmul_rn(b, r);
  const double e0 = __fma_rn(-q0, d, b);
  const double q1 = __fma_rn(e0, r, q0);
  const double e1 = __fma_rn(-q1, d, b);
  long long pq = __double_as_longlong(q1);
  if (e1 != 0.0 && (pq & 1) == 0) {
    // |exact| > |q1| iff e1 / d has q1's sign
    const bool up = (__double_as_longlong(e1) ^ __double_as_longlong(d) ^ pq) >= 0;
    pq += up ? 1 : -1;
  }
  const double y = __longlong_as_double(pq);
  if (!op_fast(y)) return false;
  const double M = pgd::m_reg(y);
  x = __dsub_rn(__dadd_rn(y, M), M);
  return op_fast(x);
}

// x = sqrt(d) for an exact posit value d > 0 with |E| <= 75: s = RN(sqrt d)
// (correctly rounded), e = d - s s exact (fma: the residual of a correctly
// rounded square root is representable), so the exact root is above s iff
// e > 0; y = the odd one of s and its neighbour on that side (round to odd at
// 53 bits), then RN(y + M) - M is the posit of the exact root (as div_r).
// |E_x| <= 38: the caller checks op_fast(x) before using x as an operand.
__device__ __forceinline__ double sqrt_r(double d) {
  const double s = __dsqrt_rn(d);
  const double e = __fma_rn(-s, s, d);
  long long ps = __double_as_longlong(s);
  if (e != 0.0 && (ps & 1) == 0) ps += e > 0.0 ? 1 : -1;
  const double y = __longlong_as_double(ps);
  const double M = pgd::m_reg(y);
  return __dsub_rn(__dadd_rn(y, M), M);
}

}  // namespace pld
