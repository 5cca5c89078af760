// lanes.cuh -- shared pieces of the panel-side kernels:
// pivot keys, block reductions, and the decoded lane values with the
// decoded-domain MAC / generic fallback that the LU leaf, the TRSMs, the
// diagonal-block Cholesky and the tiny GEMM use.  Device code only (plus two
// launch-size helpers and the launch-error check).
//
// Order contract (reading Q6): every element receives its updates
// one product at a time in ascending k, so every traversal here (blocked,
// recursive, fused, distributed) gives the bits of the textbook loops.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <stdio.h>
#include <stddef.h>
#include <cooperative_groups.h>
#include "gemm.cuh"
#include "internal.h"

namespace pl {

using p32::add;
using p32::div;
using p32::mul;
using p32::sub;

constexpr int TB = 32;                 // in-block TRSM / potf2 leaf width (one warp)

// abs of a pattern compared as a signed int: NaR stays INT32_MIN (the minimum)
__device__ __forceinline__ int32_t abs_key(uint32_t a) {
  const int32_t s = (int32_t)a;
  return s < 0 ? (int32_t)(0u - a) : s;
}

// 64-bit pivot key: larger abs first, then the smaller row (reading Q10)
__device__ __forceinline__ unsigned long long piv_key(uint32_t a, int64_t r) {
  const uint32_t k = (uint32_t)abs_key(a) ^ 0x80000000u;                 // signed -> unsigned order
  return ((unsigned long long)k << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)r);
}

__device__ __forceinline__ unsigned long long block_max(unsigned long long v, unsigned long long* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xFFFFFFFFu, v, o);
    v = w > v ? w : v;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long w = __shfl_xor_sync(0xFFFFFFFFu, v, o);
      v = w > v ? w : v;
    }
  }
  return v;   // valid in thread 0
}

// ---- decoded lane values for the in-block kernels -----------------------------
// A value that lives in a register across many posit updates is kept decoded
// (the GEMM's accumulator format, csrc/gemm.cuh) so that each update
// c <- c (-) a (x) b runs the decoded-domain MAC (one rounding for the product,
// one for the difference, as always) instead of decode -> mul -> encode ->
// decode -> sub -> encode.  Conservative range guards route any update whose
// operands or result could leave the MAC's exact range (zero / NaR operands,
// |E| > 37 operands, |E| > 75 values) to the generic pattern path; both are
// bit-identical by construction.
struct LaneVal {
  pg::Acc a;       // decoded (valid when dec)
  uint32_t pat;    // pattern (valid when !dec)
  bool dec;
};

__device__ __forceinline__ void lv_load(LaneVal& v, uint32_t x) {
  v.pat = x;
  v.dec = pg::acc_decode(x, v.a) && (x == 0u || (v.a.E <= 75 && v.a.E >= -75));
}

__device__ __forceinline__ uint32_t lv_pattern(const LaneVal& v) { return v.dec ? pg::acc_encode(v.a) : v.pat; }

// operand view of a lane value: B format (hidden@30), fast iff nonzero and |E| <= 37
__device__ __forceinline__ bool lv_operand(const LaneVal& v) {
  return v.dec && v.a.E > -1000 && v.a.E <= 37 && v.a.E >= -37;
}

// A-format decode of a pattern operand: fast iff nonzero, not NaR, |E| <= 37
__device__ __forceinline__ bool fast_a(uint32_t x, uint4& d) {
  uint32_t sp = 0u;
  d = pg::stage_decode<31>(x, 0u, sp);
  return sp == 0u && (int32_t)d.y <= 37 && (int32_t)d.y >= -37;
}

// c <- c (-) a (x) b; a = pattern (with its A-format decode), b = operand lane
// value broadcast as (M, E, sg) plus its pattern bp.
__device__ __forceinline__ void lv_fms(LaneVal& c, uint32_t ap, bool afast, const uint4& ad, uint32_t bM, int32_t bE,
                                       int32_t bsg, bool bfast, uint32_t bp) {
  if (afast && bfast && c.dec) {
    uint32_t bad = 0u;
    pg::mac(c.a, ad.x, (int32_t)ad.y, (int32_t)ad.z, bM, bE, -bsg, pg::CalcConst(), bad);
    c.dec = c.a.E <= 75 && c.a.E >= -75 ? true : (c.a.E < -1000);
    if (!c.dec) c.pat = pg::acc_encode(c.a);                 // |E| in (75, 107]: exact, leave the fast range
  } else {
    const uint32_t r = sub(lv_pattern(c), mul(ap, bp));
    lv_load(c, r);
  }
}

// lv_fms with the GEMM's shared-memory tables (or any table type)
template <class Tab>
__device__ __forceinline__ void lv_fms_t(LaneVal& c, uint32_t ap, bool afast, const uint4& ad, uint32_t bM, int32_t bE,
                                         int32_t bsg, bool bfast, uint32_t bp, const Tab& K) {
  if (afast && bfast && c.dec) {
    uint32_t bad = 0u;
    pg::mac(c.a, ad.x, (int32_t)ad.y, (int32_t)ad.z, bM, bE, -bsg, K, bad);
    c.dec = c.a.E <= 75 && c.a.E >= -75 ? true : (c.a.E < -1000);
    if (!c.dec) c.pat = pg::acc_encode(c.a);
  } else {
    const uint32_t r = sub(lv_pattern(c), mul(ap, bp));
    lv_load(c, r);
  }
}

inline unsigned grid_for(int64_t count, int threads) {
  int64_t g = (count + threads - 1) / threads;
  const int64_t cap = (int64_t)pb_num_sms() * 64;
  if (g > cap) g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

inline unsigned rows_grid(int64_t rows, int threads) {
  int64_t g = (rows + threads - 1) / threads;
  const int64_t cap = (int64_t)pb_num_sms() * 4;
  if (g > cap) g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace pl

static inline int last_launch() {
  return cudaPeekAtLastError() == cudaSuccess ? 0 : POSIT_ECUDA;
}
