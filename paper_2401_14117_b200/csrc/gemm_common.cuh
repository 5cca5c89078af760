// gemm_common.cuh -- pieces shared by the two GEMM/SYRK kernel families
// (k_gemm: the integer-pipe MAC, gemm.cu; k_gemm_d: the binary64-pipe MAC,
// gemm_d.cu): the generic per-operation slow path and the tile-load helpers.
#pragma once
#include <stdint.h>
#include "posit32.cuh"
#include "gemm.cuh"

namespace pg {

// Generic per-operation MAC on patterns (the slow path; bit-identical to the
// fast path by the contract).
static __device__ __forceinline__ uint32_t mac_generic(uint32_t c, uint32_t a, uint32_t b, int neg) {
  const uint32_t p = p32::mul(a, b);
  return p32::add(c, neg ? p32::neg(p) : p);
}

// Generic path over one k-slab for one accumulator (noinline and all-scalar
// arguments: keeps the fast loop's accumulators in registers).  Returns the
// new accumulator (x = M, y = E, z = s) and w = 1 if the result cannot live
// in the fast accumulator.
static __device__ __noinline__ uint4 slow_slab(uint32_t M, int32_t E, int32_t sg, const uint32_t* A, int64_t lda,
                                        const uint32_t* B, int64_t ldb, int neg, int64_t r, int64_t cc, int64_t k0,
                                        int kmax, int transb, int transa) {
  Acc acc{M, E, sg};
  uint32_t c = acc_encode(acc);
  for (int kk = 0; kk < kmax; kk++) {
    const int64_t l = k0 + kk;
    const uint32_t a = transa ? A[l * lda + r] : A[r * lda + l];
    const uint32_t b = transb ? B[cc * ldb + l] : B[l * ldb + cc];
    c = mac_generic(c, a, b, neg);
  }
  const uint32_t bad = acc_decode(c, acc) ? 0u : 1u;
  return make_uint4(acc.M, (uint32_t)acc.E, (uint32_t)acc.sg, bad);
}

// Whole chain of one output with the generic path (the recompute of a thread
// whose fast accumulator left the fast range).
static __device__ __noinline__ uint32_t slow_chain(const uint32_t* A, int64_t lda, const uint32_t* B, int64_t ldb,
                                            const uint32_t* C, int64_t ldc, int beta, int neg, int64_t K, int64_t r,
                                            int64_t cc, int transb, int transa) {
  uint32_t c = beta ? C[r * ldc + cc] : 0u;
  for (int64_t l = 0; l < K; l++) {
    const uint32_t a = transa ? A[l * lda + r] : A[r * lda + l];
    const uint32_t b = transb ? B[cc * ldb + l] : B[l * ldb + cc];
    c = mac_generic(c, a, b, neg);
  }
  return c;
}

// Four consecutive words of a row, the ones at index >= avail (or all if
// !row_ok) replaced by 1.0 (a harmless operand for padded tile slots): one
// 128-bit read-only load when the quad is complete and 16-byte aligned.
static __device__ __forceinline__ void load_quad(const uint32_t* p, bool row_ok, int64_t avail, uint32_t* out) {
  if (row_ok && avail >= 4 && (((uintptr_t)p) & 15u) == 0u) {
    uint4 v;
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
  } else {
#pragma unroll
    for (int q = 0; q < 4; q++) out[q] = (row_ok && q < avail) ? __ldg(p + q) : p32::ONE;
  }
}

// cp.async of one quad into shared memory (16 B when complete and aligned,
// else word by word; slots past the matrix are left untouched and replaced by
// 1.0 at decode time)
static __device__ __forceinline__ void cp_quad(uint32_t* dst, const uint32_t* p, bool row_ok, int64_t avail) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  if (row_ok && avail >= 4 && (((uintptr_t)p) & 15u) == 0u) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(p));
  } else {
#pragma unroll
    for (int q = 0; q < 4; q++)
      if (row_ok && q < avail) asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d + 4u * q), "l"(p + q));
  }
}

}  // namespace pg
