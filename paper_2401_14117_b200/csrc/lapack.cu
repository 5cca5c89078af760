// lapack.cu -- the panel steps around the trailing update (SURVEY 8(a) rows
// a8-a11): LU panel (pivot search by signed compare of patterns, row swap,
// posit division, in-panel update), laswp, the two TRSM variants, potf2, and
// the elementwise / conversion kernels.  All on the device, stream-ordered.
//
// Order contract (reading Q6): every element receives its updates
// one product at a time in ascending k; the TRSMs are blocked into a small
// in-block substitution plus a fast-path GEMM for the rows/columns beyond the
// block, which is a traversal change only.
#include <cuda_runtime.h>
#include <stdint.h>
#include "gemm.cuh"
#include "internal.h"

namespace pl {

using p32::add;
using p32::div;
using p32::mul;
using p32::sub;

constexpr int PIV_THREADS = 1024;

// abs of a pattern compared as a signed int: NaR stays INT32_MIN (the minimum)
__device__ __forceinline__ int32_t abs_key(uint32_t a) {
  const int32_t s = (int32_t)a;
  return s < 0 ? (int32_t)(0u - a) : s;
}

// Column j of the m x b panel: pivot search over rows j..m-1 (max abs, ties ->
// smallest row, reading Q10), ipiv, swap inside the panel, divide (Q8, Q11).
__global__ void __launch_bounds__(PIV_THREADS) k_panel_pivot(uint32_t* A, int64_t lda, int64_t m, int64_t b, int64_t j,
                                                             int32_t* ipiv, int32_t* info, int64_t row_base) {
  __shared__ unsigned long long red[PIV_THREADS / 32];
  __shared__ int64_t s_p;
  __shared__ uint32_t s_v;
  unsigned long long best = 0ull;
  for (int64_t r = j + threadIdx.x; r < m; r += blockDim.x) {
    const uint32_t key = (uint32_t)abs_key(A[r * lda + j]) ^ 0x80000000u;   // signed -> unsigned order
    const unsigned long long k64 = ((unsigned long long)key << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)r);
    best = k64 > best ? k64 : best;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xFFFFFFFFu, best, o);
    best = other > best ? other : best;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    best = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xFFFFFFFFu, best, o);
      best = other > best ? other : best;
    }
    if (threadIdx.x == 0) {
      const int64_t p = (int64_t)(0xFFFFFFFFu - (uint32_t)(best & 0xFFFFFFFFull));
      s_p = p;
      s_v = A[p * lda + j];
      ipiv[j] = (int32_t)(row_base + p + 1);
      if (s_v == 0u && *info == 0) *info = (int32_t)(row_base + j + 1);
    }
  }
  __syncthreads();
  const int64_t p = s_p;
  const uint32_t v = s_v;
  if (v == 0u) return;                      // zero pivot: no swap, no division (Q11)
  if (p != j) {
    for (int64_t c = threadIdx.x; c < b; c += blockDim.x) {
      const uint32_t t = A[j * lda + c];
      A[j * lda + c] = A[p * lda + c];
      A[p * lda + c] = t;
    }
    __syncthreads();
  }
  for (int64_t r = j + 1 + threadIdx.x; r < m; r += blockDim.x) A[r * lda + j] = div(A[r * lda + j], v);
}

// a_rq <- a_rq (-) a_rj (x) a_jq for j < r < m, j < q < b  (one thread per element)
__global__ void k_panel_update(uint32_t* A, int64_t lda, int64_t m, int64_t b, int64_t j) {
  const int64_t w = b - j - 1;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (m - j - 1) * w) return;
  const int64_t r = j + 1 + e / w, q = j + 1 + e % w;
  A[r * lda + q] = sub(A[r * lda + q], mul(A[r * lda + j], A[j * lda + q]));
}

// rows k1..k2-1 swapped with ipiv[k]-1-base, in order, for columns [0, ncols)
__global__ void k_laswp(uint32_t* A, int64_t lda, int64_t ncols, int64_t k1, int64_t k2, const int32_t* ipiv,
                        int64_t base) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  for (int64_t k = k1; k < k2; k++) {
    const int64_t r2 = (int64_t)ipiv[k] - 1 - base;
    if (r2 != k) {
      const uint32_t t = A[k * lda + c];
      A[k * lda + c] = A[r2 * lda + c];
      A[r2 * lda + c] = t;
    }
  }
}

// In-block forward substitution, unit lower: rows i0..i0+ib-1 of B, one thread per column.
__global__ void k_trsm_llnu_block(const uint32_t* L, int64_t ldl, uint32_t* B, int64_t ldb, int64_t i0, int64_t ib,
                                  int64_t n) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  for (int64_t i = i0; i < i0 + ib; i++) {
    uint32_t v = B[i * ldb + c];
    for (int64_t k = i0; k < i; k++) v = sub(v, mul(L[i * ldl + k], B[k * ldb + c]));
    B[i * ldb + c] = v;
  }
}

// In-block right solve with L^T, non-unit: columns j0..j0+jb-1 of B, one thread per row.
__global__ void k_trsm_rltn_block(const uint32_t* L, int64_t ldl, uint32_t* B, int64_t ldb, int64_t j0, int64_t jb,
                                  int64_t m, const int32_t* stop) {
  if (stop != nullptr && *stop != 0) return;
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= m) return;
  for (int64_t j = j0; j < j0 + jb; j++) {
    uint32_t v = B[r * ldb + j];
    for (int64_t k = j0; k < j; k++) v = sub(v, mul(B[r * ldb + k], L[j * ldl + k]));
    B[r * ldb + j] = div(v, L[j * ldl + j]);
  }
}

// Unblocked Cholesky of the b x b diagonal block (lower), one CTA (reading Q9).
__global__ void __launch_bounds__(1024) k_potf2(uint32_t* A, int64_t lda, int64_t b, int32_t* info, int64_t row_base) {
  __shared__ int s_fail;
  __shared__ uint32_t s_d;
  if (*info != 0) return;                       // an earlier block failed: stop
  for (int64_t k = 0; k < b; k++) {
    if (threadIdx.x == 0) {
      const uint32_t v = A[k * lda + k];
      if ((int32_t)v <= 0) {                     // zero, negative or NaR pivot
        s_fail = 1;
        *info = (int32_t)(row_base + k + 1);
      } else {
        s_fail = 0;
        s_d = p32::sqrt(v);
        A[k * lda + k] = s_d;
      }
    }
    __syncthreads();
    if (s_fail) return;
    const uint32_t d = s_d;
    for (int64_t i = k + 1 + threadIdx.x; i < b; i += blockDim.x) A[i * lda + k] = div(A[i * lda + k], d);
    __syncthreads();
    const int64_t w = b - k - 1;
    for (int64_t e = threadIdx.x; e < w * w; e += blockDim.x) {
      const int64_t i = k + 1 + e / w, jj = k + 1 + e % w;
      if (jj <= i) A[i * lda + jj] = sub(A[i * lda + jj], mul(A[i * lda + k], A[jj * lda + k]));
    }
    __syncthreads();
  }
}

__global__ void k_vec_op(int op, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t x = a[i];
    uint32_t r;
    switch (op) {
      case POSIT_OP_ADD: r = add(x, b[i]); break;
      case POSIT_OP_SUB: r = sub(x, b[i]); break;
      case POSIT_OP_MUL: r = mul(x, b[i]); break;
      case POSIT_OP_DIV: r = div(x, b[i]); break;
      default: r = p32::sqrt(x); break;
    }
    out[i] = r;
  }
}

__global__ void k_from_f64(const double* x, uint32_t* out, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = p32::from_f64(x[i]);
}

__global__ void k_to_f64(const uint32_t* p, double* out, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = p32::to_f64(p[i]);
}

inline unsigned grid_for(int64_t count, int threads) {
  int64_t g = (count + threads - 1) / threads;
  if (g > 148 * 64) g = 148 * 64;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace pl

using namespace pl;

static int last_launch() {
  return cudaPeekAtLastError() == cudaSuccess ? 0 : POSIT_ECUDA;
}

int pb_getrf_panel(int64_t m, int64_t b, uint32_t* A, int64_t lda, int32_t* ipiv, int32_t* info, int64_t row_base,
                   const int32_t* stop, cudaStream_t st) {
  (void)stop;
  const int64_t jmax = m < b ? m : b;
  for (int64_t j = 0; j < jmax; j++) {
    k_panel_pivot<<<1, PIV_THREADS, 0, st>>>(A, lda, m, b, j, ipiv, info, row_base);
    const int64_t cnt = (m - j - 1) * (b - j - 1);
    if (cnt > 0) k_panel_update<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(A, lda, m, b, j);
  }
  return last_launch();
}

int pb_laswp(int64_t ncols, uint32_t* A, int64_t lda, int64_t k1, int64_t k2, const int32_t* ipiv, int64_t ipiv_base,
             cudaStream_t st) {
  if (ncols <= 0 || k2 <= k1) return 0;
  k_laswp<<<(unsigned)((ncols + 255) / 256), 256, 0, st>>>(A, lda, ncols, k1, k2, ipiv, ipiv_base);
  return last_launch();
}

static constexpr int64_t TRSM_BLK = 16;

int pb_trsm_llnu(int64_t m, int64_t n, const uint32_t* L, int64_t ldl, uint32_t* B, int64_t ldb, cudaStream_t st) {
  if (m <= 0 || n <= 0) return 0;
  for (int64_t i0 = 0; i0 < m; i0 += TRSM_BLK) {
    const int64_t ib = (m - i0) < TRSM_BLK ? (m - i0) : TRSM_BLK;
    k_trsm_llnu_block<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(L, ldl, B, ldb, i0, ib, n);
    if (i0 + ib < m) {
      pg::Params P{m - i0 - ib, n, ib, L + (i0 + ib) * ldl + i0, ldl, B + i0 * ldb, ldb, B + (i0 + ib) * ldb, ldb,
                   1, 1, nullptr};
      const int rc = pb_launch_gemm(P, false, false, st);
      if (rc) return rc;
    }
  }
  return last_launch();
}

int pb_trsm_rltn(int64_t m, int64_t n, const uint32_t* L, int64_t ldl, uint32_t* B, int64_t ldb, const int32_t* stop,
                 cudaStream_t st) {
  if (m <= 0 || n <= 0) return 0;
  for (int64_t j0 = 0; j0 < n; j0 += TRSM_BLK) {
    const int64_t jb = (n - j0) < TRSM_BLK ? (n - j0) : TRSM_BLK;
    k_trsm_rltn_block<<<(unsigned)((m + 127) / 128), 128, 0, st>>>(L, ldl, B, ldb, j0, jb, m, stop);
    if (j0 + jb < n) {
      // B[:, j0+jb:] -= B[:, j0:j0+jb] * L[j0+jb:, j0:j0+jb]^T   (NT GEMM, K = jb)
      pg::Params P{m, n - j0 - jb, jb, B + j0, ldb, L + (j0 + jb) * ldl + j0, ldl, B + j0 + jb, ldb, 1, 1, stop};
      const int rc = pb_launch_gemm(P, true, false, st);
      if (rc) return rc;
    }
  }
  return last_launch();
}

int pb_potf2(int64_t b, uint32_t* A, int64_t lda, int32_t* info, int64_t row_base, cudaStream_t st) {
  k_potf2<<<1, 1024, 0, st>>>(A, lda, b, info, row_base);
  return last_launch();
}

int pb_vec_op(int op, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count, cudaStream_t st) {
  if (count <= 0) return 0;
  k_vec_op<<<grid_for(count, 256), 256, 0, st>>>(op, a, b, out, count);
  return last_launch();
}

int pb_from_f64(const double* x, uint32_t* out, int64_t count, cudaStream_t st) {
  if (count <= 0) return 0;
  k_from_f64<<<grid_for(count, 256), 256, 0, st>>>(x, out, count);
  return last_launch();
}

int pb_to_f64(const uint32_t* p, double* out, int64_t count, cudaStream_t st) {
  if (count <= 0) return 0;
  k_to_f64<<<grid_for(count, 256), 256, 0, st>>>(p, out, count);
  return last_launch();
}
