// lapack.cu -- the panel steps around the trailing update (SURVEY 8(a) rows
// a8-a11): LU panel (pivot search by signed compare of patterns, row swap,
// posit division, in-panel update), laswp, the two TRSM variants, potf2, and
// the elementwise / conversion kernels.  All on the device, stream-ordered.
//
// Order contract (reading Q6): every element receives its updates
// one product at a time in ascending k.  The panel and the diagonal-block
// Cholesky are recursive (LAPACK getrf2 / potrf2 traversal) and the TRSMs are
// blocked into a 32-wide in-block substitution plus a fast-path GEMM for the
// rows/columns beyond the block -- traversal changes only, so the bits equal
// the textbook loops.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
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

// ---- LU leaf (column by column, multi-CTA) ----------------------------------
// Workspace: key[0..w) (uint64, zeroed per leaf) and a CTA counter.
struct LeafWs {
  unsigned long long key[64];
  unsigned int done;
};

// key[0] <- max over rows 0..m-1 of column 0
__global__ void k_leaf_colmax(const uint32_t* A, int64_t lda, int64_t m, LeafWs* ws) {
  __shared__ unsigned long long red[32];
  unsigned long long best = 0ull;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = piv_key(A[r * lda], r);
    best = k > best ? k : best;
  }
  best = block_max(best, red);
  if (threadIdx.x == 0) atomicMax(&ws->key[0], best);
}

// Column j: p = the key's row; ipiv, info; swap rows j and p on the leaf's
// other columns (CTA 0); divide rows j+1..m-1 of column j by the pivot v.  The
// two words of column j that move (A[j][j], A[p][j]) are written by the CTA
// that finishes last, after every CTA has read v (threadfence counter).
__global__ void k_leaf_swap_div(uint32_t* A, int64_t lda, int64_t m, int64_t w, int64_t j, LeafWs* ws,
                                int32_t* ipiv, int32_t* info, int64_t row_base) {
  __shared__ bool last;
  const unsigned long long key = ws->key[j];
  const int64_t p = (int64_t)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull));
  const uint32_t v = A[p * lda + j];
  const uint32_t ajj = A[j * lda + j];
  if (v == 0u) {                                          // zero pivot: no swap, no division (Q11)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ipiv[j] = (int32_t)(row_base + p + 1);
      if (*info == 0) *info = (int32_t)(row_base + j + 1);
    }
    return;
  }
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) ipiv[j] = (int32_t)(row_base + p + 1);
    if (p != j) {
      for (int64_t c = threadIdx.x; c < w; c += blockDim.x) {
        if (c == j) continue;
        const uint32_t t = A[j * lda + c];
        A[j * lda + c] = A[p * lda + c];
        A[p * lda + c] = t;
      }
    }
  }
  for (int64_t r = j + 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x)
    if (r != p) A[r * lda + j] = div(A[r * lda + j], v);
  // last CTA: the moved words of column j
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&ws->done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    ws->done = 0u;
    if (p != j) {
      A[j * lda + j] = v;
      A[p * lda + j] = div(ajj, v);
    }
  }
}

// a_rq <- a_rq (-) a_rj (x) a_jq for j < r < m, j < q < w; the new column j+1
// feeds key[j+1] (rows j+1..m-1).
__global__ void k_leaf_update(uint32_t* A, int64_t lda, int64_t m, int64_t w, int64_t j, LeafWs* ws) {
  __shared__ unsigned long long red[32];
  const int64_t wq = w - j - 1;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long best = 0ull;
  if (e < (m - j - 1) * wq) {
    const int64_t r = j + 1 + e / wq, q = j + 1 + e % wq;
    const uint32_t nv = sub(A[r * lda + q], mul(A[r * lda + j], A[j * lda + q]));
    A[r * lda + q] = nv;
    if (q == j + 1) best = piv_key(nv, r);
  }
  best = block_max(best, red);
  if (threadIdx.x == 0 && best != 0ull) atomicMax(&ws->key[j + 1], best);
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

// ---- TRSM in-block kernels (32-wide, right-looking across a warp) -----------
// Unit lower, left: rows i0..i0+ib-1 of B (ib <= 32).  CTA = 32 warps = 32
// columns; the 32 x 32 tile goes through shared memory (coalesced); warp w
// owns column w with lane = row: step k broadcasts the final b_k by shuffle
// and rows i > k apply b_i <- b_i (-) l_ik (x) b_k (ascending k per element).
__global__ void __launch_bounds__(1024) k_trsm_llnu_blk(const uint32_t* L, int64_t ldl, uint32_t* B, int64_t ldb,
                                                        int64_t i0, int64_t ib, int64_t n) {
  __shared__ uint32_t sb[TB][TB + 1];
  __shared__ uint32_t sl[TB][TB + 1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * TB;
  if (wid < ib) {
    sl[wid][lane] = lane < wid ? L[(i0 + wid) * ldl + i0 + lane] : 0u;
    sb[wid][lane] = (c0 + lane < n) ? B[(i0 + wid) * ldb + c0 + lane] : 0u;
  }
  __syncthreads();
  uint32_t b = lane < ib ? sb[lane][wid] : 0u;
  for (int k = 0; k < ib - 1; k++) {
    const uint32_t bk = __shfl_sync(0xFFFFFFFFu, b, k);
    if (lane > k && lane < ib) b = sub(b, mul(sl[lane][k], bk));
  }
  if (lane < ib) sb[lane][wid] = b;
  __syncthreads();
  if (wid < ib && c0 + lane < n) B[(i0 + wid) * ldb + c0 + lane] = sb[wid][lane];
}

// Right, lower, transposed, non-unit: columns j0..j0+jb-1 of B (jb <= 32).
// Warp per row of B, lane = column (coalesced): step k finalises b_k <- b_k (/)
// l_kk, broadcasts it, and columns j > k apply b_j <- b_j (-) b_k (x) l_jk.
__global__ void __launch_bounds__(1024) k_trsm_rltn_blk(const uint32_t* L, int64_t ldl, uint32_t* B, int64_t ldb,
                                                        int64_t j0, int64_t jb, int64_t m, const int32_t* stop) {
  __shared__ uint32_t sl[TB][TB + 1];
  if (stop != nullptr && *stop != 0) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (wid < jb) sl[wid][lane] = lane <= wid ? L[(j0 + wid) * ldl + j0 + lane] : 0u;
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * 32 + wid;
  if (r >= m) return;
  uint32_t b = lane < jb ? B[r * ldb + j0 + lane] : 0u;
  for (int k = 0; k < jb; k++) {
    if (lane == k) b = div(b, sl[k][k]);
    const uint32_t bk = __shfl_sync(0xFFFFFFFFu, b, k);
    if (lane > k && lane < jb) b = sub(b, mul(bk, sl[lane][k]));
  }
  if (lane < jb) B[r * ldb + j0 + lane] = b;
}

// ---- Cholesky leaf: b <= 32 diagonal block in shared memory, one CTA ---------
// Textbook loop (reading Q9): for k: if signed(a_kk) <= 0 -> info = k+1, stop;
// a_kk <- sqrt(a_kk); a_ik <- a_ik (/) a_kk; a_ij <- a_ij (-) a_ik (x) a_jk.
__global__ void __launch_bounds__(1024) k_potf2_leaf(uint32_t* A, int64_t lda, int64_t b, int32_t* info,
                                                     int64_t row_base) {
  __shared__ uint32_t s[TB][TB + 1];
  __shared__ int fail;
  if (*info != 0) return;                                  // an earlier block failed: stop
  const int i = threadIdx.x >> 5, j = threadIdx.x & 31;    // row, column
  const bool in = i < b && j <= i;
  if (in) s[i][j] = A[i * lda + j];
  if (threadIdx.x == 0) fail = 0;
  __syncthreads();
  int k = 0;
  for (; k < b; k++) {
    if (threadIdx.x == 0) {
      const uint32_t v = s[k][k];
      if ((int32_t)v <= 0) {                               // zero, negative or NaR pivot
        fail = 1;
        *info = (int32_t)(row_base + k + 1);
      } else {
        s[k][k] = p32::sqrt(v);
      }
    }
    __syncthreads();
    if (fail) break;
    if (j == k && i > k && i < b) s[i][k] = div(s[i][k], s[k][k]);
    __syncthreads();
    if (in && j > k) s[i][j] = sub(s[i][j], mul(s[i][k], s[j][k]));
    __syncthreads();
  }
  if (in) A[i * lda + j] = s[i][j];
}

// ---- one-RHS solves for the accuracy report (Rgetrs / Rpotrs) -----
// One CTA; the right-hand side lives in shared memory.  Reference-BLAS trsv
// loop order (reading Q21): forward substitution in ascending k, back
// substitution in descending k, each step "x_k final, then update the rest".
constexpr int SOLVE_THREADS = 1024;

__global__ void __launch_bounds__(SOLVE_THREADS) k_getrs(int64_t n, const uint32_t* LU, int64_t lda,
                                                         const int32_t* ipiv, uint32_t* b) {
  extern __shared__ uint32_t sx[];
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) sx[i] = b[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int64_t k = 0; k < n; k++) {                       // apply P
      const int64_t p = (int64_t)ipiv[k] - 1;
      if (p != k) { const uint32_t t = sx[k]; sx[k] = sx[p]; sx[p] = t; }
    }
  }
  __syncthreads();
  for (int64_t k = 0; k < n; k++) {                         // L y = P b (unit lower)
    const uint32_t yk = sx[k];
    for (int64_t i = k + 1 + threadIdx.x; i < n; i += blockDim.x) sx[i] = sub(sx[i], mul(LU[i * lda + k], yk));
    __syncthreads();
  }
  for (int64_t k = n - 1; k >= 0; k--) {                    // U x = y
    if (threadIdx.x == 0) sx[k] = div(sx[k], LU[k * lda + k]);
    __syncthreads();
    const uint32_t xk = sx[k];
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x) sx[i] = sub(sx[i], mul(LU[i * lda + k], xk));
    __syncthreads();
  }
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) b[i] = sx[i];
}

__global__ void __launch_bounds__(SOLVE_THREADS) k_potrs(int64_t n, const uint32_t* L, int64_t lda, uint32_t* b) {
  extern __shared__ uint32_t sx[];
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) sx[i] = b[i];
  __syncthreads();
  for (int64_t k = 0; k < n; k++) {                         // L y = b
    if (threadIdx.x == 0) sx[k] = div(sx[k], L[k * lda + k]);
    __syncthreads();
    const uint32_t yk = sx[k];
    for (int64_t i = k + 1 + threadIdx.x; i < n; i += blockDim.x) sx[i] = sub(sx[i], mul(L[i * lda + k], yk));
    __syncthreads();
  }
  for (int64_t k = n - 1; k >= 0; k--) {                    // L^T x = y
    if (threadIdx.x == 0) sx[k] = div(sx[k], L[k * lda + k]);
    __syncthreads();
    const uint32_t xk = sx[k];
    for (int64_t i = threadIdx.x; i < k; i += blockDim.x) sx[i] = sub(sx[i], mul(L[k * lda + i], xk));
    __syncthreads();
  }
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) b[i] = sx[i];
}

// ---- elementwise / conversion ------------------------------------------------
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

inline unsigned rows_grid(int64_t rows, int threads) {
  int64_t g = (rows + threads - 1) / threads;
  if (g > 148 * 4) g = 148 * 4;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace pl

using namespace pl;

static int last_launch() {
  return cudaPeekAtLastError() == cudaSuccess ? 0 : POSIT_ECUDA;
}

size_t pb_panel_ws_bytes() { return sizeof(LeafWs); }

static int64_t panel_leaf() {
  static int64_t leaf = -1;
  if (leaf < 0) {
    const char* e = getenv("POSIT_PANEL_LEAF");
    leaf = e ? atoll(e) : 32;
    if (leaf < 1) leaf = 1;
    if (leaf > 64) leaf = 64;
  }
  return leaf;
}

// Unblocked leaf (w <= 64 columns): per column one swap/divide launch and one
// update launch that also searches the next column's pivot.
static int getrf_leaf(int64_t m, int64_t w, uint32_t* A, int64_t lda, int32_t* ipiv, int32_t* info, int64_t row_base,
                      LeafWs* ws, cudaStream_t st) {
  if (cudaMemsetAsync(ws, 0, sizeof(LeafWs), st) != cudaSuccess) return POSIT_ECUDA;
  pb_count_launch();
  k_leaf_colmax<<<rows_grid(m, 256), 256, 0, st>>>(A, lda, m, ws);
  const int64_t jmax = m < w ? m : w;
  for (int64_t j = 0; j < jmax; j++) {
    pb_count_launch();
    k_leaf_swap_div<<<rows_grid(m - j - 1, 256), 256, 0, st>>>(A, lda, m, w, j, ws, ipiv, info, row_base);
    const int64_t cnt = (m - j - 1) * (w - j - 1);
    if (cnt > 0) {
      pb_count_launch();
      k_leaf_update<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(A, lda, m, w, j, ws);
    }
  }
  return last_launch();
}

// Recursive panel LU (the traversal of LAPACK getrf2): factor the left half,
// apply its swaps to the right half, U12 by TRSM, the right half's update by
// the fast GEMM, factor the right half, apply its swaps to the left half.
// Every element still receives its products one at a time in ascending k
// (reading Q6), so the bits equal the column-by-column loop.
int pb_getrf_panel(int64_t m, int64_t b, uint32_t* A, int64_t lda, int32_t* ipiv, int32_t* info, int64_t row_base,
                   void* ws, cudaStream_t st) {
  const int64_t w = m < b ? m : b;
  const int64_t leaf = panel_leaf();
  if (w <= leaf) return getrf_leaf(m, b, A, lda, ipiv, info, row_base, static_cast<LeafWs*>(ws), st);
  int64_t w1 = ((w / 2 + leaf - 1) / leaf) * leaf;
  if (w1 >= w) w1 = w - leaf;
  int rc;
  if ((rc = pb_getrf_panel(m, w1, A, lda, ipiv, info, row_base, ws, st))) return rc;
  if ((rc = pb_laswp(b - w1, A + w1, lda, 0, w1, ipiv, row_base, st))) return rc;
  if ((rc = pb_trsm_llnu(w1, b - w1, A, lda, A + w1, lda, st))) return rc;
  if (m > w1) {
    pg::Params P{m - w1, b - w1, w1, A + w1 * lda, lda, A + w1, lda, A + w1 * lda + w1, lda, 1, 1, nullptr};
    if ((rc = pb_launch_gemm(P, false, false, st))) return rc;
    if ((rc = pb_getrf_panel(m - w1, b - w1, A + w1 * lda + w1, lda, ipiv + w1, info, row_base + w1, ws, st)))
      return rc;
    if ((rc = pb_laswp(w1, A + w1 * lda, lda, 0, w - w1, ipiv + w1, row_base + w1, st))) return rc;
  }
  return last_launch();
}

int pb_laswp(int64_t ncols, uint32_t* A, int64_t lda, int64_t k1, int64_t k2, const int32_t* ipiv, int64_t ipiv_base,
             cudaStream_t st) {
  if (ncols <= 0 || k2 <= k1) return 0;
  pb_count_launch();
  k_laswp<<<(unsigned)((ncols + 255) / 256), 256, 0, st>>>(A, lda, ncols, k1, k2, ipiv, ipiv_base);
  return last_launch();
}

int pb_trsm_llnu(int64_t m, int64_t n, const uint32_t* L, int64_t ldl, uint32_t* B, int64_t ldb, cudaStream_t st) {
  if (m <= 0 || n <= 0) return 0;
  for (int64_t i0 = 0; i0 < m; i0 += TB) {
    const int64_t ib = (m - i0) < TB ? (m - i0) : TB;
    if (ib > 1) {
      pb_count_launch();
      k_trsm_llnu_blk<<<(unsigned)((n + TB - 1) / TB), 1024, 0, st>>>(L, ldl, B, ldb, i0, ib, n);
    }
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
  for (int64_t j0 = 0; j0 < n; j0 += TB) {
    const int64_t jb = (n - j0) < TB ? (n - j0) : TB;
    pb_count_launch();
    k_trsm_rltn_blk<<<(unsigned)((m + 31) / 32), 1024, 0, st>>>(L, ldl, B, ldb, j0, jb, m, stop);
    if (j0 + jb < n) {
      // B[:, j0+jb:] -= B[:, j0:j0+jb] * L[j0+jb:, j0:j0+jb]^T   (NT GEMM, K = jb)
      pg::Params P{m, n - j0 - jb, jb, B + j0, ldb, L + (j0 + jb) * ldl + j0, ldl, B + j0 + jb, ldb, 1, 1, stop};
      const int rc = pb_launch_gemm(P, true, false, st);
      if (rc) return rc;
    }
  }
  return last_launch();
}

// Recursive diagonal-block Cholesky (the traversal of LAPACK potrf2): leaf
// blocks of <= 32 in shared memory, TRSM + SYRK between them.  Every stage
// is a no-op once *info != 0.
int pb_potf2(int64_t b, uint32_t* A, int64_t lda, int32_t* info, int64_t row_base, cudaStream_t st) {
  if (b <= 0) return 0;
  if (b <= TB) {
    pb_count_launch();
    k_potf2_leaf<<<1, 1024, 0, st>>>(A, lda, b, info, row_base);
    return last_launch();
  }
  int64_t b1 = ((b / 2 + TB - 1) / TB) * TB;
  if (b1 >= b) b1 = b - TB;
  int rc;
  if ((rc = pb_potf2(b1, A, lda, info, row_base, st))) return rc;
  if ((rc = pb_trsm_rltn(b - b1, b1, A, lda, A + b1 * lda, lda, info, st))) return rc;
  pg::Params P{b - b1, b - b1, b1, A + b1 * lda, lda, A + b1 * lda, lda, A + b1 * lda + b1, lda, 1, 1, info};
  if ((rc = pb_launch_gemm(P, true, true, st))) return rc;
  return pb_potf2(b - b1, A + b1 * lda + b1, lda, info, row_base + b1, st);
}

int pb_solve(bool chol, int64_t n, const uint32_t* A, int64_t lda, const int32_t* ipiv, uint32_t* b, cudaStream_t st) {
  if (n <= 0) return 0;
  const size_t smem = (size_t)n * sizeof(uint32_t);
  if (smem > 200 * 1024) return POSIT_ENOTSUP;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_getrs, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_potrs, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  pb_count_launch();
  if (chol) k_potrs<<<1, SOLVE_THREADS, smem, st>>>(n, A, lda, b);
  else k_getrs<<<1, SOLVE_THREADS, smem, st>>>(n, A, lda, ipiv, b);
  return last_launch();
}

int pb_vec_op(int op, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count, cudaStream_t st) {
  if (count <= 0) return 0;
  pb_count_launch();
  k_vec_op<<<grid_for(count, 256), 256, 0, st>>>(op, a, b, out, count);
  return last_launch();
}

int pb_from_f64(const double* x, uint32_t* out, int64_t count, cudaStream_t st) {
  if (count <= 0) return 0;
  pb_count_launch();
  k_from_f64<<<grid_for(count, 256), 256, 0, st>>>(x, out, count);
  return last_launch();
}

int pb_to_f64(const uint32_t* p, double* out, int64_t count, cudaStream_t st) {
  if (count <= 0) return 0;
  pb_count_launch();
  k_to_f64<<<grid_for(count, 256), 256, 0, st>>>(p, out, count);
  return last_launch();
}
