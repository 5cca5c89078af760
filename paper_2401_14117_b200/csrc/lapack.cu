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

// ---- LU leaf (column by column, multi-CTA) ----------------------------------
// Workspace: key[0..w) (uint64, zeroed per leaf) and a CTA counter.
constexpr int LEAF_MAXCTA = 160;
constexpr int TAIL_WMAX = 1024;   // widest leaf: the fused LU of a factorisation's last columns
struct LeafWs {
  unsigned long long key[TAIL_WMAX];
  unsigned int done;
  uint32_t rowp[64];       // cooperative leaf: the pivot row and the current row, published
  uint32_t rowj[64];
  // one-sync cooperative leaf, by column parity: each CTA's best pivot
  // candidate row for the next column, and the row at the next diagonal position
  uint32_t cand[2][LEAF_MAXCTA][64];
  uint32_t jrow[2][64];
  uint32_t tcand[2][LEAF_MAXCTA][TAIL_WMAX];   // the same for leaves up to TAIL_WMAX wide
  uint32_t tjrow[2][TAIL_WMAX];
};
constexpr size_t LEAF_WS_ZERO = offsetof(LeafWs, cand);   // the part zeroed per leaf

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

// ---- LU leaf as ONE cooperative launch ---------------------------------------
// The leaf (m rows x w <= 64 columns) is split into contiguous row ranges, one
// per CTA, kept in shared memory for all w steps.  Per column j: every CTA
// folds its pivot candidates into key[j] (64-bit atomicMax), grid sync; the
// CTAs owning rows j and p publish them, grid sync; then each CTA swaps,
// divides and updates its own rows (textbook order, Q8/Q10/Q11) and folds the
// next column's candidates.  Bit-identical to the per-column launches.
namespace cg = cooperative_groups;
constexpr int COOP_THREADS = 256;

__global__ void __launch_bounds__(1024) k_leaf_coop(uint32_t* A, int64_t lda, int64_t m, int64_t w,
                                                            int64_t rows_per_cta, int32_t* ipiv, int32_t* info,
                                                            int64_t row_base, LeafWs* ws) {
  extern __shared__ uint32_t tile[];                  // [rows_per_cta][w]
  __shared__ unsigned long long red[32];
  __shared__ uint4 urow[64];                          // the pivot row as decoded B operands {M, E, sg, fast}
  __shared__ uint32_t urowp[64];                      // ... and as patterns
  __shared__ uint4 tp[pg::TSIZE], tx[pg::TSIZE];      // the MAC's constant tables
  const int NT = blockDim.x;
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x;
  pg::fill_tables(tp, tx, tid, NT);
  pg::MacConst K;
  K.one = 1u;
  K.sixteen = 16u;
  K.tp0 = (uint32_t)__cvta_generic_to_shared(tp + pg::TBIAS);
  K.tx0 = (uint32_t)__cvta_generic_to_shared(tx + pg::TBIAS) - 30u * 16u;
  const int64_t rb = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t re = (rb + rows_per_cta) < m ? (rb + rows_per_cta) : m;
  const int nr = re > rb ? (int)(re - rb) : 0;
  const int W = (int)w;
  for (int e = tid; e < nr * W; e += NT) tile[e] = A[(rb + e / W) * lda + e % W];
  __syncthreads();
  // candidates of column 0
  {
    unsigned long long best = 0ull;
    for (int i = tid; i < nr; i += NT) {
      const unsigned long long k = piv_key(tile[i * W], rb + i);
      best = k > best ? k : best;
    }
    best = block_max(best, red);
    if (tid == 0 && best != 0ull) atomicMax(&ws->key[0], best);
  }
  const int64_t jmax = m < w ? m : w;
  for (int64_t j = 0; j < jmax; j++) {
    grid.sync();
    const unsigned long long key = __ldcg(&ws->key[j]);
    const int64_t p = (int64_t)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull));
    // publish rows p and j
    if (p >= rb && p < re) for (int c = tid; c < W; c += NT) ws->rowp[c] = tile[(p - rb) * W + c];
    if (j >= rb && j < re) for (int c = tid; c < W; c += NT) ws->rowj[c] = tile[(j - rb) * W + c];
    grid.sync();
    const uint32_t v = __ldcg(ws->rowp + j);
    if (blockIdx.x == 0 && tid == 0) {
      ipiv[j] = (int32_t)(row_base + p + 1);
      if (v == 0u && *info == 0) *info = (int32_t)(row_base + j + 1);
    }
    if (v != 0u && p != j) {                          // swap rows j and p (whole leaf width)
      if (j >= rb && j < re) for (int c = tid; c < W; c += NT) tile[(j - rb) * W + c] = __ldcg(ws->rowp + c);
      if (p >= rb && p < re) for (int c = tid; c < W; c += NT) tile[(p - rb) * W + c] = __ldcg(ws->rowj + c);
    }
    __syncthreads();
    // the row now at position j (the pivot row), decoded once as B operands
    const uint32_t* rowj = (v != 0u && p != j) ? ws->rowp : ws->rowj;
    for (int c = tid; c < W; c += NT) {
      LaneVal t;
      const uint32_t x = __ldcg(rowj + c);                // L2 (written by another CTA before the grid sync)
      lv_load(t, x);
      urow[c] = make_uint4(t.a.M, (uint32_t)t.a.E, (uint32_t)t.a.sg, lv_operand(t) ? 1u : 0u);
      urowp[c] = x;
    }
    // divide column j below the diagonal (Q8; skipped for a zero pivot, Q11):
    // decoded division by the shared divisor, generic outside its range
    const int64_t i0 = (j + 1 > rb ? j + 1 : rb) - rb;
    if (v != 0u) {
      pg::Acc dv;
      const bool dok = pg::acc_decode(v, dv) && v != 0x80000000u && dv.E <= 37 && dv.E >= -37;
      const double rcp = dok ? __drcp_rn((double)dv.M) * 4294967296.0 : 0.0;
      for (int64_t i = i0 + tid; i < nr; i += NT) {
        const uint32_t x = tile[i * W + j];
        LaneVal t;
        lv_load(t, x);
        bool done = false;
        if (dok && t.dec) done = pg::acc_div(t.a, dv.M, dv.E, dv.sg, rcp, K);
        tile[i * W + j] = done ? pg::acc_encode(t.a) : div(x, v);
      }
    }
    __syncthreads();
    // update columns j+1..w-1 of rows j+1..m-1 with row j (= the pivot row), then fold column j+1
    const int wq = W - (int)j - 1;
    unsigned long long best = 0ull;
    if (wq > 0) {
      const uint32_t cnt = nr > i0 ? (uint32_t)(nr - i0) * (uint32_t)wq : 0u;      // 32-bit index math (rows per CTA are few)
      for (uint32_t e = tid; e < cnt; e += NT) {
        const uint32_t ii = e / (uint32_t)wq;
        const int i = (int)i0 + (int)ii;
        const int q = (int)j + 1 + (int)(e - ii * (uint32_t)wq);
        // decoded-domain c (-) l (x) u (generic outside the MAC's exact range)
        const uint32_t lp = tile[i * W + j];
        uint4 ad;
        const bool af = fast_a(lp, ad);
        const uint4 ub = urow[q];
        LaneVal c;
        lv_load(c, tile[i * W + q]);
        lv_fms_t(c, lp, af, ad, ub.x, (int32_t)ub.y, (int32_t)ub.z, ub.w != 0u, urowp[q], K);
        const uint32_t nv = lv_pattern(c);
        tile[i * W + q] = nv;
        if (q == j + 1) {
          const unsigned long long k = piv_key(nv, rb + i);
          best = k > best ? k : best;
        }
      }
      best = block_max(best, red);
      if (tid == 0 && best != 0ull) atomicMax(&ws->key[j + 1], best);
    }
    __syncthreads();
  }
  for (int e = tid; e < nr * W; e += NT) A[(rb + e / W) * lda + e % W] = tile[e];
}

// The same leaf with ONE grid sync per column.  Instead of publishing rows j
// and p after the pivot is known (a second grid sync), every CTA publishes,
// before the sync, its own best candidate row for the next column and (its
// owner) the row at the next diagonal position, double-buffered by column
// parity; after the sync the winner's candidate row IS the pivot row.  The
// arithmetic per element is the decoded-domain update of k_leaf_coop, in the
// same textbook order.
// cand: [2][LEAF_MAXCTA][WMAX] candidate rows, jrow: [2][WMAX] diagonal rows
template <int WMAX>
__device__ __forceinline__ void leaf_publish(const uint32_t* tile, int W, int64_t rb, int nr, int64_t jn,
                                             unsigned long long best, uint32_t* cand, uint32_t* jrow, int par,
                                             int tid, int NT) {
  if (best != 0ull) {
    const int64_t r = (int64_t)(0xFFFFFFFFu - (uint32_t)(best & 0xFFFFFFFFull));
    const int li = (int)(r - rb);
    uint32_t* dst = cand + ((size_t)par * LEAF_MAXCTA + blockIdx.x) * WMAX;
    for (int c = tid; c < W; c += NT) dst[c] = tile[li * W + c];
  }
  if (jn >= rb && jn < rb + nr)
    for (int c = tid; c < W; c += NT) jrow[par * WMAX + c] = tile[(int)(jn - rb) * W + c];
}

template <int WMAX>
__global__ void __launch_bounds__(1024) k_leaf_coop1(uint32_t* A, int64_t lda, int64_t m, int64_t w,
                                                     int64_t rows_per_cta, int32_t* ipiv, int32_t* info,
                                                     int64_t row_base, LeafWs* ws, uint32_t* cand, uint32_t* jrow) {
  extern __shared__ uint32_t tile[];                  // [rows_per_cta][w]
  __shared__ unsigned long long red[32];
  __shared__ unsigned long long cbest;                // this CTA's best candidate key (next column)
  __shared__ uint32_t srow[2 * WMAX];                 // the published rows p and j of the current column
  __shared__ uint4 urow[WMAX];                        // the pivot row as decoded B operands {M, E, sg, fast}
  __shared__ uint32_t urowp[WMAX];                    // ... and as patterns
  __shared__ uint4 tp[pg::TSIZE], tx[pg::TSIZE];      // the MAC's constant tables
  const int NT = blockDim.x;
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x;
  pg::fill_tables(tp, tx, tid, NT);
  pg::MacConst K;
  K.one = 1u;
  K.sixteen = 16u;
  K.tp0 = (uint32_t)__cvta_generic_to_shared(tp + pg::TBIAS);
  K.tx0 = (uint32_t)__cvta_generic_to_shared(tx + pg::TBIAS) - 30u * 16u;
  const int64_t rb = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t re = (rb + rows_per_cta) < m ? (rb + rows_per_cta) : m;
  const int nr = re > rb ? (int)(re - rb) : 0;
  const int W = (int)w;
  for (int e = tid; e < nr * W; e += NT) tile[e] = A[(rb + e / W) * lda + e % W];
  __syncthreads();
  {
    unsigned long long best = 0ull;
    for (int i = tid; i < nr; i += NT) {
      const unsigned long long k = piv_key(tile[i * W], rb + i);
      best = k > best ? k : best;
    }
    best = block_max(best, red);
    if (tid == 0) {
      cbest = best;
      if (best != 0ull) atomicMax(&ws->key[0], best);
    }
    __syncthreads();
    leaf_publish<WMAX>(tile, W, rb, nr, 0, cbest, cand, jrow, 0, tid, NT);
  }
  const int64_t jmax = m < w ? m : w;
  for (int64_t j = 0; j < jmax; j++) {
    const int par = (int)(j & 1);
    grid.sync();
    const unsigned long long key = __ldcg(&ws->key[j]);
    const int64_t p = (int64_t)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull));
    // rows p and j in one round trip (threads 0..W-1: row p; W..2W-1: row j)
    {
      const uint32_t* cp = cand + ((size_t)par * LEAF_MAXCTA + (size_t)(p / rows_per_cta)) * WMAX;
      const uint32_t* jp = jrow + par * WMAX;
      for (int t = tid; t < 2 * W; t += NT) srow[t] = t < W ? __ldcg(cp + t) : __ldcg(jp + (t - W));
    }
    __syncthreads();
    const uint32_t v = srow[j];
    if (blockIdx.x == 0 && tid == 0) {
      ipiv[j] = (int32_t)(row_base + p + 1);
      if (v == 0u && *info == 0) *info = (int32_t)(row_base + j + 1);
    }
    const bool swp = v != 0u && p != j;
    if (swp) {                                        // swap rows j and p (whole leaf width)
      if (j >= rb && j < re) for (int c = tid; c < W; c += NT) tile[(j - rb) * W + c] = srow[c];
      if (p >= rb && p < re) for (int c = tid; c < W; c += NT) tile[(p - rb) * W + c] = srow[W + c];
    }
    const int usrc = swp ? 0 : W;                     // the row now at position j
    for (int c = tid; c < W; c += NT) {
      LaneVal t;
      const uint32_t x = srow[usrc + c];
      lv_load(t, x);
      urow[c] = make_uint4(t.a.M, (uint32_t)t.a.E, (uint32_t)t.a.sg, lv_operand(t) ? 1u : 0u);
      urowp[c] = x;
    }
    __syncthreads();
    const int i0 = (int)((j + 1 > rb ? j + 1 : rb) - rb);
    if (v != 0u) {                                    // Q8 (one division each); skipped for a zero pivot (Q11)
      pg::Acc dv;
      const bool dok = pg::acc_decode(v, dv) && v != 0x80000000u && dv.E <= 37 && dv.E >= -37;
      const double rcp = dok ? __drcp_rn((double)dv.M) * 4294967296.0 : 0.0;
      for (int i = i0 + tid; i < nr; i += NT) {
        const uint32_t x = tile[i * W + (int)j];
        LaneVal t;
        lv_load(t, x);
        bool done = false;
        if (dok && t.dec) done = pg::acc_div(t.a, dv.M, dv.E, dv.sg, rcp, K);
        tile[i * W + (int)j] = done ? pg::acc_encode(t.a) : div(x, v);
      }
    }
    __syncthreads();
    const int wq = W - (int)j - 1;
    if (wq > 0) {
      unsigned long long best = 0ull;
      const uint32_t cnt = nr > i0 ? (uint32_t)(nr - i0) * (uint32_t)wq : 0u;
      for (uint32_t e = tid; e < cnt; e += NT) {
        const uint32_t ii = e / (uint32_t)wq;
        const int i = i0 + (int)ii;
        const int q = (int)j + 1 + (int)(e - ii * (uint32_t)wq);
        const uint32_t lp = tile[i * W + (int)j];
        uint4 ad;
        const bool af = fast_a(lp, ad);
        const uint4 ub = urow[q];
        LaneVal c;
        lv_load(c, tile[i * W + q]);
        lv_fms_t(c, lp, af, ad, ub.x, (int32_t)ub.y, (int32_t)ub.z, ub.w != 0u, urowp[q], K);
        const uint32_t nv = lv_pattern(c);
        tile[i * W + q] = nv;
        if (q == (int)j + 1) {
          const unsigned long long k = piv_key(nv, rb + i);
          best = k > best ? k : best;
        }
      }
      best = block_max(best, red);
      if (tid == 0) {
        cbest = best;
        if (best != 0ull) atomicMax(&ws->key[j + 1], best);
      }
      __syncthreads();
      if (j + 1 < jmax) leaf_publish<WMAX>(tile, W, rb, nr, j + 1, cbest, cand, jrow, par ^ 1, tid, NT);
    }
    __syncthreads();
  }
  for (int e = tid; e < nr * W; e += NT) A[(rb + e / W) * lda + e % W] = tile[e];
}

// Pivot key over a strided column whose rows carry global indices (the 2D
// block-cyclic panel, where a rank's rows are not contiguous): max over rows
// with grow[i] >= row_min of  ((abs(a) + 2^31) << 31) | (2^31 - 1 - grow[i]),
// i.e. larger abs first, then the smaller global row (reading Q10), as a
// non-negative int64 suitable for a MAX all-reduce.  0 if no row qualifies.
__global__ void __launch_bounds__(1024) k_iamax_key(int64_t m, const uint32_t* col, int64_t stride,
                                                    const int32_t* grow, int64_t row_min, long long* out) {
  __shared__ unsigned long long red[32];
  unsigned long long best = 0ull;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const int64_t g = grow[i];
    if (g < row_min) continue;
    const uint64_t a = (uint64_t)((int64_t)abs_key(col[i * stride]) + 2147483648ll);
    const unsigned long long k = (a << 31) | (uint64_t)(2147483647ll - g);
    best = k > best ? k : best;
  }
  best = block_max(best, red);
  if (threadIdx.x == 0) *out = (long long)best;
}

// laswp: rows k1..k2-1 swapped with ipiv[k]-1-base, in order, on columns
// [0, ncols).  One CTA per 32 columns.  Instead of walking the swaps through
// global memory (a dependent load/store chain per swap), the CTA gathers every
// row the swaps touch into shared memory (the k2-k1 rows themselves plus each
// distinct pivot row), applies the swaps there in order, and scatters the rows
// back: the global traffic is independent loads and stores.
constexpr int SWP_MAX = 256;   // swaps per pass (longer ranges run in passes)
constexpr int SWP_COLS = 32;
constexpr int SWP_HASH_BITS = 10, SWP_HASH = 1 << SWP_HASH_BITS;   // >= 2 x SWP_MAX entries

__global__ void __launch_bounds__(256) k_laswp(uint32_t* A, int64_t lda, int64_t ncols, int64_t k1, int64_t k2,
                                               const int32_t* ipiv, int64_t base) {
  extern __shared__ uint32_t swp_smem[];
  uint32_t (*val)[SWP_COLS] = reinterpret_cast<uint32_t (*)[SWP_COLS]>(swp_smem);   // [2 * SWP_MAX][SWP_COLS]
  __shared__ int32_t tgt[SWP_MAX];      // pivot row of swap s (relative row index)
  __shared__ int16_t slot[SWP_MAX];     // slot holding that row
  __shared__ int16_t perm[2 * SWP_MAX]; // after the swaps, slot q holds the row gathered into slot perm[q]
  __shared__ int hkey[SWP_HASH];        // pivot row -> first swap index using it (outside the block)
  __shared__ int hval[SWP_HASH];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * SWP_COLS + lane;
  for (int64_t s0 = k1; s0 < k2; s0 += SWP_MAX) {
    const int ns = (int)((k2 - s0) < SWP_MAX ? (k2 - s0) : SWP_MAX);
    for (int s = threadIdx.x; s < ns; s += blockDim.x) tgt[s] = ipiv[s0 + s] - 1 - (int32_t)base;
    __syncthreads();
    // slot of each pivot row: inside the block -> its own row slot; outside ->
    // the slot of its first occurrence (ns + index), so repeated pivots share it.
    // First occurrences by a shared-memory hash (open addressing, atomicMin).
    for (int h = threadIdx.x; h < SWP_HASH; h += blockDim.x) { hkey[h] = -1; hval[h] = 0x7FFFFFFF; }
    __syncthreads();
    for (int s = threadIdx.x; s < ns; s += blockDim.x) {
      const int32_t p = tgt[s];
      if (p >= s0 && p < s0 + ns) continue;
      uint32_t h = ((uint32_t)p * 2654435761u) >> (32 - SWP_HASH_BITS);
      while (true) {
        const int old = atomicCAS(&hkey[h], -1, p);
        if (old == -1 || old == p) { atomicMin(&hval[h], s); break; }
        h = (h + 1) & (SWP_HASH - 1);
      }
    }
    __syncthreads();
    for (int s = threadIdx.x; s < ns; s += blockDim.x) {
      const int32_t p = tgt[s];
      int sl;
      if (p >= s0 && p < s0 + ns) {
        sl = (int)(p - s0);
      } else {
        uint32_t h = ((uint32_t)p * 2654435761u) >> (32 - SWP_HASH_BITS);
        while (hkey[h] != p) h = (h + 1) & (SWP_HASH - 1);
        sl = ns + hval[h];
      }
      slot[s] = (int16_t)sl;
    }
    __syncthreads();
    // gather (warps 1..): each warp has up to 8 row segments in flight; meanwhile
    // warp 0 composes the swaps on slot indices: slot q ends up holding the row
    // gathered into slot perm[q] (no data moves in the sequential part)
    if (wid == 0) {
      for (int q = lane; q < 2 * ns; q += 32) perm[q] = (int16_t)q;
      __syncwarp();
      if (lane == 0) {
        for (int s = 0; s < ns; s++) {
          const int q = slot[s];
          if (q != s) {
            const int16_t t = perm[s];
            perm[s] = perm[q];
            perm[q] = t;
          }
        }
      }
    } else {
      const int nwg = nw - 1, w = wid - 1;
      for (int sb = w * 16; sb < ns; sb += nwg * 16) {
        uint32_t v0[16], v1[16];
#pragma unroll
        for (int u = 0; u < 16; u++) {
          const int s = sb + u;
          const bool in = s < ns && c < ncols;
          v0[u] = in ? A[(s0 + s) * lda + c] : 0u;
          v1[u] = (in && slot[s] == ns + s) ? A[(int64_t)tgt[s] * lda + c] : 0u;
        }
#pragma unroll
        for (int u = 0; u < 16; u++) {
          const int s = sb + u;
          if (s < ns) {
            val[s][lane] = v0[u];
            if (slot[s] == ns + s) val[ns + s][lane] = v1[u];
          }
        }
      }
    }
    __syncthreads();
    // scatter: position slot q receives slot perm[q]
    for (int s = wid; s < ns; s += nw) {
      if (c < ncols) {
        A[(s0 + s) * lda + c] = val[perm[s]][lane];
        if (slot[s] == ns + s) A[(int64_t)tgt[s] * lda + c] = val[perm[ns + s]][lane];
      }
    }
    __syncthreads();
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
  LaneVal b;
  lv_load(b, lane < ib ? sb[lane][wid] : 0u);
  for (int k = 0; k < ib - 1; k++) {
    const bool bf = lv_operand(b);
    const uint32_t bM = __shfl_sync(0xFFFFFFFFu, b.a.M, k);
    const int32_t bE = __shfl_sync(0xFFFFFFFFu, b.a.E, k);
    const int32_t bs = __shfl_sync(0xFFFFFFFFu, b.a.sg, k);
    const bool bfk = __shfl_sync(0xFFFFFFFFu, (int)bf, k) != 0;
    const uint32_t bpk = __shfl_sync(0xFFFFFFFFu, lane == k ? lv_pattern(b) : 0u, k);   // for the generic path
    if (lane > k && lane < ib) {
      const uint32_t ap = sl[lane][k];
      uint4 ad;
      const bool af = fast_a(ap, ad);
      lv_fms(b, ap, af, ad, bM, bE, bs, bfk, bpk);
    }
  }
  if (lane < ib) sb[lane][wid] = lv_pattern(b);
  __syncthreads();
  if (wid < ib && c0 + lane < n) B[(i0 + wid) * ldb + c0 + lane] = sb[wid][lane];
}

// The same, NW columns (warps) per CTA and L's block staged decoded: for
// narrow right-hand sides (the panel-internal TRSMs) the 32-column CTA puts all
// the (issue-bound) steps on one SM; 8-column CTAs spread them.
template <int NW>
__global__ void __launch_bounds__(NW * 32) k_trsm_llnu_blkw(const uint32_t* L, int64_t ldl, uint32_t* B, int64_t ldb,
                                                           int64_t i0, int64_t ib, int64_t n) {
  __shared__ uint32_t sb[TB][NW + 1];
  __shared__ uint4 sld[TB][TB];           // L[i0 + r][i0 + c] decoded A-format {M, E, sigma (0: slow), pattern}
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t c0 = (int64_t)blockIdx.x * NW;
  for (int r = wid; r < ib; r += NW) {
    const uint32_t x = lane < r ? L[(i0 + r) * ldl + i0 + lane] : 0u;
    uint4 d;
    const bool f = fast_a(x, d);
    sld[r][lane] = make_uint4(d.x, d.y, f ? d.z : 0u, x);
    if (lane < NW) sb[r][lane] = (c0 + lane < n) ? B[(i0 + r) * ldb + c0 + lane] : 0u;
  }
  __syncthreads();
  LaneVal b;
  lv_load(b, lane < ib ? sb[lane][wid] : 0u);
  for (int k = 0; k < ib - 1; k++) {
    const bool bf = lv_operand(b);
    const uint32_t bM = __shfl_sync(0xFFFFFFFFu, b.a.M, k);
    const int32_t bE = __shfl_sync(0xFFFFFFFFu, b.a.E, k);
    const int32_t bs = __shfl_sync(0xFFFFFFFFu, b.a.sg, k);
    const bool bfk = __shfl_sync(0xFFFFFFFFu, (int)bf, k) != 0;
    const uint32_t bpk = __shfl_sync(0xFFFFFFFFu, lane == k ? lv_pattern(b) : 0u, k);   // for the generic path
    if (lane > k && lane < ib) {
      const uint4 ad = sld[lane][k];
      lv_fms(b, ad.w, ad.z != 0u, ad, bM, bE, bs, bfk, bpk);
    }
  }
  if (lane < ib) sb[lane][wid] = lv_pattern(b);
  __syncthreads();
  for (int r = wid; r < ib; r += NW)
    if (lane < NW && c0 + lane < n) B[(i0 + r) * ldb + c0 + lane] = sb[r][lane];
}

// The same in-block solve with one thread per column of B (default).  Columns
// are independent, so a thread runs its column's substitution alone: rows in
// groups of LC_G, each group first taking the updates from every earlier
// (final) row of the block in ascending k -- LC_G independent MAC chains -- and
// then the in-group triangle, still ascending k per element (Q6).  No shuffles
// and no idle lanes.  The MACs run branch-free in k-slabs of <= 16 (the
// GEMM's exactness argument, csrc/gemm.cuh: operands |E| <= 37, accumulators
// |E| <= 75 at the slab start); a slab whose operands or accumulators fall
// outside runs the generic pattern path instead.  L's 32 x 32 block is staged
// decoded (read as a broadcast); a column's final rows stay in the thread's
// own shared slots.
constexpr int LC_T = 32, LC_SLAB = 16;

__device__ __forceinline__ void lc_renorm(LaneVal& v) {
  if (v.dec && !(v.a.E <= 75 && v.a.E >= -75) && v.a.E > pg::E_ZERO_LIMIT) {
    v.pat = pg::acc_encode(v.a);
    v.dec = false;
  }
}

template <int LC_G>
__global__ void __launch_bounds__(LC_T) k_trsm_llnu_col(const uint32_t* L, int64_t ldl, uint32_t* B, int64_t ldb,
                                                        int64_t i0, int64_t ib, int64_t n, int one) {
  __shared__ uint4 sl[TB][TB];          // L[i0 + r][i0 + c] decoded A-format {M, E, sigma, pattern}
  __shared__ uint4 sb[TB][LC_T];        // final rows of each thread's column: B-format {M, E, sg, pattern}
  __shared__ uint32_t ps[LC_G][LC_T];   // generic path: the group's values as patterns
  __shared__ uint32_t lmask[TB];        // bit c of row r: L[r][c] is a fast operand (rows >= ib: all ones)
  __shared__ uint4 tp[pg::TSIZE], tx[pg::TSIZE];
  const int lane = threadIdx.x;
  const int64_t col = (int64_t)blockIdx.x * LC_T + lane;
  const bool live = col < n;
  pg::fill_tables(tp, tx, lane, LC_T);
  // stage L's block (row r: lane = column, coalesced) and the column's ib
  // values of B: all loads first (in flight together), then decode L in place
  // with the fast masks by ballot (a compact loop: this code runs once)
#pragma unroll
  for (int r = 0; r < TB; r++) {
    sl[r][lane].w = r >= ib ? 0x40000000u : (lane < r ? L[(i0 + r) * ldl + i0 + lane] : 0u);   // rows >= ib: dummy 1.0
    sb[r][lane].w = (live && r < ib) ? B[(i0 + r) * ldb + col] : 0u;     // the input, until row r is final
  }
  __syncwarp();
#pragma unroll 1
  for (int r = 0; r < TB; r++) {
    const uint32_t x = sl[r][lane].w;
    uint4 d;
    const bool f = fast_a(x, d);
    sl[r][lane] = make_uint4(d.x, d.y, d.z, x);
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, f);
    if (lane == 0) lmask[r] = r >= ib ? 0xFFFFFFFFu : (bal & ((1u << r) - 1u));
  }
  pg::MacConst K;
  K.one = (uint32_t)one;
  K.sixteen = 16u * K.one;
  K.tp0 = (uint32_t)__cvta_generic_to_shared(tp + pg::TBIAS);
  K.tx0 = (uint32_t)__cvta_generic_to_shared(tx + pg::TBIAS) - 30u * 16u;
  __syncthreads();
  if (!live) return;
  uint32_t bmask = 0u;                    // bit k: final row k is a fast B operand
  for (int g0 = 0; g0 < ib; g0 += LC_G) {
    LaneVal v[LC_G];
    uint32_t lg = 0xFFFFFFFFu;
#pragma unroll
    for (int u = 0; u < LC_G; u++) {
      lv_load(v[u], sb[g0 + u][lane].w);
      lg &= lmask[g0 + u];
    }
    // the updates from the final rows k < g0, ascending k, in slabs
    for (int k0 = 0; k0 < g0; k0 += LC_SLAB) {
      const int kn = (g0 - k0) < LC_SLAB ? (g0 - k0) : LC_SLAB;
      const uint32_t sm = ((1u << kn) - 1u) << k0;
      bool ok = (bmask & sm) == sm && (lg & sm) == sm;
#pragma unroll
      for (int u = 0; u < LC_G; u++) ok = ok && v[u].dec;
      if (ok) {
        for (int k = k0; k < k0 + kn; k++) {
          const uint4 bk = sb[k][lane];
          uint32_t bad = 0u;
#pragma unroll
          for (int u = 0; u < LC_G; u++) {
            const uint4 ad = sl[g0 + u][k];
            pg::mac<pg::MacConst, false>(v[u].a, ad.x, (int32_t)ad.y, (int32_t)ad.z, bk.x, (int32_t)bk.y,
                                         -(int32_t)bk.z, K, bad);
          }
        }
#pragma unroll
        for (int u = 0; u < LC_G; u++) lc_renorm(v[u]);
      } else {
#pragma unroll
        for (int u = 0; u < LC_G; u++) ps[u][lane] = lv_pattern(v[u]);
#pragma unroll 1
        for (int k = k0; k < k0 + kn; k++) {
          const uint32_t bp = sb[k][lane].w;
#pragma unroll 1
          for (int u = 0; u < LC_G; u++) ps[u][lane] = sub(ps[u][lane], mul(sl[g0 + u][k].w, bp));
        }
#pragma unroll
        for (int u = 0; u < LC_G; u++) lv_load(v[u], ps[u][lane]);
      }
    }
    // the in-group triangle: row g0 + u is final once its predecessors are
    int ugen = LC_G;
#pragma unroll
    for (int u = 0; u < LC_G; u++) {
      if (ugen == LC_G) {
        const bool opf = lv_operand(v[u]);
        bool ok = opf;
#pragma unroll
        for (int w = u + 1; w < LC_G; w++) ok = ok && v[w].dec && ((lmask[g0 + w] >> (g0 + u)) & 1u);
        if (!ok) {
          ugen = u;
        } else {
          const uint32_t pat = pg::acc_encode(v[u].a);
          sb[g0 + u][lane] = make_uint4(v[u].a.M, (uint32_t)v[u].a.E, (uint32_t)v[u].a.sg, pat);
          bmask |= 1u << (g0 + u);
          if (g0 + u < ib) B[(i0 + g0 + u) * ldb + col] = pat;
          uint32_t bad = 0u;
#pragma unroll
          for (int w = u + 1; w < LC_G; w++) {
            const uint4 ad = sl[g0 + w][g0 + u];
            pg::mac<pg::MacConst, false>(v[w].a, ad.x, (int32_t)ad.y, (int32_t)ad.z, v[u].a.M, v[u].a.E, -v[u].a.sg,
                                         K, bad);
          }
        }
      }
    }
    if (ugen < LC_G) {                    // the rest of the triangle on patterns
#pragma unroll
      for (int u = 0; u < LC_G; u++)
        if (u >= ugen) ps[u][lane] = lv_pattern(v[u]);
#pragma unroll 1
      for (int u = ugen; u < LC_G; u++) {
        const uint32_t pat = ps[u][lane];
        LaneVal f;
        lv_load(f, pat);
        const bool opf = lv_operand(f);
        sb[g0 + u][lane] = make_uint4(f.a.M, (uint32_t)f.a.E, (uint32_t)f.a.sg, pat);
        if (opf) bmask |= 1u << (g0 + u);
        if (g0 + u < ib) B[(i0 + g0 + u) * ldb + col] = pat;
#pragma unroll 1
        for (int w = u + 1; w < LC_G; w++) ps[w][lane] = sub(ps[w][lane], mul(sl[g0 + w][g0 + u].w, pat));
      }
    }
  }
}

// Right, lower, transposed, non-unit: columns j0..j0+jb-1 of B (jb <= 16).
// Half-warp per row of B (two rows per warp), lane = column (coalesced):
// step k finalises b_k <- b_k (/) l_kk, broadcasts it within the half-warp,
// and columns j > k apply b_j <- b_j (-) b_k (x) l_jk (ascending k).
constexpr int TBR = 16;

__global__ void __launch_bounds__(1024) k_trsm_rltn_blk(const uint32_t* L, int64_t ldl, uint32_t* B, int64_t ldb,
                                                        int64_t j0, int64_t jb, int64_t m, const int32_t* stop) {
  __shared__ uint32_t sl[TBR][TBR + 1];
  if (stop != nullptr && *stop != 0) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int col = lane & (TBR - 1), half = lane & TBR;
  if (threadIdx.x < TBR * TBR) {
    const int rr = threadIdx.x / TBR, cc = threadIdx.x % TBR;
    if (rr < jb) sl[rr][cc] = cc <= rr ? L[(j0 + rr) * ldl + j0 + cc] : 0u;
  }
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * 64 + wid * 2 + (half ? 1 : 0);
  if ((int64_t)blockIdx.x * 64 + wid * 2 >= m) return;          // whole warp out of range
  const bool live = r < m && col < jb;
  LaneVal b;
  lv_load(b, live ? B[r * ldb + j0 + col] : 0u);
  for (int k = 0; k < jb; k++) {
    if (col == k && live) lv_load(b, div(lv_pattern(b), sl[k][k]));
    const bool bf = lv_operand(b);
    const int src = half | k;
    const uint32_t bM = __shfl_sync(0xFFFFFFFFu, b.a.M, src);
    const int32_t bE = __shfl_sync(0xFFFFFFFFu, b.a.E, src);
    const int32_t bs = __shfl_sync(0xFFFFFFFFu, b.a.sg, src);
    const bool bfk = __shfl_sync(0xFFFFFFFFu, (int)bf, src) != 0;
    const uint32_t bpk = __shfl_sync(0xFFFFFFFFu, col == k ? lv_pattern(b) : 0u, src);   // for the generic path
    if (live && col > k) {
      const uint32_t ap = sl[col][k];
      uint4 ad;
      const bool af = fast_a(ap, ad);
      lv_fms(b, ap, af, ad, bM, bE, bs, bfk, bpk);
    }
  }
  if (live) B[r * ldb + j0 + col] = lv_pattern(b);
}

// ---- fused right TRSM (Cholesky L21 = A21 L11^-T), n <= 256 ----------------
// Rows of B are independent, so one CTA solves FR_ROWS whole rows: B's tile
// lives in shared memory (patterns); per W-column block J a group of W lanes
// per row runs the in-block substitution (lane = column, as k_trsm_rltn_blk),
// publishes the block's W final values decoded, and every thread then updates
// its own columns of the later blocks with them (the fast MAC with the
// GEMM's shared-memory constant tables; L's block column staged decoded,
// k-major so a lane group reads consecutive words).  Per element the updates
// still arrive one at a time in ascending k (Q6).
constexpr int FR_NMAX = 256, FR_W = 16;

template <int W, int FR_ROWS>
struct FrSmem {
  uint32_t b[FR_ROWS][FR_NMAX + 1];          // the CTA's rows of B (patterns)
  uint4 ld[W][FR_NMAX];                       // L[j][c0 + k] decoded A-format {M, E, sigma (0: slow), pattern}
  uint4 bop[FR_ROWS][W];                      // block J's final values, B-format {M, E, sg (0: slow), pattern}
  uint32_t lblk[W][W + 1];                    // L's diagonal block J (patterns)
  uint4 lblkd[W][W];                          // the same, decoded A-format {M, E, sigma, fast}
  uint4 ldiag[W];                             // L[c0 + k][c0 + k] as a divisor {M hidden@30, E, sg, fast}
  double ldrcp[W];                            // RN(2^32 / M) of each diagonal divisor
  int colfast[FR_NMAX];                       // column j's staged L values all fast-path operands
  int rowfast[FR_ROWS];                       // row r's block-J values all fast-path operands
  uint4 tp[pg::TSIZE];                        // the MAC's per-scale constant tables
  uint4 tx[pg::TSIZE];
};

template <int W, int FR_ROWS>
__global__ void __launch_bounds__(FR_ROWS * W, 2) k_trsm_rltn_fused(const uint32_t* L, int64_t ldl, uint32_t* B,
                                                                 int64_t ldb, int64_t m, int64_t n, const int32_t* stop,
                                                                 int one) {
  constexpr int NT = FR_ROWS * W;
  extern __shared__ __align__(16) unsigned char fr_raw[];
  FrSmem<W, FR_ROWS>& S = *reinterpret_cast<FrSmem<W, FR_ROWS>*>(fr_raw);
  if (stop != nullptr && *stop != 0) return;
  const int tid = threadIdx.x;
  const int r = tid / W, c = tid % W;                  // row of the tile, column within a block
  const int grp = (tid & 31) & ~(W - 1);               // first lane of this row's lane group
  const int64_t r0 = (int64_t)blockIdx.x * FR_ROWS;
  const int64_t rows = (m - r0) < FR_ROWS ? (m - r0) : FR_ROWS;
  pg::fill_tables(S.tp, S.tx, tid, NT);
  pg::MacConst K;
  K.one = (uint32_t)one; K.sixteen = 16u * K.one;
  K.tp0 = (uint32_t)__cvta_generic_to_shared(S.tp + pg::TBIAS);
  K.tx0 = (uint32_t)__cvta_generic_to_shared(S.tx + pg::TBIAS) - 30u * 16u;
  for (int e = tid; e < FR_ROWS * (int)n; e += NT) {
    const int rr = e / (int)n, cc = e % (int)n;
    S.b[rr][cc] = rr < rows ? B[(r0 + rr) * ldb + cc] : 0u;
  }
  const int nblk = (int)((n + W - 1) / W);
  for (int J = 0; J < nblk; J++) {
    const int c0 = J * W;
    const int jb = (int)((n - c0) < W ? (n - c0) : W);
    __syncthreads();
    // stage: L's diagonal block J (patterns) and L[j][c0 + k] for j >= c0 + jb (decoded)
    for (int e = tid; e < W * W; e += NT) {
      const int rr = e / W, cc = e % W;
      if (rr < jb && cc <= rr) {
        const uint32_t x = L[(c0 + rr) * ldl + c0 + cc];
        S.lblk[rr][cc] = x;
        uint4 d;
        const bool f = fast_a(x, d);
        S.lblkd[rr][cc] = make_uint4(d.x, d.y, d.z, f ? 1u : 0u);
        if (rr == cc) {
          pg::Acc a;
          const bool ok = pg::acc_decode(x, a) && x != 0u && a.E <= 37 && a.E >= -37;
          S.ldiag[rr] = make_uint4(a.M, (uint32_t)a.E, (uint32_t)a.sg, ok ? 1u : 0u);
          S.ldrcp[rr] = ok ? __drcp_rn((double)a.M) * 4294967296.0 : 0.0;
        }
      }
    }
    const int nrest = (int)n - c0 - jb;
    for (int jj = tid; jj < nrest; jj += NT) {            // thread per column j: its jb values are contiguous
      const int j = c0 + jb + jj;
      int f = 1;
      if (jb == W) {                                      // full block: all W loads in flight together
        uint32_t xs[W];
#pragma unroll
        for (int k = 0; k < W; k++) xs[k] = L[(int64_t)j * ldl + c0 + k];
#pragma unroll
        for (int k = 0; k < W; k++) {
          uint4 d;
          const bool fk = fast_a(xs[k], d);
          S.ld[k][j] = make_uint4(d.x, d.y, d.z, xs[k]);
          f &= (int)fk;
        }
      } else {
        for (int k = 0; k < jb; k++) {
          const uint32_t x = L[(int64_t)j * ldl + c0 + k];
          uint4 d;
          const bool fk = fast_a(x, d);
          S.ld[k][j] = make_uint4(d.x, d.y, d.z, x);
          f &= (int)fk;
        }
      }
      S.colfast[j] = f;
    }
    __syncthreads();
    // in-block substitution: W lanes per row, lane = column
    {
      const bool live = r < rows && c < jb;
      LaneVal v;
      lv_load(v, live ? S.b[r][c0 + c] : 0u);
      for (int k = 0; k < jb; k++) {
        if (c == k && live) {
          const uint4 dv = S.ldiag[k];
          bool done = false;
          if (v.dec && dv.w != 0u) done = pg::acc_div(v.a, dv.x, (int32_t)dv.y, (int32_t)dv.z, S.ldrcp[k], K);
          if (done) {
            if (!(v.a.E <= 75 && v.a.E >= -75) && v.a.E > -1000) { v.pat = pg::acc_encode(v.a); v.dec = false; }
          } else {
            lv_load(v, div(lv_pattern(v), S.lblk[k][k]));
          }
        }
        const bool bf = lv_operand(v);
        const int src = grp | k;
        const uint32_t bM = __shfl_sync(0xFFFFFFFFu, v.a.M, src);
        const int32_t bE = __shfl_sync(0xFFFFFFFFu, v.a.E, src);
        const int32_t bs = __shfl_sync(0xFFFFFFFFu, v.a.sg, src);
        const bool bfk = __shfl_sync(0xFFFFFFFFu, (int)bf, src) != 0;
        const bool bdk = __shfl_sync(0xFFFFFFFFu, (int)v.dec, src) != 0;
        const uint32_t bpraw = __shfl_sync(0xFFFFFFFFu, v.pat, src);
        if (live && c > k) {
          const uint4 ad = S.lblkd[c][k];
          if (ad.w != 0u && bfk && v.dec) {
            uint32_t bad = 0u;
            pg::mac(v.a, ad.x, (int32_t)ad.y, (int32_t)ad.z, bM, bE, -bs, K, bad);
            if (!(v.a.E <= 75 && v.a.E >= -75) && v.a.E > -1000) { v.pat = pg::acc_encode(v.a); v.dec = false; }
          } else {
            pg::Acc bk{bM, bE, bs};
            const uint32_t bp = bdk ? pg::acc_encode(bk) : bpraw;        // b_k's pattern (rare path)
            lv_load(v, sub(lv_pattern(v), mul(S.lblk[c][k], bp)));
          }
        }
      }
      const bool opf = lv_operand(v) || !live;
      const unsigned grpmask = (W == 32 ? 0xFFFFFFFFu : ((1u << W) - 1u)) << grp;
      const bool allf = (__ballot_sync(0xFFFFFFFFu, opf) & grpmask) == grpmask;
      if (live) {
        const uint32_t x = lv_pattern(v);
        S.b[r][c0 + c] = x;
        S.bop[r][c] = make_uint4(v.a.M, (uint32_t)v.a.E, (uint32_t)(-v.a.sg), x);   // sign pre-negated: c (-) a b
      }
      if (c == 0) S.rowfast[r] = allf ? 1 : 0;
    }
    __syncthreads();
    // updates of the later blocks: thread (r, c) owns columns c0 + jb + c + W t.
    // A column whose k-loop has only fast operands and an accumulator within
    // |E| <= 75 stays inside the MAC's exact range for all jb <= 16 steps
    // (|Ep| <= 75, |E| grows by <= 1 per step, cancellation stops at >= -106).
    // Four of the thread's columns are advanced together (independent chains
    // for ILP); a group with any slow column runs the generic path.
    if (r < rows) {
      const bool rf = S.rowfast[r] != 0;
      constexpr int G = 4;
      for (int col0 = c0 + jb + c; col0 < (int)n; col0 += G * W) {
        pg::Acc a[G];
        uint32_t x[G];
        bool ok = rf;
#pragma unroll
        for (int u = 0; u < G; u++) {
          const int col = col0 + u * W;
          const bool in = col < (int)n;
          x[u] = in ? S.b[r][col] : 0u;
          const bool d = pg::acc_decode(x[u], a[u]) && (x[u] == 0u || (a[u].E <= 75 && a[u].E >= -75));
          ok = ok && d && (!in || S.colfast[col] != 0);
        }
        if (ok) {
          uint32_t bad = 0u;
#pragma unroll 2
          for (int k = 0; k < jb; k++) {
            const uint4 bd = S.bop[r][k];
#pragma unroll
            for (int u = 0; u < G; u++) {
              const uint4 ad = S.ld[k][min(col0 + u * W, (int)n - 1)];
              pg::mac(a[u], ad.x, (int32_t)ad.y, (int32_t)ad.z, bd.x, (int32_t)bd.y, (int32_t)bd.z, K, bad);
            }
          }
#pragma unroll
          for (int u = 0; u < G; u++)
            if (col0 + u * W < (int)n) S.b[r][col0 + u * W] = pg::acc_encode(a[u]);
        } else {
#pragma unroll 1
          for (int u = 0; u < G; u++) {
            const int col = col0 + u * W;
            if (col >= (int)n) break;
            uint32_t y = x[u];
            for (int k = 0; k < jb; k++) y = sub(y, mul(S.ld[k][col].w, S.bop[r][k].w));
            S.b[r][col] = y;
          }
        }
      }
    }
  }
  __syncthreads();
  for (int e = tid; e < FR_ROWS * (int)n; e += NT) {
    const int rr = e / (int)n, cc = e % (int)n;
    if (rr < rows) B[(r0 + rr) * ldb + cc] = S.b[rr][cc];
  }
}

// ---- Cholesky leaf: b <= 32 diagonal block, one CTA, thread (i, j) owns a_ij --
// Textbook loop (reading Q9): for k: if signed(a_kk) <= 0 -> info = k+1, stop;
// a_kk <- sqrt(a_kk); a_ik <- a_ik (/) a_kk; a_ij <- a_ij (-) a_ik (x) a_jk.
// Warp = column j, lane = row i, so the divisions of step k are one warp's
// work; column k is published through shared memory as patterns plus decoded
// operands, and each thread keeps its element decoded across the k loop.
__global__ void __launch_bounds__(1024) k_potf2_leaf(uint32_t* A, int64_t lda, int64_t b, int32_t* info,
                                                     int64_t row_base) {
  __shared__ uint32_t colp[TB];          // column k patterns
  __shared__ uint4 cola[TB];             // column k, A-format decode (hidden@31) + fast flag in .w
  __shared__ uint4 colb[TB];             // column k, B-format decode (hidden@30) + fast flag in .w
  __shared__ int fail;
  if (*info != 0) return;                                  // an earlier block failed: stop
  const int j = threadIdx.x >> 5, i = threadIdx.x & 31;    // column (warp), row (lane)
  const bool in = i < b && j <= i && j < b;
  LaneVal v;
  lv_load(v, in ? A[i * lda + j] : 0u);
  if (threadIdx.x == 0) fail = 0;
  __syncthreads();
  int k = 0;
  for (; k < b; k++) {
    if (j == k) {                                          // warp k: pivot, then the column's divisions
      uint32_t d = 0u;
      if (i == k) {
        d = lv_pattern(v);
        if ((int32_t)d > 0) {
          lv_load(v, p32::sqrt(d));
          d = lv_pattern(v);
        }
      }
      d = __shfl_sync(0xFFFFFFFFu, d, k);
      if ((int32_t)d <= 0) {                               // zero, negative or NaR pivot
        if (i == k) { fail = 1; *info = (int32_t)(row_base + k + 1); }
      } else if (in && i > k) {
        // decoded division by the shared divisor (one reciprocal), generic outside its range
        pg::Acc dv;
        const bool dok = pg::acc_decode(d, dv) && dv.E <= 37 && dv.E >= -37;
        bool done = false;
        if (dok && v.dec) {
          done = pg::acc_div(v.a, dv.M, dv.E, dv.sg, __drcp_rn((double)dv.M) * 4294967296.0, pg::CalcConst());
          if (done && !(v.a.E <= 75 && v.a.E >= -75) && v.a.E > pg::E_ZERO_LIMIT) {
            v.pat = pg::acc_encode(v.a);
            v.dec = false;
          }
        }
        if (!done) lv_load(v, div(lv_pattern(v), d));
        const uint32_t x = lv_pattern(v);
        colp[i] = x;
        uint4 ad;
        cola[i] = fast_a(x, ad) ? make_uint4(ad.x, ad.y, ad.z, 1u) : make_uint4(0u, 0u, 0u, 0u);
        colb[i] = lv_operand(v) ? make_uint4(v.a.M, (uint32_t)v.a.E, (uint32_t)v.a.sg, 1u) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
    __syncthreads();
    if (fail) break;
    if (in && j > k) {
      const uint4 ad = cola[i], bd = colb[j];
      lv_fms(v, colp[i], ad.w != 0u, ad, bd.x, (int32_t)bd.y, (int32_t)bd.z, bd.w != 0u, colp[j]);
    }
    __syncthreads();
  }
  if (in) A[i * lda + j] = lv_pattern(v);
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

// C <- (alpha (x) T) (+) (beta (x) C), elementwise (the Eq.2 epilogue, SPEC S:200 order)
__global__ void k_axpby(uint32_t alpha, const uint32_t* T, int64_t ldt, uint32_t beta, uint32_t* C, int64_t ldc,
                        int64_t m, int64_t n) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m * n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    C[i * ldc + j] = add(mul(alpha, T[i * ldt + j]), mul(beta, C[i * ldc + j]));
  }
}

// Four elements per thread per iteration (two 16-byte loads in, one 16-byte
// store out, or the reverse) when both arrays are 16-byte aligned; a scalar
// tail.  HBM-bound: 12 bytes per element.
__global__ void k_from_f64(const double* x, uint32_t* out, int64_t count) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if ((((uintptr_t)x | (uintptr_t)out) & 15u) == 0u) {
    const int64_t nq = count / 4;
    const double2* x2 = reinterpret_cast<const double2*>(x);
    uint4* o4 = reinterpret_cast<uint4*>(out);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += stride) {
      const double2 a = __ldcs(x2 + 2 * q), b = __ldcs(x2 + 2 * q + 1);
      __stcs(o4 + q, make_uint4(p32::from_f64(a.x), p32::from_f64(a.y), p32::from_f64(b.x), p32::from_f64(b.y)));
    }
    done = nq * 4;
  }
  for (int64_t i = done + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
    out[i] = p32::from_f64(x[i]);
}

__global__ void k_to_f64(const uint32_t* p, double* out, int64_t count) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if ((((uintptr_t)p | (uintptr_t)out) & 15u) == 0u) {
    const int64_t nq = count / 4;
    const uint4* p4 = reinterpret_cast<const uint4*>(p);
    double2* o2 = reinterpret_cast<double2*>(out);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += stride) {
      const uint4 v = __ldcs(p4 + q);
      __stcs(o2 + 2 * q, make_double2(p32::to_f64(v.x), p32::to_f64(v.y)));
      __stcs(o2 + 2 * q + 1, make_double2(p32::to_f64(v.z), p32::to_f64(v.w)));
    }
    done = nq * 4;
  }
  for (int64_t i = done + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
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
  static const int64_t leaf = [] {
    const char* e = getenv("POSIT_PANEL_LEAF");
    int64_t v = e ? atoll(e) : 32;
    return v < 1 ? (int64_t)1 : (v > 64 ? (int64_t)64 : v);
  }();
  return leaf;
}

// Unblocked leaf (w <= 64 columns): per column one swap/divide launch and one
// update launch that also searches the next column's pivot.
static int getrf_leaf(int64_t m, int64_t w, uint32_t* A, int64_t lda, int32_t* ipiv, int32_t* info, int64_t row_base,
                      LeafWs* ws, bool allow_coop, cudaStream_t st) {
  if (cudaMemsetAsync(ws, 0, LEAF_WS_ZERO, st) != cudaSuccess) return POSIT_ECUDA;
  // one cooperative launch when the rows fit the CTAs' shared memory
  struct CoopCfg { int coop; int nsm; };
  static const CoopCfg cfg = [] {
    CoopCfg c{1, 148};
    const char* e = getenv("POSIT_LEAF_COOP");
    c.coop = e ? atoi(e) : 1;
    int dev = 0, ok = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&c.nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&ok, cudaDevAttrCooperativeLaunch, dev);
    if (!ok) c.coop = 0;
    cudaFuncSetAttribute(k_leaf_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(k_leaf_coop1<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(k_leaf_coop1<TAIL_WMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    return c;
  }();
  const int coop = cfg.coop, nsm = cfg.nsm;
  // on the caller's stream: one CTA of 256 threads per SM; on a side stream
  // (lookahead, sharing the SMs with the trailing GEMM): a few CTAs of 1024
  static const int force = [] {                 // POSIT_LEAF_CTAS = 16 / 148: force one configuration (tests, sweeps)
    const char* e = getenv("POSIT_LEAF_CTAS");
    return e ? atoi(e) : 0;
  }();
  const bool wide = force ? force > 16 : allow_coop;
  static const int side_ctas = [] {              // side-stream leaf CTAs (1024 threads each)
    const char* e = getenv("POSIT_SIDE_LEAF_CTAS");
    const int v = e ? atoi(e) : 16;
    return v > 0 ? v : 16;
  }();
  int nctas = wide ? nsm : (nsm < side_ctas ? nsm : side_ctas);
  int nthr = wide ? COOP_THREADS : 1024;
  if (force > 0 && force != 16 && force != 148) { nctas = force < nsm ? force : nsm; nthr = COOP_THREADS; }
  const int64_t rpc = (m + nctas - 1) / nctas;
  const size_t smem = (size_t)rpc * (size_t)w * sizeof(uint32_t);
  if (coop && smem <= 160 * 1024 && w <= TAIL_WMAX) {
    int64_t mm = m, ww = w, rr = rpc, rbase = row_base, ld = lda;
    const bool wide_w = w > 64;
    uint32_t* cand = wide_w ? &ws->tcand[0][0][0] : &ws->cand[0][0][0];
    uint32_t* jrow = wide_w ? &ws->tjrow[0][0] : &ws->jrow[0][0];
    void* args[] = {&A, &ld, &mm, &ww, &rr, &ipiv, &info, &rbase, &ws, &cand, &jrow};
    const unsigned grid = (unsigned)((m + rpc - 1) / rpc);
    // coop 1: one grid sync per column (default); coop 2: two (publish after the pivot is known; w <= 64)
    const void* kfn = nullptr;
    if (grid <= (unsigned)LEAF_MAXCTA && (coop != 2 || wide_w))
      kfn = wide_w ? (const void*)k_leaf_coop1<TAIL_WMAX> : (const void*)k_leaf_coop1<64>;
    else if (!wide_w)
      kfn = (const void*)k_leaf_coop;
    if (kfn != nullptr) {
      pb_count_launch();
      if (cudaLaunchCooperativeKernel(kfn, dim3(grid), dim3(nthr), args, smem, st) == cudaSuccess)
        return last_launch();
      (void)cudaGetLastError();                        // fall back to the per-column launches
    }
  }
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

// The fused tail: LU with partial pivoting of the whole remaining m x w block
// (w <= TAIL_WMAX) as ONE cooperative right-looking launch (one grid sync per
// column), instead of the last few blocked steps whose recursive panels are
// latency-bound.  Same per-element order (Q6).  Returns POSIT_ENOTSUP when the
// block does not fit the CTAs' shared memory (the caller keeps the blocked path).
int pb_getrf_tail(int64_t m, int64_t w, uint32_t* A, int64_t lda, int32_t* ipiv, int32_t* info, int64_t row_base,
                  void* ws, cudaStream_t st) {
  if (m <= 0 || w <= 0) return 0;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t rpc = (m + nsm - 1) / nsm;
  if (w > TAIL_WMAX || (size_t)rpc * (size_t)w * sizeof(uint32_t) > 160 * 1024) return POSIT_ENOTSUP;
  return getrf_leaf(m, w, A, lda, ipiv, info, row_base, static_cast<LeafWs*>(ws), true, st);
}

// Recursive panel LU (the traversal of LAPACK getrf2): factor the left half,
// apply its swaps to the right half, U12 by TRSM, the right half's update by
// the fast GEMM, factor the right half, apply its swaps to the left half.
// Every element still receives its products one at a time in ascending k
// (reading Q6), so the bits equal the column-by-column loop.
int pb_getrf_panel(int64_t m, int64_t b, uint32_t* A, int64_t lda, int32_t* ipiv, int32_t* info, int64_t row_base,
                   void* ws, bool allow_coop, cudaStream_t st) {
  const int64_t w = m < b ? m : b;
  const int64_t leaf = panel_leaf();
  if (w <= leaf) return getrf_leaf(m, b, A, lda, ipiv, info, row_base, static_cast<LeafWs*>(ws), allow_coop, st);
  int64_t w1 = ((w / 2 + leaf - 1) / leaf) * leaf;
  if (w1 >= w) w1 = w - leaf;
  int rc;
  if ((rc = pb_getrf_panel(m, w1, A, lda, ipiv, info, row_base, ws, allow_coop, st))) return rc;
  if ((rc = pb_laswp(b - w1, A + w1, lda, 0, w1, ipiv, row_base, st))) return rc;
  if ((rc = pb_trsm_llnu(w1, b - w1, A, lda, A + w1, lda, st))) return rc;
  if (m > w1) {
    pg::Params P{m - w1, b - w1, w1, A + w1 * lda, lda, A + w1, lda, A + w1 * lda + w1, lda, 1, 1, nullptr};
    if ((rc = pb_launch_gemm(P, false, false, st))) return rc;
    if ((rc = pb_getrf_panel(m - w1, b - w1, A + w1 * lda + w1, lda, ipiv + w1, info, row_base + w1, ws, allow_coop,
                             st)))
      return rc;
    if ((rc = pb_laswp(w1, A + w1 * lda, lda, 0, w - w1, ipiv + w1, row_base + w1, st))) return rc;
  }
  return last_launch();
}

int pb_laswp(int64_t ncols, uint32_t* A, int64_t lda, int64_t k1, int64_t k2, const int32_t* ipiv, int64_t ipiv_base,
             cudaStream_t st) {
  if (ncols <= 0 || k2 <= k1) return 0;
  constexpr size_t smem = 2 * SWP_MAX * SWP_COLS * sizeof(uint32_t);
  static const bool attr = [] {
    return cudaFuncSetAttribute(k_laswp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess;
  }();
  (void)attr;
  pb_count_launch();
  k_laswp<<<(unsigned)((ncols + SWP_COLS - 1) / SWP_COLS), 256, smem, st>>>(A, lda, ncols, k1, k2, ipiv, ipiv_base);
  return last_launch();
}

int pb_trsm_llnu(int64_t m, int64_t n, const uint32_t* L, int64_t ldl, uint32_t* B, int64_t ldb, cudaStream_t st) {
  if (m <= 0 || n <= 0) return 0;
  // thread per column (row groups of 4; -1 = auto) once the columns fill the
  // SMs: one such launch costs ~46 us whatever its width up to 592 warps,
  // the warp-per-column kernel ~34 us per wave of 148 CTAs (r02v launch lists)
  static const int col_env = [] {
    const char* e = getenv("POSIT_LLNU_COL");
    const int v = e == nullptr ? -1 : atoi(e);
    return v == 0 || v == 4 || v == 8 ? v : -1;
  }();
  const int use_col = col_env >= 0 ? col_env : (n > 148 * TB ? 4 : 0);
  static const int blk_env = [] {                 // warp-per-column CTA width: 8 (default) or 32 columns
    const char* e = getenv("POSIT_LLNU_BLK");
    return e ? atoi(e) : 8;
  }();
  for (int64_t i0 = 0; i0 < m; i0 += TB) {
    const int64_t ib = (m - i0) < TB ? (m - i0) : TB;
    if (ib > 1) {
      pb_count_launch();
      if (use_col == 8)
        k_trsm_llnu_col<8><<<(unsigned)((n + LC_T - 1) / LC_T), LC_T, 0, st>>>(L, ldl, B, ldb, i0, ib, n, 1);
      else if (use_col == 4)
        k_trsm_llnu_col<4><<<(unsigned)((n + LC_T - 1) / LC_T), LC_T, 0, st>>>(L, ldl, B, ldb, i0, ib, n, 1);
      else if (blk_env == 8)
        k_trsm_llnu_blkw<8><<<(unsigned)((n + 7) / 8), 256, 0, st>>>(L, ldl, B, ldb, i0, ib, n);
      else
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
  if (n <= FR_NMAX) {
    // one fused launch: each CTA solves FR_ROWS whole rows
    // variant: W lanes per row x FR_ROWS rows per CTA (env POSIT_RLTN = "W,ROWS")
    static const int var = [] {
      const char* e = getenv("POSIT_RLTN");
      int w = 16, r = 16;
      if (e) sscanf(e, "%d,%d", &w, &r);
      cudaFuncSetAttribute(k_trsm_rltn_fused<16, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(FrSmem<16, 16>));
      cudaFuncSetAttribute(k_trsm_rltn_fused<16, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(FrSmem<16, 32>));
      cudaFuncSetAttribute(k_trsm_rltn_fused<8, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(FrSmem<8, 16>));
      cudaFuncSetAttribute(k_trsm_rltn_fused<8, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(FrSmem<8, 32>));
      return w * 100 + r;
    }();
    pb_count_launch();
#define PB_RLTN(W_, R_)                                                                                              \
  k_trsm_rltn_fused<W_, R_><<<(unsigned)((m + R_ - 1) / R_), R_ * W_, sizeof(FrSmem<W_, R_>), st>>>(L, ldl, B, ldb, m, \
                                                                                                   n, stop, 1)
    if (var == 1632) PB_RLTN(16, 32);
    else if (var == 816) PB_RLTN(8, 16);
    else if (var == 832) PB_RLTN(8, 32);
    else PB_RLTN(16, 16);
#undef PB_RLTN
    return last_launch();
  }
  for (int64_t j0 = 0; j0 < n; j0 += TBR) {
    const int64_t jb = (n - j0) < TBR ? (n - j0) : TBR;
    pb_count_launch();
    k_trsm_rltn_blk<<<(unsigned)((m + 63) / 64), 1024, 0, st>>>(L, ldl, B, ldb, j0, jb, m, stop);
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
// Tiny GEMM / SYRK (the panel-internal updates: m, n <= 128, K <= 64): one
// thread per output element, its chain of K updates in ascending k (Q6), each
// the decoded-domain MAC with the generic fallback.  A single-CTA launch of the
// tiled kernel spends ~56 us on such a shape (long per-thread loops on one SM);
// this one is bound by one short chain.  alpha = +1 adds: b enters negated
// (exact).  SYRK: lower triangle only.  A no-op once *stop != 0.
__global__ void __launch_bounds__(256) k_gemm_tiny(pg::Params P, int transb, int syrk) {
  if (P.stop != nullptr && *P.stop != 0) return;
  const int64_t i = (int64_t)blockIdx.y * 16 + (threadIdx.x >> 4);
  const int64_t j = (int64_t)blockIdx.x * 16 + (threadIdx.x & 15);
  if (i >= P.m || j >= P.n || (syrk && j > i)) return;
  LaneVal c;
  lv_load(c, P.beta ? P.C[i * P.ldc + j] : 0u);
  // operands in chunks of 8, all loads of a chunk in flight before its chain
  constexpr int CH = 8;
  const int64_t sa = P.transa ? P.lda : 1, sa0 = P.transa ? i : i * P.lda;
  const int64_t sb = transb ? 1 : P.ldb, sb0 = transb ? j * P.ldb : j;
  for (int64_t q0 = 0; q0 < P.k; q0 += CH) {
    uint32_t a[CH], b[CH];
#pragma unroll
    for (int u = 0; u < CH; u++) {
      const bool in = q0 + u < P.k;
      a[u] = in ? P.A[sa0 + (q0 + u) * sa] : 0u;
      b[u] = in ? P.B[sb0 + (q0 + u) * sb] : 0u;
    }
#pragma unroll
    for (int u = 0; u < CH; u++) {
      if (q0 + u < P.k) {
        const uint32_t bp = P.neg ? b[u] : 0u - b[u];   // c (+) a b = c (-) a (-b), negation exact
        uint4 ad;
        const bool af = fast_a(a[u], ad);
        LaneVal bv;
        lv_load(bv, bp);
        lv_fms(c, a[u], af, ad, bv.a.M, bv.a.E, bv.a.sg, lv_operand(bv), bp);
      }
    }
  }
  P.C[i * P.ldc + j] = lv_pattern(c);
}

int pb_launch_gemm_tiny(const pg::Params& P, bool transb, bool syrk, cudaStream_t st) {
  pb_count_launch();
  const dim3 grid((unsigned)((P.n + 15) / 16), (unsigned)((P.m + 15) / 16));
  k_gemm_tiny<<<grid, 256, 0, st>>>(P, transb ? 1 : 0, syrk ? 1 : 0);
  return last_launch();
}

// Small SYRK inside the diagonal-block Cholesky: C_lower <- C_lower (-) A A^T
// with one thread per lower element (ascending k per element, Q6).  For
// n <= 256 and k = 32 the GEMM kernel would run on a handful of CTAs with long
// per-thread loops; here every element is its own (short) chain.  A no-op
// once *stop != 0.
__global__ void __launch_bounds__(256) k_syrk_tiny(int64_t n, int64_t k, const uint32_t* A, int64_t lda, uint32_t* C,
                                                   int64_t ldc, const int32_t* stop) {
  if (stop != nullptr && *stop != 0) return;
  const int64_t i = (int64_t)blockIdx.y * 16 + (threadIdx.x >> 4);
  const int64_t j = (int64_t)blockIdx.x * 16 + (threadIdx.x & 15);
  if ((int64_t)blockIdx.x > (int64_t)blockIdx.y || i >= n || j > i) return;
  LaneVal c;
  lv_load(c, C[i * ldc + j]);
  for (int64_t q = 0; q < k; q++) {
    const uint32_t ap = A[i * lda + q], bp = A[j * lda + q];
    uint4 ad;
    const bool af = fast_a(ap, ad);
    LaneVal bv;
    lv_load(bv, bp);
    lv_fms(c, ap, af, ad, bv.a.M, bv.a.E, bv.a.sg, lv_operand(bv), bp);
  }
  C[i * ldc + j] = lv_pattern(c);
}

int pb_potf2(int64_t b, uint32_t* A, int64_t lda, int32_t* info, int64_t row_base, cudaStream_t st) {
  if (b <= 0) return 0;
  static const int mode = [] {                   // 1: blocked right-looking, 32-wide (default); 0: recursive
    const char* e = getenv("POSIT_POTF2");
    return e ? atoi(e) : 1;
  }();
  if (mode == 1 && b <= 256) {
    // right-looking by 32-wide block columns: leaf, the rows below by TRSM,
    // the trailing lower triangle by the one-thread-per-element SYRK
    for (int64_t j0 = 0; j0 < b; j0 += TB) {
      const int64_t jb = (b - j0) < TB ? (b - j0) : TB;
      uint32_t* Ajj = A + j0 * lda + j0;
      pb_count_launch();
      k_potf2_leaf<<<1, 1024, 0, st>>>(Ajj, lda, jb, info, row_base + j0);
      const int64_t r = b - j0 - jb;
      if (r > 0) {
        int rc;
        if ((rc = pb_trsm_rltn(r, jb, Ajj, lda, Ajj + jb * lda, lda, info, st))) return rc;
        pb_count_launch();
        const unsigned t = (unsigned)((r + 15) / 16);
        k_syrk_tiny<<<dim3(t, t), 256, 0, st>>>(r, jb, Ajj + jb * lda, lda, Ajj + jb * lda + jb, lda, info);
      }
    }
    return last_launch();
  }
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
  static const bool attr = [] {
    cudaFuncSetAttribute(k_getrs, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_potrs, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return true;
  }();
  (void)attr;
  pb_count_launch();
  if (chol) k_potrs<<<1, SOLVE_THREADS, smem, st>>>(n, A, lda, b);
  else k_getrs<<<1, SOLVE_THREADS, smem, st>>>(n, A, lda, ipiv, b);
  return last_launch();
}

int pb_iamax_key(int64_t m, const uint32_t* col, int64_t stride, const int32_t* grow, int64_t row_min, long long* out,
                 cudaStream_t st) {
  pb_count_launch();
  k_iamax_key<<<1, 1024, 0, st>>>(m, col, stride, grow, row_min, out);
  return last_launch();
}

int pb_vec_op(int op, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count, cudaStream_t st) {
  if (count <= 0) return 0;
  pb_count_launch();
  k_vec_op<<<grid_for(count, 256), 256, 0, st>>>(op, a, b, out, count);
  return last_launch();
}

int pb_axpby(uint32_t alpha, const uint32_t* T, int64_t ldt, uint32_t beta, uint32_t* C, int64_t ldc, int64_t m,
             int64_t n, cudaStream_t st) {
  if (m <= 0 || n <= 0) return 0;
  pb_count_launch();
  k_axpby<<<grid_for(m * n, 256), 256, 0, st>>>(alpha, T, ldt, beta, C, ldc, m, n);
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
