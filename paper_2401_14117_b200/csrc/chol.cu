// chol.cu -- the diagonal-block Cholesky (potf2) and the
// tiny one-thread-per-output GEMM / SYRK it and the LU panel use.
#include "lanes.cuh"

namespace pl {

// ---- Cholesky leaf: b <= 32 diagonal block, one CTA, thread (i, j) owns a_ij --
// Textbook loop (reading Q9): for k: if signed(a_kk) <= 0 -> info = k+1, stop;
// a_kk <- sqrt(a_kk); a_ik <- a_ik (/) a_kk; a_ij <- a_ij (-) a_ik (x) a_jk.
// Warp = column j, lane = row i, so the divisions of step k are one warp's
// work; column k is published through shared memory as patterns plus decoded
// operands, and each thread keeps its element decoded across the k loop.
__global__ void __launch_bounds__(1024) k_potf2_leaf(uint32_t* A, int64_t lda, int64_t b, int32_t* info,
                                                     int64_t row_base) {
  // column k is published in buffer k & 1: warp k + 1 finishes its own step-k
  // update, then factors column k + 1 before the barrier, so one barrier per
  // column suffices (the buffer it overwrites was last read before the previous one)
  __shared__ uint32_t colp[2][TB];       // column k patterns
  __shared__ uint4 cola[2][TB];          // column k, A-format decode (hidden@31) + fast flag in .w
  __shared__ uint4 colb[2][TB];          // column k, B-format decode (hidden@30) + fast flag in .w
  __shared__ int fail;
  if (*info != 0) return;                                  // an earlier block failed: stop
  const int j = threadIdx.x >> 5, i = threadIdx.x & 31;    // column (warp), row (lane)
  const bool in = i < b && j <= i && j < b;
  LaneVal v;
  lv_load(v, in ? A[i * lda + j] : 0u);
  if (threadIdx.x == 0) fail = 0;
  // warp j factors its column (pivot sqrt, then the divisions) and publishes it
  auto factor = [&](int k) {
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
      const int q = k & 1;
      colp[q][i] = x;
      uint4 ad;
      cola[q][i] = fast_a(x, ad) ? make_uint4(ad.x, ad.y, ad.z, 1u) : make_uint4(0u, 0u, 0u, 0u);
      colb[q][i] = lv_operand(v) ? make_uint4(v.a.M, (uint32_t)v.a.E, (uint32_t)v.a.sg, 1u) : make_uint4(0u, 0u, 0u, 0u);
    }
  };
  __syncthreads();                                         // fail = 0 visible
  if (j == 0 && b > 0) factor(0);
  __syncthreads();
  for (int k = 0; k < b; k++) {
    if (fail) break;
    const int q = k & 1;
    if (in && j > k) {
      const uint4 ad = cola[q][i], bd = colb[q][j];
      lv_fms(v, colp[q][i], ad.w != 0u, ad, bd.x, (int32_t)bd.y, (int32_t)bd.z, bd.w != 0u, colp[q][j]);
    }
    if (j == k + 1 && j < b) factor(k + 1);
    __syncthreads();
  }
  if (in) A[i * lda + j] = lv_pattern(v);
}

}  // namespace pl

using namespace pl;

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

// Diagonal-block Cholesky: right-looking by 32-wide block columns (leaf of
// <= 32 in one CTA, the rows below by the fused TRSM, the trailing lower
// triangle by the one-thread-per-element SYRK), or (POSIT_POTF2=0) the
// recursive potrf2 traversal.  Every stage is a no-op once *info != 0.
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

