// gemm.cu -- Posit(32,2) GEMM (NN, NT) and SYRK-lower kernels + launchers.
// See gemm.cuh for the arithmetic and the order contract.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <initializer_list>
#include <utility>
#include <type_traits>
#include "gemm.cuh"
#include "gemm_common.cuh"
#include "internal.h"

#ifndef PG_KK_UNROLL
#define PG_KK_UNROLL 4   // with the 4 x 2 tiles (r05l: C2 1194 -> 1197; unroll 2 was best for 4 x 4)
#endif

namespace pg {

constexpr int KK_UNROLL = PG_KK_UNROLL;   // k-steps of the fast loop unrolled (each TM x TN MACs)
#ifndef PG_KK_UNROLL_SYRK
#define PG_KK_UNROLL_SYRK 1   // r04z / r05a: SYRK 1135 -> 1141 Gflop/s, C3 184.5 -> 183.6 ms
#endif
constexpr int KK_UNROLL_SYRK = PG_KK_UNROLL_SYRK;   // the same for the SYRK instantiations
#ifndef PG_CPASYNC
#define PG_CPASYNC 1
#endif
#ifndef PG_GROUP_M
#define PG_GROUP_M 32
#endif
constexpr int GROUP_M = PG_GROUP_M;       // row tiles per rasterisation group

// Tile configuration.  One CTA = BM x BN outputs, NTHR threads, each thread a
// TM x TN register tile of decoded accumulators; operands staged in k-slabs
// of BK, double-buffered in shared memory as decoded (M, w) pairs.
template <int BM_, int BN_, int TM_, int TN_, int MINB_, int EFF100 = 100>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, TM = TM_, TN = TN_, BK = 16, MINB = MINB_;
  static constexpr double EFF = EFF100 / 100.0;   // measured full-size rate relative to the 64 x 128 tile
  static constexpr int NTX = BN / TN, NTY = BM / TM, NTHR = NTX * NTY;
  static constexpr int AQN = BM * BK / 4, BQN = BN * BK / 4;    // quads per tile
  static constexpr int AQ = (AQN + NTHR - 1) / NTHR;            // A quads per thread (last may idle)
  static constexpr int BQ = (BQN + NTHR - 1) / NTHR;
  // MAC variants (see gemm.cuh): product table by Ea + Eb for 4 x 4 tiles (PBS),
  // else the PIX table, with the signs folded in (PIXS)
  static constexpr bool PBS = (PG_PROD_BY_SUM != 0) && (TM * TN >= 16);
  static constexpr bool PIX = !PBS && (PG_PIX == 2 || (PG_PIX == 1 && MINB == 1));
  static constexpr bool PIXS = PIX && PG_PIXS != 0;
  // staged operand: {M, E, sigma, w}, or with PIXS only {M, w} (one LDS.64)
  using SV = std::conditional_t<PIXS, uint2, uint4>;
  struct Smem {
    SV a[2][BK][BM];
    SV b[2][BK][BN];
#if PG_CPASYNC
    uint32_t ra[BM * BK];                 // raw patterns of the next slab (cp.async target, by quad)
    uint32_t rb[BK * BN];
#endif
    uint4 tp[3 * PIX_NE > TSIZE ? 3 * PIX_NE : TSIZE];   // PIX layout (up to 3 copies) or by scale
    uint4 tx[TSIZE];
  };
};

// staged-operand accessors ({M, E, sigma, w} or {M, w})
template <class V> __device__ __forceinline__ V sv(const uint4& d);
template <> __device__ __forceinline__ uint4 sv<uint4>(const uint4& d) { return d; }
template <> __device__ __forceinline__ uint2 sv<uint2>(const uint4& d) { return make_uint2(d.x, d.w); }
__device__ __forceinline__ int32_t sv_E(const uint4& v) { return (int32_t)v.y; }
__device__ __forceinline__ int32_t sv_s(const uint4& v) { return (int32_t)v.z; }
__device__ __forceinline__ uint32_t sv_w(const uint4& v) { return v.w; }
__device__ __forceinline__ int32_t sv_E(const uint2&) { return 0; }     // unused by the PIXS MAC
__device__ __forceinline__ int32_t sv_s(const uint2&) { return 1; }
__device__ __forceinline__ uint32_t sv_w(const uint2& v) { return v.y; }

template <class C, bool TRANS_B, bool SYRK>
__global__ void __launch_bounds__(C::NTHR, C::MINB) k_gemm(Params P) {
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, TM = C::TM, TN = C::TN, NTHR = C::NTHR;
  constexpr int AQ = C::AQ, BQ = C::BQ;
  // product table by Ea + Eb for the 16-warp (4 x 4) tiles, by Ep for the 32-warp (4 x 2) ones (r05p)
  constexpr bool PBS = C::PBS, PIX = C::PIX, PIXS = C::PIXS;
  constexpr bool CEM = PG_CECM == 2 || (PG_CECM == 1 && C::MINB == 1) || (PG_CECM == 3 && C::MINB > 1);
  constexpr bool MSL = PG_MSM_SEL == 2 || (PG_MSM_SEL == 1 && C::MINB == 1);
  constexpr uint32_t WM = PIX ? 32u : 16u;   // staged .w = WM E (+ table base on the B side)
  constexpr uint32_t SOFF = PIXS ? PIX_SOFF : 0u;   // + this for a negative operand
  extern __shared__ __align__(16) unsigned char smem_raw[];
  typename C::Smem& S = *reinterpret_cast<typename C::Smem*>(smem_raw);

  const int tid = threadIdx.x;
  const int tx = tid % C::NTX;             // column group
  const int ty = tid / C::NTX;             // row group
  // grouped rasterisation: consecutive CTAs sweep the column tiles of a group
  // of GROUP_M row tiles, so a wave re-reads its A rows and B columns from L2
  const int64_t nbn = gridDim.x, nbm = gridDim.y;
  const int64_t pid = (int64_t)blockIdx.y * nbn + blockIdx.x;
  const int64_t per_group = (int64_t)GROUP_M * nbn;
  const int64_t gfirst = (pid / per_group) * GROUP_M;
  const int64_t gsize = (nbm - gfirst) < GROUP_M ? (nbm - gfirst) : GROUP_M;
  const int64_t row0 = (gfirst + (pid % per_group) % gsize) * BM;
  const int64_t col0 = ((pid % per_group) / gsize) * BN;
  // let a programmatic-dependent successor (an independent update) start its
  // CTAs on SMs this grid's last wave leaves idle
  asm volatile("griddepcontrol.launch_dependents;");
  if (SYRK && col0 > row0 + BM - 1) return;   // tile entirely above the diagonal
  if (P.stop != nullptr && *P.stop != 0) return;

  const uint32_t flip = P.neg ? 1u : 0u;
  fill_tables<PBS, !PIX>(S.tp, S.tx, tid, NTHR);     // visible after the first __syncthreads_or
  if constexpr (PIX) fill_prod_pix<PIXS>(S.tp, tid, NTHR);
  MacConst K;
  K.one = (uint32_t)P.one; K.sixteen = 16u * K.one; K.m2p30 = 0xC0000000u * K.one;
  K.tp0 = (uint32_t)__cvta_generic_to_shared(S.tp + (PIX ? 2 * PIX_SB : TBIAS));
  K.tx0 = (uint32_t)__cvta_generic_to_shared(S.tx + TBIAS) - 30u * 16u;   // indexed by Ex + 30

  // ---- accumulators -------------------------------------------------------
  Acc acc[TM][TN];
  bool bad = false;
  uint32_t badacc = 0u;
#pragma unroll
  for (int i = 0; i < TM; i++) {
#pragma unroll
    for (int j = 0; j < TN; j++) {
      const int64_t r = row0 + ty * TM + i, cc = col0 + tx * TN + j;
      uint32_t cv = 0u;
      if (P.beta && r < P.m && cc < P.n) cv = P.C[r * P.ldc + cc];
      if (!acc_decode(cv, acc[i][j])) bad = true;
    }
  }

  // ---- staging: A tile BM x BK and B tile BK x BN, in quads of 4 words
  uint32_t ra[AQ * 4], rb[BQ * 4];

  auto load_tile = [&](int64_t k0) {
#pragma unroll
    for (int h = 0; h < AQ; h++) {
      const int e = tid + h * NTHR;                   // (row, k quad)
      if (e >= C::AQN) break;
      if (!P.transa) {                                // (row, k quad)
        const int ar = e / (BK / 4), ak = (e % (BK / 4)) * 4;
        const int64_t r = row0 + ar, kq = k0 + ak;
        load_quad(P.A + r * P.lda + kq, r < P.m, P.k - kq, &ra[h * 4]);
      } else {                                        // (k row, row quad): A stored k x m
        const int ak = e / (BM / 4), ar = (e % (BM / 4)) * 4;
        const int64_t kk = k0 + ak, rq = row0 + ar;
        load_quad(P.A + kk * P.lda + rq, kk < P.k, P.m - rq, &ra[h * 4]);
      }
    }
#pragma unroll
    for (int h = 0; h < BQ; h++) {
      const int e = tid + h * NTHR;
      if (e >= C::BQN) break;
      if (!TRANS_B) {                                 // (k row, col quad)
        const int bk = e / (BN / 4), bc = (e % (BN / 4)) * 4;
        const int64_t kk = k0 + bk, cq = col0 + bc;
        load_quad(P.B + kk * P.ldb + cq, kk < P.k, P.n - cq, &rb[h * 4]);
      } else {                                        // (col, k quad)
        const int bc = e / (BK / 4), bk = (e % (BK / 4)) * 4;
        const int64_t kq = k0 + bk, cc = col0 + bc;
        load_quad(P.B + cc * P.ldb + kq, cc < P.n, P.k - kq, &rb[h * 4]);
      }
    }
  };
  auto store_tile = [&](int buf) -> uint32_t {
    uint32_t sp = 0u;
#pragma unroll
    for (int h = 0; h < AQ; h++) {
      const int e = tid + h * NTHR;
      if (e >= C::AQN) break;
      if (!P.transa) {
        const int ar = e / (BK / 4), ak = (e % (BK / 4)) * 4;
#pragma unroll
        for (int q = 0; q < 4; q++) S.a[buf][ak + q][ar] = sv<typename C::SV>(stage_decode<31, WM, SOFF>(ra[h * 4 + q], 0u, sp));
      } else {
        const int ak = e / (BM / 4), ar = (e % (BM / 4)) * 4;
#pragma unroll
        for (int q = 0; q < 4; q++) S.a[buf][ak][ar + q] = sv<typename C::SV>(stage_decode<31, WM, SOFF>(ra[h * 4 + q], 0u, sp));
      }
    }
#pragma unroll
    for (int h = 0; h < BQ; h++) {
      const int e = tid + h * NTHR;
      if (e >= C::BQN) break;
      if (!TRANS_B) {
        const int bk = e / (BN / 4), bc = (e % (BN / 4)) * 4;
#pragma unroll
        for (int q = 0; q < 4; q++) S.b[buf][bk][bc + q] = sv<typename C::SV>(stage_decode<30, WM, SOFF>(rb[h * 4 + q], flip, sp, K.tp0));
      } else {
        const int bc = e / (BK / 4), bk = (e % (BK / 4)) * 4;
#pragma unroll
        for (int q = 0; q < 4; q++) S.b[buf][bk + q][bc] = sv<typename C::SV>(stage_decode<30, WM, SOFF>(rb[h * 4 + q], flip, sp, K.tp0));
      }
    }
    return sp;
  };


#if PG_CPASYNC
  // cp.async staging: each thread copies its own quads of the next slab into
  // the raw buffers and later decodes exactly those quads (no cross-thread
  // dependency on the raw data, so only its own wait_group is needed)
  auto issue_tile = [&](int64_t k0) {
#pragma unroll
    for (int h = 0; h < AQ; h++) {
      const int e = tid + h * NTHR;
      if (e >= C::AQN) break;
      if (!P.transa) {
        const int ar = e / (BK / 4), ak = (e % (BK / 4)) * 4;
        const int64_t r = row0 + ar, kq = k0 + ak;
        cp_quad(&S.ra[e * 4], P.A + r * P.lda + kq, r < P.m, P.k - kq);
      } else {
        const int ak = e / (BM / 4), ar = (e % (BM / 4)) * 4;
        const int64_t kk = k0 + ak, rq = row0 + ar;
        cp_quad(&S.ra[e * 4], P.A + kk * P.lda + rq, kk < P.k, P.m - rq);
      }
    }
#pragma unroll
    for (int h = 0; h < BQ; h++) {
      const int e = tid + h * NTHR;
      if (e >= C::BQN) break;
      if (!TRANS_B) {
        const int bk = e / (BN / 4), bc = (e % (BN / 4)) * 4;
        const int64_t kk = k0 + bk, cq = col0 + bc;
        cp_quad(&S.rb[e * 4], P.B + kk * P.ldb + cq, kk < P.k, P.n - cq);
      } else {
        const int bc = e / (BK / 4), bk = (e % (BK / 4)) * 4;
        const int64_t kq = k0 + bk, cc = col0 + bc;
        cp_quad(&S.rb[e * 4], P.B + cc * P.ldb + kq, cc < P.n, P.k - kq);
      }
    }
    asm volatile("cp.async.commit_group;");
  };
  auto decode_tile = [&](int buf, int64_t k0) -> uint32_t {
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    uint32_t sp = 0u;
#pragma unroll
    for (int h = 0; h < AQ; h++) {
      const int e = tid + h * NTHR;
      if (e >= C::AQN) break;
      if (!P.transa) {
        const int ar = e / (BK / 4), ak = (e % (BK / 4)) * 4;
        const bool rok = row0 + ar < P.m;
        const int64_t av = P.k - (k0 + ak);
#pragma unroll
        for (int q = 0; q < 4; q++)
          S.a[buf][ak + q][ar] = sv<typename C::SV>(stage_decode<31, WM, SOFF>((rok && q < av) ? S.ra[e * 4 + q] : p32::ONE, 0u, sp));
      } else {
        const int ak = e / (BM / 4), ar = (e % (BM / 4)) * 4;
        const bool rok = k0 + ak < P.k;
        const int64_t av = P.m - (row0 + ar);
#pragma unroll
        for (int q = 0; q < 4; q++)
          S.a[buf][ak][ar + q] = sv<typename C::SV>(stage_decode<31, WM, SOFF>((rok && q < av) ? S.ra[e * 4 + q] : p32::ONE, 0u, sp));
      }
    }
#pragma unroll
    for (int h = 0; h < BQ; h++) {
      const int e = tid + h * NTHR;
      if (e >= C::BQN) break;
      if (!TRANS_B) {
        const int bk = e / (BN / 4), bc = (e % (BN / 4)) * 4;
        const bool rok = k0 + bk < P.k;
        const int64_t av = P.n - (col0 + bc);
#pragma unroll
        for (int q = 0; q < 4; q++)
          S.b[buf][bk][bc + q] = sv<typename C::SV>(stage_decode<30, WM, SOFF>((rok && q < av) ? S.rb[e * 4 + q] : p32::ONE, flip, sp, K.tp0));
      } else {
        const int bc = e / (BK / 4), bk = (e % (BK / 4)) * 4;
        const bool rok = col0 + bc < P.n;
        const int64_t av = P.k - (k0 + bk);
#pragma unroll
        for (int q = 0; q < 4; q++)
          S.b[buf][bk + q][bc] = sv<typename C::SV>(stage_decode<30, WM, SOFF>((rok && q < av) ? S.rb[e * 4 + q] : p32::ONE, flip, sp, K.tp0));
      }
    }
    return sp;
  };
#endif

  const int64_t ntiles = (P.k + BK - 1) / BK;
#if PG_CPASYNC
  if (ntiles > 0) issue_tile(0);
  int special = ntiles > 0 ? __syncthreads_or((int)decode_tile(0, 0)) : 0;
#else
  if (ntiles > 0) {
    load_tile(0);
  }
  int special = ntiles > 0 ? __syncthreads_or((int)store_tile(0)) : 0;
#endif

  for (int64_t t = 0; t < ntiles; t++) {
    const int cur = (int)(t & 1);
    const int64_t k0 = t * BK;
#if PG_CPASYNC
    if (t + 1 < ntiles) issue_tile(k0 + BK);
#else
    if (t + 1 < ntiles) load_tile(k0 + BK);
#endif
    const int kmax = (int)min((int64_t)BK, P.k - k0);
    if (!special) {
      // the accumulators must start the slab within the range that keeps every
      // MAC of the slab exact (E_ACC_SLAB, see mac); clamp for the table bounds
#pragma unroll
      for (int i = 0; i < TM; i++)
#pragma unroll
        for (int j = 0; j < TN; j++) {
          bad = bad | (acc[i][j].E > E_ACC_SLAB);
          acc[i][j].E = min(acc[i][j].E, E_CLAMP);
        }
      if (kmax == BK) {
#pragma unroll (SYRK ? KK_UNROLL_SYRK : KK_UNROLL)
        for (int kk = 0; kk < BK; kk++) {
          typename C::SV av[TM], bv[TN];
#pragma unroll
          for (int i = 0; i < TM; i++) av[i] = S.a[cur][kk][ty * TM + i];
#pragma unroll
          for (int j = 0; j < TN; j++) bv[j] = S.b[cur][kk][tx * TN + j];
#pragma unroll
          for (int i = 0; i < TM; i++)
#pragma unroll
            for (int j = 0; j < TN; j++)
              mac<MacConst, false, PG_PRESCALED != 0, PBS, CEM, PIX, PIXS, MSL>(acc[i][j], av[i].x, sv_E(av[i]), sv_s(av[i]), bv[j].x,
                                                                sv_E(bv[j]), sv_s(bv[j]), K, badacc, sv_w(av[i]), sv_w(bv[j]));
        }
      } else {
        for (int kk = 0; kk < kmax; kk++) {
          typename C::SV av[TM], bv[TN];
#pragma unroll
          for (int i = 0; i < TM; i++) av[i] = S.a[cur][kk][ty * TM + i];
#pragma unroll
          for (int j = 0; j < TN; j++) bv[j] = S.b[cur][kk][tx * TN + j];
#pragma unroll
          for (int i = 0; i < TM; i++)
#pragma unroll
            for (int j = 0; j < TN; j++)
              mac<MacConst, false, PG_PRESCALED != 0, PBS, CEM, PIX, PIXS, MSL>(acc[i][j], av[i].x, sv_E(av[i]), sv_s(av[i]), bv[j].x,
                                                                sv_E(bv[j]), sv_s(bv[j]), K, badacc, sv_w(av[i]), sv_w(bv[j]));
        }
      }
    } else if (!bad) {
      // generic path for this k-slab (a zero / NaR / extreme operand is present)
#pragma unroll
      for (int i = 0; i < TM; i++) {
#pragma unroll
        for (int j = 0; j < TN; j++) {
          const int64_t r = row0 + ty * TM + i, cc = col0 + tx * TN + j;
          if (r < P.m && cc < P.n) {
            const uint4 o = slow_slab(acc[i][j].M, acc[i][j].E, acc[i][j].sg, P.A, P.lda, P.B, P.ldb, P.neg, r, cc,
                                      k0, kmax, TRANS_B ? 1 : 0, P.transa);
            acc[i][j].M = o.x; acc[i][j].E = (int32_t)o.y; acc[i][j].sg = (int32_t)o.z; bad = bad | (o.w != 0u);
          }
        }
      }
    }
#if PG_CPASYNC
    if (t + 1 < ntiles) special = __syncthreads_or((int)decode_tile(cur ^ 1, k0 + BK));
#else
    if (t + 1 < ntiles) special = __syncthreads_or((int)store_tile(cur ^ 1));
#endif
  }

  // ---- epilogue ------------------------------------------------------------
  if (bad) {
    // recompute this thread's outputs from scratch with the generic path
    for (int e = 0; e < TM * TN; e++) {
      const int64_t r = row0 + ty * TM + e / TN, cc = col0 + tx * TN + e % TN;
      if (r < P.m && cc < P.n && (!SYRK || cc <= r)) P.C[r * P.ldc + cc] = slow_chain(P.A, P.lda, P.B, P.ldb, P.C, P.ldc, P.beta, P.neg, P.k, r, cc, TRANS_B ? 1 : 0,
                                            P.transa);
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < TM; i++) {
#pragma unroll
    for (int j = 0; j < TN; j++) {
      const int64_t r = row0 + ty * TM + i, cc = col0 + tx * TN + j;
      if (r < P.m && cc < P.n && (!SYRK || cc <= r)) P.C[r * P.ldc + cc] = acc_encode(acc[i][j]);
    }
  }
}

// Naive reference kernel: one thread per output, generic per-operation path.
__global__ void k_gemm_naive(Params P, int transb, int syrk) {
  const int64_t cc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = blockIdx.y;
  if (r >= P.m || cc >= P.n || (syrk && cc > r)) return;
  if (P.stop != nullptr && *P.stop != 0) return;
  uint32_t c = P.beta ? P.C[r * P.ldc + cc] : 0u;
  for (int64_t l = 0; l < P.k; l++) {
    const uint32_t a = P.transa ? P.A[l * P.lda + r] : P.A[r * P.lda + l];
    const uint32_t b = transb ? P.B[cc * P.ldb + l] : P.B[l * P.ldb + cc];
    c = mac_generic(c, a, b, P.neg);
  }
  P.C[r * P.ldc + cc] = c;
}

}  // namespace pg

// ---- launchers (called from capi.cu) ----------------------------------------
namespace {
// Tile configurations: 4 x 2 accumulators per thread (64 registers), so 32
// warps are resident per SM -- more warps hide the pipe contention of the
// MAC's integer stream better than a 4 x 4 tile's extra ILP (r05g-r05i, r05q:
// C2 1171 -> 1200 Gflop/s, SYRK 1165 -> 1179; 2 x 4 per thread ~1020, 4 x 8
// per thread 893).
using G1 = pg::Cfg<64, 128, 4, 2, 1, 100>;   // 1024 thr, 1 CTA / SM (the GEMM default)
using G2 = pg::Cfg<64, 64, 4, 2, 2, 99>;     // 512 thr, 2 CTAs / SM (the SYRK default)
using G3 = pg::Cfg<32, 128, 4, 2, 2, 99>;    // 512 thr, 2 CTAs / SM, short-and-wide (LU TRSM updates)
using G4 = pg::Cfg<128, 32, 4, 2, 2, 99>;    // 512 thr, 2 CTAs / SM, tall-and-narrow (Cholesky TRSM updates)

template <class C>
int launch_cfg(const pg::Params& P, bool transb, bool syrk, cudaStream_t st, bool pdl = false) {
  const dim3 grid((unsigned)((P.n + C::BN - 1) / C::BN), (unsigned)((P.m + C::BM - 1) / C::BM));
  if (grid.y > 65535u) return PB_ERR_TOO_LARGE;
  const size_t smem = sizeof(typename C::Smem);
  auto kern = transb ? (syrk ? pg::k_gemm<C, true, true> : pg::k_gemm<C, true, false>)
                     : (syrk ? pg::k_gemm<C, false, true> : pg::k_gemm<C, false, false>);
  static PbOncePerDevice attrs;                // one-time init per device, all four instantiations
  pb_once_per_device(attrs, [smem] {
    cudaFuncSetAttribute(pg::k_gemm<C, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(pg::k_gemm<C, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(pg::k_gemm<C, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(pg::k_gemm<C, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  pb_count_launch();
  if (pdl) {
    // programmatic dependent launch: this grid may start while the previous
    // kernel on the stream (which triggers at entry) runs its last wave; only
    // for launches that do not read that kernel's output
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(C::NTHR);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, P) == cudaSuccess) return 0;
    (void)cudaGetLastError();
  }
  kern<<<grid, C::NTHR, smem, st>>>(P);
  return 0;
}

int variant() {
  static const int v = [] {
    const char* e = getenv("POSIT_GEMM_VARIANT");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// Modelled time of a launch with config C: the busiest SM runs ceil(tiles /
// SMs) CTAs of NTHR x 16 accumulators each; an SM with 512 resident threads
// issues at the full rate, one with only 256 (a lone small CTA) at ~2/3 of it
// (measured: tools/tune_gemm.py, tall-narrow and short-wide trailing shapes).
template <class C>
double model_time(int64_t m, int64_t n, bool syrk, int64_t nsm) {
  const int64_t rb = (m + C::BM - 1) / C::BM, cb = (n + C::BN - 1) / C::BN;
  int64_t tiles = rb * cb;
  if (syrk) tiles = tiles / 2 + rb;                       // lower-triangle tiles (approx.)
  const int64_t per_sm = (tiles + nsm - 1) / nsm;
  const int64_t resident = (per_sm < C::MINB ? per_sm : C::MINB) * C::NTHR;
  const double rate = (resident >= 512 ? 1.0 : 0.66) * C::EFF;
  return (double)per_sm * C::BM * C::BN / rate;
}
}  // namespace

// Picks the tile shape with the smallest modelled time for this problem;
// near-ties (within 10%) go to the 64 x 128 tile.  All configurations compute the same
// bits (same per-element order), so the choice is performance only.
static int64_t tiny_outputs() {
  static const int64_t v = [] {
    const char* e = getenv("POSIT_TINY_OUTPUTS");
    return e ? (int64_t)atoll(e) : (int64_t)65536;
  }();
  return v;
}

int pb_launch_gemm(const pg::Params& P, bool transb, bool syrk, cudaStream_t st, bool pdl) {
  if (P.m == 0 || P.n == 0) return 0;
  static const int pdl_env = [] {
    const char* e = getenv("POSIT_PDL");
    return e ? atoi(e) : 1;
  }();
  pdl = pdl && pdl_env != 0;
  // tiny shapes (the panel-internal updates): one thread per output
  static const int tiny_env = [] {
    const char* e = getenv("POSIT_GEMM_TINY");
    return e ? atoi(e) : 1;
  }();
  if (tiny_env && P.k >= 1 && P.k <= 64 && P.m <= 128 && P.n <= 128) return pb_launch_gemm_tiny(P, transb, syrk, st);
  // few outputs and a short K (the panel recursion at small heights): the tiled kernel would run a few
  // CTAs with long per-thread loops (480 x 32 x 32: 54 us), one chain per output is shorter
  if (tiny_env && P.k >= 1 && P.k <= 128 && P.m * P.n <= tiny_outputs()) return pb_launch_gemm_tiny(P, transb, syrk, st);
  // tall and skinny with a short K (the panel recursion's innermost updates, m x 32 x 32): a 64-column tile
  // would idle half its threads on one row of CTAs
  if (tiny_env == 2 && P.k >= 1 && P.k <= 32 && P.n <= 32 && !syrk) return pb_launch_gemm_tiny(P, transb, syrk, st);
  int v = variant();
  // the binary64-pipe MAC (gemm_d.cu) unless POSIT_GEMM_PATH=0 or an integer-MAC tile is forced (11..14)
  if ((pb_dpath() && v == 0) || v >= 21) return pb_launch_gemm_d(P, transb, syrk, st, pdl, v);
  if (v == 0) {
    // the smallest modelled time; near-ties (within 10%) go to the first candidate
    auto pick = [&](int v0, double w0, std::initializer_list<std::pair<int, double>> rest) {
      int vb = v0;
      double best = w0;
      for (const auto& c : rest)
        if (c.second < best * 0.9) { vb = c.first; best = c.second; }
      return vb;
    };
    const int base = syrk ? 12 : 11;
    const int64_t ns = pb_num_sms();
    v = pick(base, base == 12 ? model_time<G2>(P.m, P.n, syrk, ns) : model_time<G1>(P.m, P.n, syrk, ns),
             {{base == 12 ? 11 : 12, base == 12 ? model_time<G1>(P.m, P.n, syrk, ns) : model_time<G2>(P.m, P.n, syrk, ns)},
              {13, model_time<G3>(P.m, P.n, syrk, ns)}, {14, model_time<G4>(P.m, P.n, syrk, ns)}});
  }
  switch (v) {
    case 12: return launch_cfg<G2>(P, transb, syrk, st, pdl);
    case 13: return launch_cfg<G3>(P, transb, syrk, st, pdl);
    case 14: return launch_cfg<G4>(P, transb, syrk, st, pdl);
    default: return launch_cfg<G1>(P, transb, syrk, st, pdl);
  }
}

int pb_launch_gemm_naive(const pg::Params& P, bool transb, bool syrk, cudaStream_t st) {
  if (P.m == 0 || P.n == 0) return 0;
  const dim3 grid((unsigned)((P.n + 127) / 128), (unsigned)P.m);
  if (P.m > 65535) return PB_ERR_TOO_LARGE;
  pb_count_launch();
  pg::k_gemm_naive<<<grid, 128, 0, st>>>(P, transb ? 1 : 0, syrk ? 1 : 0);
  return 0;
}
