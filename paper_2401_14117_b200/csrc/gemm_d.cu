// gemm_d.cu -- Posit(32,2) GEMM (NN, NT, TN, TT) and SYRK-lower on the
// binary64 pipe (the D-MAC of gemm_d.cuh) + launcher.
//
// Same tiling as k_gemm (gemm.cu): a CTA owns BM x BN outputs, each thread a
// TM x TN register tile; k-slabs of 16 are copied raw into shared memory with
// cp.async while the previous slab computes, then decoded ONCE per staged
// element into its exact binary64 value (8 bytes instead of the integer
// MAC's 16-byte decoded form).  A slab with a zero, NaR or |scale| > 37
// operand runs the generic per-operation path for the whole CTA; a thread
// whose accumulator starts a slab above scale 91 recomputes its outputs with
// the generic path (same bits: the order contract, Q6).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <initializer_list>
#include <utility>
#include "gemm.cuh"
#include "gemm_common.cuh"
#include "gemm_d.cuh"
#include "lanes_d.cuh"
#include "internal.h"

#ifndef PGD_KK_UNROLL
#define PGD_KK_UNROLL 4
#endif

namespace pg {

constexpr int KK_UNROLL_D = PGD_KK_UNROLL;
// k-slab depth (one CTA barrier and one special-operand check per slab).  r2q1 A/B: with one
// 1024-thread CTA per SM (D1) a barrier idles the SM, and 32-deep slabs gain (C2 2802 -> 2903
// Gflop/s, C4 1126.7 -> 1092.5 ms); with two 512-thread CTAs per SM (D2..D4, the SYRK's tiles) the
// other CTA covers the barrier and 16 stays ahead (C3 83.5 vs 84.4 ms).
#ifndef PGD_BK
#define PGD_BK 32                    // tiles with one CTA per SM
#endif
#ifndef PGD_BK2
#define PGD_BK2 16                   // tiles with two CTAs per SM
#endif
static_assert(PGD_BK % 4 == 0 && PGD_BK2 % 4 == 0 && 107 - PGD_BK <= E_ACC_SLAB && 107 - PGD_BK2 <= E_ACC_SLAB,
              "slab depth");

template <int BM_, int BN_, int TM_, int TN_, int MINB_, int EFF100 = 100>
struct CfgD {
  static constexpr int BM = BM_, BN = BN_, TM = TM_, TN = TN_, BK = MINB_ == 1 ? PGD_BK : PGD_BK2, MINB = MINB_;
  // accumulator |E| limit at a slab start: one MAC raises |E| by at most 1 and the sum needs |E| <= 107
  static constexpr int E_SLAB = 107 - BK;
  static constexpr double EFF = EFF100 / 100.0;
  static constexpr int NTX = BN / TN, NTY = BM / TM, NTHR = NTX * NTY;
  static constexpr int AQN = BM * BK / 4, BQN = BN * BK / 4;
  struct Smem {
    double a[2][BK][BM];
    double b[2][BK][BN];
    uint32_t ra[BM * BK];             // raw patterns of the next slab (cp.async target, by quad)
    uint32_t rb[BK * BN];
    pgd::dtab_tt<pgd::T64_GEMM> tab[pgd::DT_SIZE];    // M(E) by biased exponent
  };
};

template <class C, bool TRANS_B, bool SYRK>
__global__ void __launch_bounds__(C::NTHR, C::MINB) k_gemm_d(Params P) {
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, TM = C::TM, TN = C::TN, NTHR = C::NTHR;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  typename C::Smem& S = *reinterpret_cast<typename C::Smem*>(smem_raw);

  const int tid = threadIdx.x;
  const int tx = tid % C::NTX;
  const int ty = tid / C::NTX;
  // grouped rasterisation (as k_gemm): a wave re-reads its A rows and B columns from L2
  const int64_t nbn = gridDim.x, nbm = gridDim.y;
  const int64_t pid = (int64_t)blockIdx.y * nbn + blockIdx.x;
  const int64_t per_group = (int64_t)32 * nbn;
  const int64_t gfirst = (pid / per_group) * 32;
  const int64_t gsize = (nbm - gfirst) < 32 ? (nbm - gfirst) : 32;
  const int64_t row0 = (gfirst + (pid % per_group) % gsize) * BM;
  const int64_t col0 = ((pid % per_group) / gsize) * BN;
  asm volatile("griddepcontrol.launch_dependents;");
  if (SYRK && col0 > row0 + BM - 1) return;
  if (P.stop != nullptr && *P.stop != 0) return;

  const uint32_t flip = P.neg ? 1u : 0u;
  for (int i = tid; i < pgd::DT_SIZE; i += NTHR) S.tab[i] = pgd::dtab_fill<pgd::T64_GEMM>(i);   // visible after the first barrier
  const uint32_t tab0 = (uint32_t)__cvta_generic_to_shared(S.tab);

  double acc[TM][TN];
  bool bad = false;
#pragma unroll
  for (int i = 0; i < TM; i++)
#pragma unroll
    for (int j = 0; j < TN; j++) {
      const int64_t r = row0 + ty * TM + i, cc = col0 + tx * TN + j;
      uint32_t cv = 0u;
      if (P.beta && r < P.m && cc < P.n) cv = P.C[r * P.ldc + cc];
      if (!pgd::d_decode(cv, acc[i][j])) bad = true;
    }

  auto issue_tile = [&](int64_t k0) {
    for (int e = tid; e < C::AQN; e += NTHR) {
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
    for (int e = tid; e < C::BQN; e += NTHR) {
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
    for (int e = tid; e < C::AQN; e += NTHR) {
      if (!P.transa) {
        const int ar = e / (BK / 4), ak = (e % (BK / 4)) * 4;
        const bool rok = row0 + ar < P.m;
        const int64_t av = P.k - (k0 + ak);
#pragma unroll
        for (int q = 0; q < 4; q++)
          S.a[buf][ak + q][ar] = pgd::stage_decode_d((rok && q < av) ? S.ra[e * 4 + q] : p32::ONE, 0u, sp);
      } else {
        const int ak = e / (BM / 4), ar = (e % (BM / 4)) * 4;
        const bool rok = k0 + ak < P.k;
        const int64_t av = P.m - (row0 + ar);
#pragma unroll
        for (int q = 0; q < 4; q++)
          S.a[buf][ak][ar + q] = pgd::stage_decode_d((rok && q < av) ? S.ra[e * 4 + q] : p32::ONE, 0u, sp);
      }
    }
    for (int e = tid; e < C::BQN; e += NTHR) {
      if (!TRANS_B) {
        const int bk = e / (BN / 4), bc = (e % (BN / 4)) * 4;
        const bool rok = k0 + bk < P.k;
        const int64_t av = P.n - (col0 + bc);
#pragma unroll
        for (int q = 0; q < 4; q++)
          S.b[buf][bk][bc + q] = pgd::stage_decode_d((rok && q < av) ? S.rb[e * 4 + q] : p32::ONE, flip, sp);
      } else {
        const int bc = e / (BK / 4), bk = (e % (BK / 4)) * 4;
        const bool rok = col0 + bc < P.n;
        const int64_t av = P.k - (k0 + bk);
#pragma unroll
        for (int q = 0; q < 4; q++)
          S.b[buf][bk + q][bc] = pgd::stage_decode_d((rok && q < av) ? S.rb[e * 4 + q] : p32::ONE, flip, sp);
      }
    }
    return sp;
  };

  const int64_t ntiles = (P.k + BK - 1) / BK;
  if (ntiles > 0) issue_tile(0);
  int special = ntiles > 0 ? __syncthreads_or((int)decode_tile(0, 0)) : 0;

  for (int64_t t = 0; t < ntiles; t++) {
    const int cur = (int)(t & 1);
    const int64_t k0 = t * BK;
    if (t + 1 < ntiles) issue_tile(k0 + BK);
    const int kmax = (int)min((int64_t)BK, P.k - k0);
    if (!special) {
#pragma unroll
      for (int i = 0; i < TM; i++)
#pragma unroll
        for (int j = 0; j < TN; j++) bad = bad | pgd::d_above(acc[i][j], C::E_SLAB);
      if (kmax == BK) {
#pragma unroll KK_UNROLL_D
        for (int kk = 0; kk < BK; kk++) {
          double av[TM], bv[TN];
#pragma unroll
          for (int i = 0; i < TM; i++) av[i] = S.a[cur][kk][ty * TM + i];
#pragma unroll
          for (int j = 0; j < TN; j++) bv[j] = S.b[cur][kk][tx * TN + j];
#pragma unroll
          for (int i = 0; i < TM; i++)
#pragma unroll
            for (int j = 0; j < TN; j++) acc[i][j] = pgd::dmac<pgd::T64_GEMM>(acc[i][j], av[i], bv[j], tab0);
        }
      } else {
        for (int kk = 0; kk < kmax; kk++) {
          double av[TM], bv[TN];
#pragma unroll
          for (int i = 0; i < TM; i++) av[i] = S.a[cur][kk][ty * TM + i];
#pragma unroll
          for (int j = 0; j < TN; j++) bv[j] = S.b[cur][kk][tx * TN + j];
#pragma unroll
          for (int i = 0; i < TM; i++)
#pragma unroll
            for (int j = 0; j < TN; j++) acc[i][j] = pgd::dmac<pgd::T64_GEMM>(acc[i][j], av[i], bv[j], tab0);
        }
      }
    } else if (!bad) {
      // generic path for this k-slab (a zero / NaR / extreme operand is present)
#pragma unroll
      for (int i = 0; i < TM; i++)
#pragma unroll
        for (int j = 0; j < TN; j++) {
          const int64_t r = row0 + ty * TM + i, cc = col0 + tx * TN + j;
          if (r < P.m && cc < P.n) {
            uint32_t c = pgd::d_encode(acc[i][j]);
            for (int kk = 0; kk < kmax; kk++) {
              const int64_t l = k0 + kk;
              const uint32_t a = P.transa ? P.A[l * P.lda + r] : P.A[r * P.lda + l];
              const uint32_t b = TRANS_B ? P.B[cc * P.ldb + l] : P.B[l * P.ldb + cc];
              c = mac_generic(c, a, b, P.neg);
            }
            if (!pgd::d_decode(c, acc[i][j])) bad = true;
          }
        }
    }
    if (t + 1 < ntiles) special = __syncthreads_or((int)decode_tile(cur ^ 1, k0 + BK));
  }

  if (bad) {
    for (int e = 0; e < TM * TN; e++) {
      const int64_t r = row0 + ty * TM + e / TN, cc = col0 + tx * TN + e % TN;
      if (r < P.m && cc < P.n && (!SYRK || cc <= r))
        P.C[r * P.ldc + cc] = slow_chain(P.A, P.lda, P.B, P.ldb, P.C, P.ldc, P.beta, P.neg, P.k, r, cc,
                                         TRANS_B ? 1 : 0, P.transa);
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < TM; i++)
#pragma unroll
    for (int j = 0; j < TN; j++) {
      const int64_t r = row0 + ty * TM + i, cc = col0 + tx * TN + j;
      if (r < P.m && cc < P.n && (!SYRK || cc <= r)) P.C[r * P.ldc + cc] = pgd::d_encode(acc[i][j]);
    }
}

// Elementwise D-MAC checks (posit_vec_op POSIT_OP_DADD / DMUL / DMAC): the
// binary64-pipe add, mul and fused-order MAC on single operations, for
// operands inside their fast range; outside it the generic ops (same bits).
__global__ void k_vec_d(int op, const uint32_t* a, const uint32_t* b, const uint32_t* c, uint32_t* out,
                        int64_t count) {
  __shared__ pgd::dtab_tt<pgd::T64_GEMM> tab[pgd::DT_SIZE];
  for (int i = threadIdx.x; i < pgd::DT_SIZE; i += blockDim.x) tab[i] = pgd::dtab_fill<pgd::T64_GEMM>(i);
  __syncthreads();
  const uint32_t tab0 = (uint32_t)__cvta_generic_to_shared(tab);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t x = a[i], y = b[i];
    uint32_t sp = 0u;
    uint32_t r;
    if (op == POSIT_OP_DMUL) {
      const double da = pgd::stage_decode_d(x, 0u, sp), db = pgd::stage_decode_d(y, 0u, sp);
      r = sp ? p32::mul(x, y) : pgd::d_encode(pgd::dmul_pos<pgd::T64_GEMM>(da, db, tab0));
    } else if (op == POSIT_OP_DADD) {
      // sum of two values of |E| <= 75 (a product's range): the D-MAC's sum step
      const double da = pgd::stage_decode_d<75>(x, 0u, sp), db = pgd::stage_decode_d<75>(y, 0u, sp);
      r = sp ? p32::add(x, y) : pgd::d_encode(pgd::dadd_pos<pgd::T64_GEMM>(da, db, tab0));
    } else if (op == POSIT_OP_DDIV) {
      // a (/) b by the D-MAC division (dividend |E| <= 91, divisor a fast operand), else the generic div
      double da, q;
      const bool aok = pgd::d_decode(x, da) && !pgd::d_above(da, E_ACC_SLAB);
      const double db = pgd::stage_decode_d(y, 0u, sp);
      r = (aok && !sp && pld::div_r(da, db, __drcp_rn(db), q)) ? pgd::d_encode(q) : p32::div(x, y);
    } else if (op == POSIT_OP_DSQRT) {
      // sqrt(a) by the D-MAC square root (a > 0, |E| <= 75), else the generic sqrt
      double da;
      const bool aok = pgd::d_decode(x, da) && pld::in_lane_range(da) && da > 0.0;
      r = aok ? pgd::d_encode(pld::sqrt_r(da)) : p32::sqrt(x);
    } else {
      // out = c (+) (a (x) b) with |Ea|, |Eb| <= 37 and |Ec| <= 91
      double dc;
      const double da = pgd::stage_decode_d(x, 0u, sp), db = pgd::stage_decode_d(y, 0u, sp);
      const bool cok = pgd::d_decode(c[i], dc) && !pgd::d_above(dc, E_ACC_SLAB);
      r = (sp || !cok) ? p32::add(c[i], p32::mul(x, y)) : pgd::d_encode(pgd::dmac<pgd::T64_GEMM>(dc, da, db, tab0));
    }
    out[i] = r;
  }
}

}  // namespace pg

namespace {
using D1 = pg::CfgD<64, 128, 4, 2, 1, 100>;   // 1024 threads, 1 CTA / SM (the GEMM default)
using D2 = pg::CfgD<64, 64, 4, 2, 2, 99>;     // 512 threads, 2 CTAs / SM (SYRK, small shapes)
using D3 = pg::CfgD<32, 128, 4, 2, 2, 99>;    // 512 threads, short-and-wide
using D4 = pg::CfgD<128, 32, 4, 2, 2, 99>;    // 512 threads, tall-and-narrow

template <class C>
int launch_cfg_d(const pg::Params& P, bool transb, bool syrk, cudaStream_t st, bool pdl) {
  const dim3 grid((unsigned)((P.n + C::BN - 1) / C::BN), (unsigned)((P.m + C::BM - 1) / C::BM));
  if (grid.y > 65535u) return PB_ERR_TOO_LARGE;
  const size_t smem = sizeof(typename C::Smem);
  auto kern = transb ? (syrk ? pg::k_gemm_d<C, true, true> : pg::k_gemm_d<C, true, false>)
                     : (syrk ? pg::k_gemm_d<C, false, true> : pg::k_gemm_d<C, false, false>);
  static PbOncePerDevice attrs;
  pb_once_per_device(attrs, [smem] {
    cudaFuncSetAttribute(pg::k_gemm_d<C, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(pg::k_gemm_d<C, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(pg::k_gemm_d<C, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(pg::k_gemm_d<C, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  pb_count_launch();
  if (pdl) {
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

template <class C>
double model_time_d(int64_t m, int64_t n, bool syrk, int64_t nsm) {
  const int64_t rb = (m + C::BM - 1) / C::BM, cb = (n + C::BN - 1) / C::BN;
  int64_t tiles = rb * cb;
  if (syrk) tiles = tiles / 2 + rb;
  const int64_t per_sm = (tiles + nsm - 1) / nsm;
  const int64_t resident = (per_sm < C::MINB ? per_sm : C::MINB) * C::NTHR;
  const double rate = (resident >= 512 ? 1.0 : 0.66) * C::EFF;
  return (double)per_sm * C::BM * C::BN / rate;
}
}  // namespace

// variant: 0 = modelled best, 21..24 = D1..D4
int pb_launch_gemm_d(const pg::Params& P, bool transb, bool syrk, cudaStream_t st, bool pdl, int v) {
  if (v == 0) {
    const int64_t ns = pb_num_sms();
    const int base = syrk ? 22 : 21;
    double best = base == 22 ? model_time_d<D2>(P.m, P.n, syrk, ns) : model_time_d<D1>(P.m, P.n, syrk, ns);
    v = base;
    const std::pair<int, double> rest[] = {
        {base == 22 ? 21 : 22, base == 22 ? model_time_d<D1>(P.m, P.n, syrk, ns) : model_time_d<D2>(P.m, P.n, syrk, ns)},
        {23, model_time_d<D3>(P.m, P.n, syrk, ns)},
        {24, model_time_d<D4>(P.m, P.n, syrk, ns)}};
    for (const auto& c : rest)
      if (c.second < best * 0.9) { v = c.first; best = c.second; }
  }
  switch (v) {
    case 22: return launch_cfg_d<D2>(P, transb, syrk, st, pdl);
    case 23: return launch_cfg_d<D3>(P, transb, syrk, st, pdl);
    case 24: return launch_cfg_d<D4>(P, transb, syrk, st, pdl);
    default: return launch_cfg_d<D1>(P, transb, syrk, st, pdl);
  }
}

int pb_vec_d(int op, const uint32_t* a, const uint32_t* b, const uint32_t* c, uint32_t* out, int64_t count,
             cudaStream_t st) {
  if (count <= 0) return 0;
  pb_count_launch();
  int64_t blocks = (count + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  pg::k_vec_d<<<(unsigned)blocks, 256, 0, st>>>(op, a, b, c, out, count);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : POSIT_ECUDA;
}
