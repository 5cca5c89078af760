// chol.cu -- the diagonal-block Cholesky (potf2) and the
// tiny one-thread-per-output GEMM / SYRK it and the LU panel use.
#include "lanes.cuh"
#include "lanes_d.cuh"

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

// ---- the whole <= 256 x 256 diagonal block in ONE launch: a thread-block cluster --
// Textbook right-looking loop (reading Q9) over all b columns, the lower
// triangle distributed over the NC CTAs of one cluster (distributed shared
// memory; a cluster barrier costs ~0.2 us, a kernel launch or grid sync
// several): CTA c owns rows i = w NC + c, one row per warp w, lane l holds
// columns j = l + 32 q (q < 8) of its row, decoded in registers for the whole
// loop -- so the lower-triangle mask is nearly warp-uniform.
// Iteration k: (1) thread k applies column k-1 to its copy of the diagonal
// chain d_k (every CTA keeps all of them, thread j holding d_j: d_j <- d_j (-)
// l_jk (x) l_jk, the operations of the element a_jj in its order, hence its
// bits) and takes l_kk = sqrt(d_k), published in shared memory with a step
// flag; (2) every thread applies column k-1 to its own elements (ascending k
// per element: Q6); (3) lane k % 32 of every row warp divides its column-k
// element by l_kk (one posit division) and pushes it into the column buffer of
// every CTA; (4) one split cluster barrier per column.  A non-positive d_k
// stops every CTA at the same step (info = row_base + k + 1, every step < k
// applied, as the oracle's loop).
constexpr int PC_Q = 8;                        // column slots per lane
constexpr int PC_B = 256;                      // largest block

struct PcSmem {
  uint32_t colp[2][PC_B];                      // column k: patterns l_jk (rows j > k)
  uint4 cola[2][PC_B];                         // A-format decode {M, E, sigma, fast}
  uint4 colb[2][PC_B];                         // B-format decode {M, E, sg, fast}
  int fail;
  int lkk_step;                                // the step whose l_kk is in lkk
  uint32_t lkk;
  uint4 tp[pg::TSIZE], tx[pg::TSIZE];          // the MAC's per-scale constant tables
};

// A LaneVal in three registers: decoded {M, E, sg}, or the pattern in M with
// E = PC_PAT when the value is outside the fast range.
constexpr int32_t PC_PAT = 0x40000000;
struct PcVal { uint32_t M; int32_t E; int32_t sg; };

__device__ __forceinline__ PcVal pc_of(const LaneVal& v) {
  return v.dec ? PcVal{v.a.M, v.a.E, v.a.sg} : PcVal{v.pat, PC_PAT, 1};
}
__device__ __forceinline__ LaneVal pc_lane(const PcVal& x) {
  LaneVal v;
  v.dec = x.E != PC_PAT;
  v.a = pg::Acc{x.M, x.E, x.sg};
  v.pat = x.M;
  return v;
}
__device__ __forceinline__ PcVal pc_load(uint32_t x) {
  LaneVal t;
  lv_load(t, x);
  return pc_of(t);
}

// x <- x (-) l_ik (x) l_jk with the column buffer's entries (fast MAC, generic fallback)
__device__ __forceinline__ void pc_fms(PcVal& x, const PcSmem& S, int q, int i, int j, const pg::MacConst& K) {
  const uint4 ad = S.cola[q][i], bd = S.colb[q][j];
  LaneVal t = pc_lane(x);
  lv_fms_t(t, S.colp[q][i], ad.w != 0u, ad, bd.x, (int32_t)bd.y, (int32_t)bd.z, bd.w != 0u, S.colp[q][j], K);
  x = pc_of(t);
}

__device__ __forceinline__ void pc_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void pc_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }

template <int NC>
__global__ void __launch_bounds__(32 * (PC_B / NC), 1)
    k_potf2_cluster(uint32_t* A, int64_t lda, int b, int32_t* info, int64_t row_base) {
  namespace cg = cooperative_groups;
  constexpr int NT = 32 * (PC_B / NC);                          // one warp per row of this CTA
  __shared__ PcSmem S;
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int i = w * NC + c;                                     // my row
  if (*info != 0) return;                                       // an earlier block failed: every CTA returns
  pg::fill_tables(S.tp, S.tx, tid, NT);
  pg::MacConst K;
  K.one = 1u; K.sixteen = 16u;
  K.tp0 = (uint32_t)__cvta_generic_to_shared(S.tp + pg::TBIAS);
  K.tx0 = (uint32_t)__cvta_generic_to_shared(S.tx + pg::TBIAS) - 30u * 16u;
  if (tid == 0) { S.fail = 0; S.lkk_step = -1; }
  PcVal v[PC_Q];
#pragma unroll
  for (int q = 0; q < PC_Q; q++) {
    const int j = l + 32 * q;
    v[q] = pc_load((i < b && j <= i) ? A[(int64_t)i * lda + j] : 0u);
  }
  PcVal dd = pc_load(tid < b ? A[(int64_t)tid * lda + tid] : 0u);   // d_j, j = tid
  __syncthreads();
  cl.sync();                                                    // every CTA running before any remote store
  volatile int* vstep = &S.lkk_step;
  bool failed = false;
  for (int k = 0; k < b; k++) {
    const int qk = k & 1, qp = qk ^ 1;
    if (k > 0) {
      pc_wait();                                                // column k - 1 published everywhere
      if (S.fail) { failed = true; break; }                     // same step in every CTA: barriers stay balanced
    }
    // (1) the diagonal chain and l_kk
    if (tid < b && tid >= k) {
      if (k > 0) pc_fms(dd, S, qp, tid, tid, K);
      if (tid == k) {
        const uint32_t dk = lv_pattern(pc_lane(dd));
        if ((int32_t)dk <= 0) {                                 // zero, negative or NaR pivot: stop
          S.fail = 1;
          if (c == 0) *info = (int32_t)(row_base + k + 1);
        } else {
          S.lkk = p32::sqrt(dk);
        }
        __threadfence_block();
        *vstep = k;
      }
    }
    // (2) column k - 1 on my elements (the column-k slot is the first active one)
    if (k > 0 && i < b) {
#pragma unroll
      for (int q = 0; q < PC_Q; q++) {
        const int j = l + 32 * q;
        if (j >= k && j <= i) pc_fms(v[q], S, qp, i, j, K);
      }
    }
    // (3) my row's column-k element: divide by l_kk and publish it to every CTA
    if (l == (k & 31) && i >= k && i < b) {
      while (*vstep != k) { }
      __threadfence_block();
      if (!S.fail) {
        const uint32_t lkk = S.lkk;
        const int qc = k >> 5;
        PcVal xs = v[0];
#pragma unroll
        for (int q = 1; q < PC_Q; q++)
          if (q == qc) xs = v[q];
        LaneVal x = pc_lane(xs);
        if (i == k) {
          lv_load(x, lkk);
        } else {
          pg::Acc dv;
          const bool dok = pg::acc_decode(lkk, dv) && dv.E <= 37 && dv.E >= -37;
          bool done = false;
          if (dok && x.dec) {
            done = pg::acc_div(x.a, dv.M, dv.E, dv.sg, __drcp_rn((double)dv.M) * 4294967296.0, K);
            if (done && !(x.a.E <= 75 && x.a.E >= -75) && x.a.E > pg::E_ZERO_LIMIT) {
              x.pat = pg::acc_encode(x.a);
              x.dec = false;
            }
          }
          if (!done) lv_load(x, div(lv_pattern(x), lkk));
          const uint32_t xp = lv_pattern(x);
          uint4 adx;
          const uint4 av = fast_a(xp, adx) ? make_uint4(adx.x, adx.y, adx.z, 1u) : make_uint4(0u, 0u, 0u, 0u);
          const uint4 bv = lv_operand(x) ? make_uint4(x.a.M, (uint32_t)x.a.E, (uint32_t)x.a.sg, 1u)
                                         : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
          for (int r = 0; r < NC; r++) {                        // push l_ik into every CTA's column buffer
            *cl.map_shared_rank(&S.colp[qk][i], r) = xp;
            *cl.map_shared_rank(&S.cola[qk][i], r) = av;
            *cl.map_shared_rank(&S.colb[qk][i], r) = bv;
          }
        }
        xs = pc_of(x);
#pragma unroll
        for (int q = 0; q < PC_Q; q++)
          if (q == qc) v[q] = xs;
      }
    }
    __syncwarp();
    pc_arrive();                                                // my pushes for column k (release)
  }
  if (!failed) pc_wait();                                       // the last arrive (a failure already waited)
#pragma unroll
  for (int q = 0; q < PC_Q; q++) {
    const int j = l + 32 * q;
    if (i < b && j <= i) A[(int64_t)i * lda + j] = lv_pattern(pc_lane(v[q]));
  }
  cl.sync();                                                    // no CTA exits while others may still read it
}

// The same cluster potf2 with binary64 lane values (lanes_d.cuh): each element
// kept as its exact binary64 value while in the fast range, the column buffer
// holding {binary64 value, fast flag, pattern} (8 + 1 + 4 bytes pushed per
// element instead of 36), the updates on the D-MAC.  The division by l_kk and
// the sqrt stay the integer-path operations (one per element / column).
#ifndef PC_PACKED                               // 1: one 16-byte {binary64, pattern, flag} entry per column element
#define PC_PACKED 1                             //    (one remote store per CTA instead of three, one LDS.128 per operand)
#endif
struct __align__(16) PcCol {
  double d;
  uint32_t p;
  uint32_t f;
};
struct PcSmemD {
#if PC_PACKED
  PcCol col[3][PC_B];                          // column k: l_jk (rows j > k); slot k % 3 (k & 1 if !DEFER)
#else
  uint32_t colp[3][PC_B];                      // column k: patterns l_jk (rows j > k); slot k % 3 (k & 1 if !DEFER)
  double cold[3][PC_B];                        // ... as binary64
  uint8_t colf[3][PC_B];                       // ... fast-operand flags
#endif
  int fail;
  int lkk_step;
  uint32_t lkk;
  int lkfast;                                  // l_kk is a fast operand: lkd, lkr valid (DDIV)
  double lkd, lkr;                             // l_kk as binary64, RN(1 / l_kk)
  uint4 tx[pg::TSIZE];                         // the division's rounding table (integer path)
};

__device__ __forceinline__ void pcd_fms(pld::LD& x, const PcSmemD& S, int q, int i, int j) {
#if PC_PACKED
  const uint4 a = *reinterpret_cast<const uint4*>(&S.col[q][i]), b = *reinterpret_cast<const uint4*>(&S.col[q][j]);
  pld::ld_fms(x, __hiloint2double((int)a.y, (int)a.x), a.w != 0u, a.z, __hiloint2double((int)b.y, (int)b.x), b.w != 0u,
              b.z);
#else
  pld::ld_fms(x, S.cold[q][i], S.colf[q][i] != 0, S.colp[q][i], S.cold[q][j], S.colf[q][j] != 0, S.colp[q][j]);
#endif
}

// push l_ik = {pattern xp, binary64 xd, fast flag xf} into slot q of every CTA's column buffer
template <int NC, class CL>
__device__ __forceinline__ void pcd_push(CL& cl, PcSmemD& S, int q, int i, uint32_t xp, double xd, uint32_t xf) {
#if PC_PACKED
  const uint4 e = make_uint4((uint32_t)__double2loint(xd), (uint32_t)__double2hiint(xd), xp, xf);
#pragma unroll
  for (int r = 0; r < NC; r++) *reinterpret_cast<uint4*>(cl.map_shared_rank(&S.col[q][i], r)) = e;
#else
#pragma unroll
  for (int r = 0; r < NC; r++) {
    *cl.map_shared_rank(&S.colp[q][i], r) = xp;
    *cl.map_shared_rank(&S.cold[q][i], r) = xd;
    *cl.map_shared_rank(&S.colf[q][i], r) = (uint8_t)xf;
  }
#endif
}

//
// DEFER = 1 (POSIT_POTF2_DEFER; 0 is the default): column k's own slot is updated,
// divided and published first; the column k - 1 update of the slots right of it
// runs after the arrive, under the cluster barrier's latency.  Measured slower
// (r2n: 0.895 vs 0.745 ms per 256^2 block): the update was already hidden under
// the diagonal thread's sqrt, and the barrier is short.
//
// DDIV (POSIT_POTF2_DDIV=1): the square root and the divisions on the
// binary64 pipe (pld::sqrt_r, pld::div_r) while d_kk, l_kk and the dividend are
// in the fast range, else the integer-path operations (same bits).  The r2m
// profile of the integer-path kernel: one lane per row warp runs the ~400
// instruction division, 8 warps per scheduler -- issue slots 53 % busy, ALU pipe
// 47 %, FP64 pipe 4 %: the divisions, not the updates, were the column's cost.  Element order is unchanged
// (every element still takes column k - 1 before column k).  The column buffer
// has three slots: a CTA still reads column k - 1 (slot (k - 1) % 3) after its
// arrive of step k, and the next write of that slot is column k + 2's, which
// follows the wait of step k + 2, i.e. every CTA's arrive of step k + 1, i.e.
// the end of every CTA's deferred update of step k.
template <int NC, int DEFER, bool DDIV>
__global__ void __launch_bounds__(32 * (PC_B / NC), 1)
    k_potf2_cluster_d(uint32_t* A, int64_t lda, int b, int32_t* info, int64_t row_base) {
  namespace cg = cooperative_groups;
  constexpr int NT = 32 * (PC_B / NC);
  __shared__ PcSmemD S;
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int i = w * NC + c;
  if (*info != 0) return;
  pg::fill_tables<false, false>(S.tx, S.tx, tid, NT);
  pg::MacConst K;
  K.one = 1u; K.sixteen = 16u;
  K.tp0 = 0u;
  K.tx0 = (uint32_t)__cvta_generic_to_shared(S.tx + pg::TBIAS) - 30u * 16u;
  if (tid == 0) { S.fail = 0; S.lkk_step = -1; }
  pld::LD v[PC_Q];
#pragma unroll
  for (int q = 0; q < PC_Q; q++) {
    const int j = l + 32 * q;
    pld::ld_load(v[q], (i < b && j <= i) ? A[(int64_t)i * lda + j] : 0u);
  }
  pld::LD dd;
  pld::ld_load(dd, tid < b ? A[(int64_t)tid * lda + tid] : 0u);
  __syncthreads();
  cl.sync();
  volatile int* vstep = &S.lkk_step;
  bool failed = false;
  for (int k = 0; k < b; k++) {
    const int qk = DEFER ? k % 3 : (k & 1), qp = DEFER ? (k + 2) % 3 : (qk ^ 1);
    const int qc = k >> 5;
    if (k > 0) {
      pc_wait();
      const int fs = *(volatile int*)&S.fail;                   // failing step + 1; a warp late to this wait
      if (fs != 0 && fs <= k) { failed = true; break; }         // may already see step k's own failure: ignore it here
    }
    if (tid < b && tid >= k) {
      if (k > 0) pcd_fms(dd, S, qp, tid, tid);
      if (tid == k) {
        const uint32_t dk = pld::ld_pattern(dd);
        if ((int32_t)dk <= 0) {
          S.fail = k + 1;
          if (c == 0) *info = (int32_t)(row_base + k + 1);
        } else if (DDIV && dd.dec) {
          const double lk = pld::sqrt_r(dd.v);
          S.lkk = pgd::d_encode(lk);
          S.lkd = lk;
          S.lkr = __drcp_rn(lk);
          S.lkfast = pld::op_fast(lk) ? 1 : 0;
        } else {
          S.lkk = p32::sqrt(dk);
          if (DDIV) {
            double lk;
            const bool ok = pgd::d_decode(S.lkk, lk) && lk != 0.0 && pld::op_fast(lk);
            S.lkd = lk;
            S.lkr = ok ? __drcp_rn(lk) : 0.0;
            S.lkfast = ok ? 1 : 0;
          }
        }
        __threadfence_block();
        *vstep = k;
      }
    }
    if (k > 0 && i < b) {
#pragma unroll
      for (int q = 0; q < PC_Q; q++) {
        const int j = l + 32 * q;
        const bool now = DEFER == 0 || q == qc;                 // DEFER: column k's slot only
        if (now && j >= k && j <= i) pcd_fms(v[q], S, qp, i, j);
      }
    }
    if (l == (k & 31) && i >= k && i < b) {
      while (*vstep != k) { }
      __threadfence_block();
      if (!S.fail) {
        const uint32_t lkk = S.lkk;
        pld::LD xs = v[0];
#pragma unroll
        for (int q = 1; q < PC_Q; q++)
          if (q == qc) xs = v[q];
        uint32_t xp;
        double xq;
        bool dq = false;                                        // the quotient came from div_r
        if (i == k) {
          xp = lkk;
        } else if (DDIV && S.lkfast && xs.dec && pld::div_r(xs.v, S.lkd, S.lkr, xq)) {
          xp = pgd::d_encode(xq);                               // a fast operand: |E| <= 37, nonzero
          dq = true;
          pcd_push<NC>(cl, S, qk, i, xp, xq, 1u);
        } else {
          LaneVal x;
          lv_load(x, pld::ld_pattern(xs));
          pg::Acc dv;
          const bool dok = pg::acc_decode(lkk, dv) && dv.E <= 37 && dv.E >= -37;
          bool done = false;
          if (dok && x.dec) {
            done = pg::acc_div(x.a, dv.M, dv.E, dv.sg, __drcp_rn((double)dv.M) * 4294967296.0, K);
            if (done && !(x.a.E <= 75 && x.a.E >= -75) && x.a.E > pg::E_ZERO_LIMIT) {
              x.pat = pg::acc_encode(x.a);
              x.dec = false;
            }
          }
          if (!done) lv_load(x, div(lv_pattern(x), lkk));
          xp = lv_pattern(x);
          uint32_t sp = 0u;
          const double xd = pgd::stage_decode_d(xp, 0u, sp);
          pcd_push<NC>(cl, S, qk, i, xp, xd, sp == 0u ? 1u : 0u);
        }
        if (dq) { xs.v = xq; xs.pat = xp; xs.dec = true; }
        else pld::ld_load(xs, xp);
#pragma unroll
        for (int q = 0; q < PC_Q; q++)
          if (q == qc) v[q] = xs;
      }
    }
    __syncwarp();
    pc_arrive();
    if (DEFER && k > 0 && i < b) {                              // column k - 1 on the slots right of column k's
#pragma unroll
      for (int q = 1; q < PC_Q; q++) {
        const int j = l + 32 * q;
        if (q > qc && j <= i) pcd_fms(v[q], S, qp, i, j);
      }
    }
  }
  if (!failed) pc_wait();
#pragma unroll
  for (int q = 0; q < PC_Q; q++) {
    const int j = l + 32 * q;
    if (i < b && j <= i) A[(int64_t)i * lda + j] = pld::ld_pattern(v[q]);
  }
  cl.sync();
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

// The same with binary64 lane values (lanes_d.cuh: the D-MAC, constants in registers)
__global__ void __launch_bounds__(256) k_gemm_tiny_d(pg::Params P, int transb, int syrk) {
  if (P.stop != nullptr && *P.stop != 0) return;
  const int64_t i = (int64_t)blockIdx.y * 16 + (threadIdx.x >> 4);
  const int64_t j = (int64_t)blockIdx.x * 16 + (threadIdx.x & 15);
  if (i >= P.m || j >= P.n || (syrk && j > i)) return;
  pld::LD c;
  pld::ld_load(c, P.beta ? P.C[i * P.ldc + j] : 0u);
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
        uint32_t sa_ = 0u, sb_ = 0u;
        const double ad = pgd::stage_decode_d(a[u], 0u, sa_), bd = pgd::stage_decode_d(bp, 0u, sb_);
        pld::ld_fms(c, ad, sa_ == 0u, a[u], bd, sb_ == 0u, bp);
      }
    }
  }
  P.C[i * P.ldc + j] = pld::ld_pattern(c);
}

int pb_launch_gemm_tiny(const pg::Params& P, bool transb, bool syrk, cudaStream_t st) {
  pb_count_launch();
  const dim3 grid((unsigned)((P.n + 15) / 16), (unsigned)((P.m + 15) / 16));
  if (pb_dpath()) k_gemm_tiny_d<<<grid, 256, 0, st>>>(P, transb ? 1 : 0, syrk ? 1 : 0);
  else k_gemm_tiny<<<grid, 256, 0, st>>>(P, transb ? 1 : 0, syrk ? 1 : 0);
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

__global__ void __launch_bounds__(256) k_syrk_tiny_d(int64_t n, int64_t k, const uint32_t* A, int64_t lda, uint32_t* C,
                                                     int64_t ldc, const int32_t* stop) {
  if (stop != nullptr && *stop != 0) return;
  const int64_t i = (int64_t)blockIdx.y * 16 + (threadIdx.x >> 4);
  const int64_t j = (int64_t)blockIdx.x * 16 + (threadIdx.x & 15);
  if ((int64_t)blockIdx.x > (int64_t)blockIdx.y || i >= n || j > i) return;
  pld::LD c;
  pld::ld_load(c, C[i * ldc + j]);
  for (int64_t q = 0; q < k; q++) {
    const uint32_t ap = A[i * lda + q], bp = A[j * lda + q];
    uint32_t sa_ = 0u, sb_ = 0u;
    const double ad = pgd::stage_decode_d(ap, 0u, sa_), bd = pgd::stage_decode_d(bp, 0u, sb_);
    pld::ld_fms(c, ad, sa_ == 0u, ap, bd, sb_ == 0u, bp);
  }
  C[i * ldc + j] = pld::ld_pattern(c);
}

// Diagonal-block Cholesky: one cluster launch for 32 < b <= 256
// (k_potf2_cluster, POSIT_POTF2=2); else (POSIT_POTF2=1) right-looking by 32-wide block
// columns (leaf of <= 32 in one CTA, the rows below by the fused TRSM, the
// trailing lower triangle by the one-thread-per-element SYRK), or
// (POSIT_POTF2=0) the recursive potrf2 traversal.  Every stage is a no-op once
// *info != 0.
int pb_potf2(int64_t b, uint32_t* A, int64_t lda, int32_t* info, int64_t row_base, cudaStream_t st) {
  if (b <= 0) return 0;
  static const int mode = [] {  // 2: one cluster launch (default); 1: blocked right-looking, 32-wide; 0: recursive
    const char* e = getenv("POSIT_POTF2");
    return e ? atoi(e) : 2;
  }();
  if (mode == 2 && b > TB && b <= PC_B) {
    // POSIT_POTF2_NC: CTAs per cluster, 16 (default since r2m: C3 86.9 -> 83.2 ms; non-portable
    // size, 16 row warps per CTA) or 8 (portable; 32 row warps per CTA)
    static const int nc = [] {
      const char* e = getenv("POSIT_POTF2_NC");
      return (e && atoi(e) == 8) ? 8 : 16;
    }();
    static PbOncePerDevice attrs;
    pb_once_per_device(attrs, [] {
      cudaFuncSetAttribute(k_potf2_cluster<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k_potf2_cluster_d<16, 0, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k_potf2_cluster_d<16, 0, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k_potf2_cluster_d<16, 1, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k_potf2_cluster_d<16, 1, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    });
    pb_count_launch();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nc);
    cfg.blockDim = dim3(32 * (PC_B / nc));
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = nc;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int32_t bb = (int32_t)b;
    const bool dm = pb_dpath();
    // POSIT_POTF2_DEFER=0: the column k - 1 update of every slot before column k's division
    static const int defer = [] {                 // r2n / r2o: 1 is slower than 0 (0.895 vs 0.745 ms per 256^2 block)
      const char* e = getenv("POSIT_POTF2_DEFER");
      return (e && atoi(e) == 1) ? 1 : 0;
    }();
    static const bool ddiv = [] {                 // POSIT_POTF2_DDIV=0: integer-path sqrt and divisions
      const char* e = getenv("POSIT_POTF2_DDIV");
      return e ? atoi(e) != 0 : true;   // measured: see DESIGN.md section 8
    }();
    cudaError_t e;
#define PB_PC(NC_, DF_, DD_) e = cudaLaunchKernelEx(&cfg, k_potf2_cluster_d<NC_, DF_, DD_>, A, lda, (int)bb, info, row_base)
    if (!dm) e = nc == 16 ? cudaLaunchKernelEx(&cfg, k_potf2_cluster<16>, A, lda, (int)bb, info, row_base)
                          : cudaLaunchKernelEx(&cfg, k_potf2_cluster<8>, A, lda, (int)bb, info, row_base);
    else if (nc == 16 && defer == 0 && ddiv) PB_PC(16, 0, true);
    else if (nc == 16 && defer == 0) PB_PC(16, 0, false);
    else if (nc == 16 && ddiv) PB_PC(16, 1, true);
    else if (nc == 16) PB_PC(16, 1, false);
    else if (defer == 0 && ddiv) PB_PC(8, 0, true);
    else if (defer == 0) PB_PC(8, 0, false);
    else if (ddiv) PB_PC(8, 1, true);
    else PB_PC(8, 1, false);
#undef PB_PC
    return e == cudaSuccess ? 0 : POSIT_ECUDA;
  }
  if (mode >= 1 && b <= 256) {
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
        if (pb_dpath()) k_syrk_tiny_d<<<dim3(t, t), 256, 0, st>>>(r, jb, Ajj + jb * lda, lda, Ajj + jb * lda + jb, lda, info);
        else k_syrk_tiny<<<dim3(t, t), 256, 0, st>>>(r, jb, Ajj + jb * lda, lda, Ajj + jb * lda + jb, lda, info);
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

