// trsm.cu -- the two TRSM variants of the path: U12 =
// L11^-1 A12 (left, lower, unit) and L21 = A21 L11^-T (right, lower,
// transposed, non-unit).
#include "lanes.cuh"
#include "lanes_d.cuh"
#include <type_traits>

namespace pl {

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

// ---- unit lower in-block solve on the binary64-pipe MAC: 8 lanes per column ----
// B[i0 .. i0 + ib) <- L11^-1 B for one 32-row block (unit diagonal), every
// column of B independent.  Eight lanes share a column, lane t owning rows
// t, t + 8, t + 16, t + 24: at step k the owner of row k (final: all its
// updates from rows < k are in) broadcasts it within the 8-lane group and
// every lane applies b_r <- b_r (-) l_rk (x) b_k to its rows r > k -- the
// textbook order per element (Q6), 31 short steps with four independent
// chains per lane, and 8x the threads of the thread-per-column kernel (whose
// 496-MAC serial chain per thread ran at ~3 warps per SM).
constexpr int G8_COLS = 32;                   // columns per CTA (256 threads)
__global__ void __launch_bounds__(256) k_trsm_llnu_g8(const uint32_t* L, int64_t ldl, uint32_t* B, int64_t ldb,
                                                      int64_t i0, int64_t ib, int64_t n) {
  __shared__ double sld[TB][TB + 1];          // L[i0 + r][i0 + c] in binary64, r > c
  __shared__ uint32_t slp[TB][TB + 1];        // the patterns
  __shared__ uint32_t slf[TB];                // bit c of row r: L[r][c] is a fast operand
  const int tid = threadIdx.x;
  const int t = tid & 7;                      // lane in the column group
  const int64_t col = (int64_t)blockIdx.x * G8_COLS + (tid >> 3);
  const bool live = col < n;
  if (tid < TB) slf[tid] = 0u;
  __syncthreads();
  for (int e = tid; e < TB * TB; e += 256) {
    const int r = e / TB, c = e % TB;
    if (r < ib && c < r) {
      const uint32_t x = L[(i0 + r) * ldl + i0 + c];
      uint32_t sp = 0u;
      sld[r][c] = pgd::stage_decode_d(x, 0u, sp);
      slp[r][c] = x;
      if (sp == 0u) atomicOr(&slf[r], 1u << c);
    }
  }
  __syncthreads();
  pld::LD v[4];
#pragma unroll
  for (int u = 0; u < 4; u++) {
    const int r = t + 8 * u;
    pld::ld_load(v[u], (live && r < ib) ? B[(i0 + r) * ldb + col] : 0u);
  }
  for (int k = 0; k + 1 < ib; k++) {
    const int own = k & 7, uk = k >> 3;
    // the owner's final value of row k
    double bv = 0.0;
    uint32_t bp = 0u;
    bool bdec = false;
#pragma unroll
    for (int u = 0; u < 4; u++)
      if (u == uk) { bv = v[u].v; bp = v[u].pat; bdec = v[u].dec; }
    if (t == own && bdec) bp = pgd::d_encode(bv);
    const int src = (tid & 31 & ~7) | own;
    bv = __shfl_sync(0xFFFFFFFFu, bv, src);
    bp = __shfl_sync(0xFFFFFFFFu, bp, src);
    bdec = __shfl_sync(0xFFFFFFFFu, (int)bdec, src) != 0;
    const bool bfast = bdec && pld::op_fast(bv);
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int r = t + 8 * u;
      if (r > k && r < ib) {
        const bool af = (slf[r] >> k) & 1u;
        pld::ld_fms(v[u], sld[r][k], af, slp[r][k], bv, bfast, bp);
      }
    }
  }
  if (live) {
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int r = t + 8 * u;
      if (r < ib) B[(i0 + r) * ldb + col] = pld::ld_pattern(v[u]);
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
constexpr int FR_NMAX = 256;

// PG_RLTN_PIX: the update loop's MAC on the PIX product table (see gemm.cuh):
// staged L and block values carry .w = 32 E (+ the table base on the B side);
// the slow path then takes L's patterns from global memory and the block's
// final patterns from the row tile.
#ifndef PG_RLTN_PIX
#define PG_RLTN_PIX 1
#endif
#if PG_RLTN_PIX
#define FR_LW(x, E) ((uint32_t)(E) * 32u)
#define FR_BW(x, E) ((uint32_t)(E) * 32u + tpx0)
#define FR_LPAT(col, k) L[(int64_t)(col) * ldl + c0 + (k)]
#else
#define FR_LW(x, E) (x)
#define FR_BW(x, E) (x)
#define FR_LPAT(col, k) S.ld[k][(col) - ch0].w
#endif

// CH: the later columns' L values are staged (and the update loop run) in
// chunks of CH columns; CH < FR_NMAX halves the shared memory (with the
// in-block MAC's product table computed in registers instead of read from
// shared memory) so that three CTAs fit an SM.
// DM: the update loop on the binary64-pipe MAC (gemm_d.cuh): L and the block's
// values staged as exact binary64 numbers (8 bytes instead of 16), the D-MAC's
// 8 KB table instead of the PIX table, and the in-block MAC's product table in
// registers -- 72 KB, three CTAs per SM.
template <int W, int FR_ROWS, int CH = FR_NMAX, bool DM = false>
struct FrSmem {
  static constexpr bool TP = CH == FR_NMAX && !DM;   // the in-block MAC's product table in shared memory
  using LT = std::conditional_t<DM, double, uint4>;
  uint32_t b[FR_ROWS][FR_NMAX + 1];          // the CTA's rows of B (patterns)
  LT ld[W][CH];                               // L[j][c0 + k] decoded: A-format {M, E, sigma, .w} or binary64
  LT bop[FR_ROWS][W];                         // block J's final values (negated), B-format or binary64
  uint32_t lblk[W][W + 1];                    // L's diagonal block J (patterns)
  uint4 lblkd[W][W];                          // the same, decoded A-format {M, E, sigma, fast}
  uint4 ldiag[W];                             // L[c0 + k][c0 + k] as a divisor {M hidden@30, E, sg, fast}
  double ldrcp[W];                            // RN(2^32 / M) of each diagonal divisor
  int colfast[FR_NMAX];                       // column j's staged L values all fast-path operands
  int rowfast[FR_ROWS];                       // row r's block-J values all fast-path operands
  uint4 tp[TP ? pg::TSIZE : 1];              // the MAC's per-scale constant tables
  uint4 tx[pg::TSIZE];
#if PG_RLTN_PIX
  uint4 tpx[DM ? 1 : pg::PIX_NE];             // the PIX product table of the update loop
#endif
  pgd::dtab_t dtab[DM ? pgd::DT_SIZE : 1];    // the D-MAC's table
};

template <int W, int FR_ROWS, int CH = FR_NMAX, int MINB = 2, bool DM = false>
__global__ void __launch_bounds__(FR_ROWS * W, MINB) k_trsm_rltn_fused(const uint32_t* L, int64_t ldl, uint32_t* B,
                                                                    int64_t ldb, int64_t m, int64_t n,
                                                                    const int32_t* stop, int one) {
  constexpr int NT = FR_ROWS * W;
  using Sm = FrSmem<W, FR_ROWS, CH, DM>;
  extern __shared__ __align__(16) unsigned char fr_raw[];
  Sm& S = *reinterpret_cast<Sm*>(fr_raw);
  if (stop != nullptr && *stop != 0) return;
  const int tid = threadIdx.x;
  const int r = tid / W, c = tid % W;                  // row of the tile, column within a block
  const int grp = (tid & 31) & ~(W - 1);               // first lane of this row's lane group
  const int64_t r0 = (int64_t)blockIdx.x * FR_ROWS;
  const int64_t rows = (m - r0) < FR_ROWS ? (m - r0) : FR_ROWS;
  pg::fill_tables<(PG_PROD_BY_SUM != 0), Sm::TP>(S.tp, S.tx, tid, NT);
  pg::MacConst K;
  K.one = (uint32_t)one; K.sixteen = 16u * K.one;
  K.tp0 = (uint32_t)__cvta_generic_to_shared(S.tp + (Sm::TP ? pg::TBIAS : 0));
  K.tx0 = (uint32_t)__cvta_generic_to_shared(S.tx + pg::TBIAS) - 30u * 16u;
#if PG_RLTN_PIX
  if constexpr (!DM) pg::fill_prod_pix<false>(S.tpx, tid, NT);
  const uint32_t tpx0 = (uint32_t)__cvta_generic_to_shared(S.tpx + 2 * pg::PIX_SB);
#endif
  if constexpr (DM)
    for (int i = tid; i < pgd::DT_SIZE; i += NT) S.dtab[i] = pgd::dtab_fill(i);
  const uint32_t dtab0 = (uint32_t)__cvta_generic_to_shared(S.dtab);
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
    // stage the L values of the later columns [ch0, ch0 + CH) (thread per column: its jb values are contiguous)
    auto stage_chunk = [&](int ch0) {
    const int nch = ((int)n - ch0) < CH ? ((int)n - ch0) : CH;
    for (int jj = tid; jj < nch; jj += NT) {
      const int j = ch0 + jj;
      int f = 1;
      if (jb == W) {                                      // full block: all W loads in flight together
        uint32_t xs[W];
#pragma unroll
        for (int k = 0; k < W; k++) xs[k] = L[(int64_t)j * ldl + c0 + k];
#pragma unroll
        for (int k = 0; k < W; k++) {
          if constexpr (DM) {
            uint32_t sp = 0u;
            S.ld[k][jj] = pgd::stage_decode_d(xs[k], 0u, sp);
            f &= (int)(sp == 0u);
          } else {
            uint4 d;
            const bool fk = fast_a(xs[k], d);
            S.ld[k][jj] = make_uint4(d.x, d.y, d.z, FR_LW(xs[k], d.y));
            f &= (int)fk;
          }
        }
      } else {
        for (int k = 0; k < jb; k++) {
          const uint32_t x = L[(int64_t)j * ldl + c0 + k];
          if constexpr (DM) {
            uint32_t sp = 0u;
            S.ld[k][jj] = pgd::stage_decode_d(x, 0u, sp);
            f &= (int)(sp == 0u);
          } else {
            uint4 d;
            const bool fk = fast_a(x, d);
            S.ld[k][jj] = make_uint4(d.x, d.y, d.z, FR_LW(x, d.y));
            f &= (int)fk;
          }
        }
      }
      S.colfast[j] = f;
    }
    };
    if (nrest > 0) stage_chunk(c0 + jb);
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
            if constexpr (Sm::TP) pg::mac(v.a, ad.x, (int32_t)ad.y, (int32_t)ad.z, bM, bE, -bs, K, bad);
            else pg::mac(v.a, ad.x, (int32_t)ad.y, (int32_t)ad.z, bM, bE, -bs, pg::CalcConst(), bad);
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
        // sign pre-negated: c (-) a b
        if constexpr (DM) {
          double vd;
          pgd::d_decode(x, vd);                             // exact (used only when the row's values are fast)
          S.bop[r][c] = -vd;
        } else {
          S.bop[r][c] = make_uint4(v.a.M, (uint32_t)v.a.E, (uint32_t)(-v.a.sg), FR_BW(x, (uint32_t)v.a.E));
        }
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
    for (int ch0 = c0 + jb; ch0 < (int)n; ch0 += CH) {
    const int chend = ((int)n - ch0) < CH ? (int)n : ch0 + CH;
    if (ch0 > c0 + jb) {                                  // the next chunk of L (the previous one is done)
      __syncthreads();
      stage_chunk(ch0);
      __syncthreads();
    }
    if (r < rows) {
      const bool rf = S.rowfast[r] != 0;
      constexpr int G = 4;
      for (int col0 = ch0 + c; col0 < chend; col0 += G * W) {
        if constexpr (DM) {
          double a[G];
          uint32_t x[G];
          bool ok = rf;
#pragma unroll
          for (int u = 0; u < G; u++) {
            const int col = col0 + u * W;
            const bool in = col < chend;
            x[u] = in ? S.b[r][col] : 0u;
            const bool d = pgd::d_decode(x[u], a[u]) && pld::in_lane_range(a[u]);
            ok = ok && d && (!in || S.colfast[col] != 0);
          }
          if (ok) {
#pragma unroll 2
            for (int k = 0; k < jb; k++) {
              const double bd = S.bop[r][k];
#pragma unroll
              for (int u = 0; u < G; u++) a[u] = pgd::dmac(a[u], S.ld[k][min(col0 + u * W, chend - 1) - ch0], bd, dtab0);
            }
#pragma unroll
            for (int u = 0; u < G; u++)
              if (col0 + u * W < chend) S.b[r][col0 + u * W] = pgd::d_encode(a[u]);
            continue;
          }
#pragma unroll 1
          for (int u = 0; u < G; u++) {
            const int col = col0 + u * W;
            if (col >= chend) break;
            uint32_t y = x[u];
            for (int k = 0; k < jb; k++) y = sub(y, mul(L[(int64_t)col * ldl + c0 + k], S.b[r][c0 + k]));
            S.b[r][col] = y;
          }
          continue;
        } else {
        pg::Acc a[G];
        uint32_t x[G];
        bool ok = rf;
#pragma unroll
        for (int u = 0; u < G; u++) {
          const int col = col0 + u * W;
          const bool in = col < chend;
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
              const uint4 ad = S.ld[k][min(col0 + u * W, chend - 1) - ch0];
#if PG_RLTN_PIX
              pg::mac<pg::MacConst, true, false, false, false, true>(a[u], ad.x, (int32_t)ad.y, (int32_t)ad.z, bd.x,
                                                                      (int32_t)bd.y, (int32_t)bd.z, K, bad, ad.w, bd.w);
#else
              pg::mac(a[u], ad.x, (int32_t)ad.y, (int32_t)ad.z, bd.x, (int32_t)bd.y, (int32_t)bd.z, K, bad);
#endif
            }
          }
#pragma unroll
          for (int u = 0; u < G; u++)
            if (col0 + u * W < chend) S.b[r][col0 + u * W] = pg::acc_encode(a[u]);
        } else {
#pragma unroll 1
          for (int u = 0; u < G; u++) {
            const int col = col0 + u * W;
            if (col >= chend) break;
            uint32_t y = x[u];
            for (int k = 0; k < jb; k++) y = sub(y, mul(FR_LPAT(col, k), S.b[r][c0 + k]));
            S.b[r][col] = y;
          }
        }
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

// ---- right TRSM on the D-MAC, element-right-looking (Cholesky L21 = A21 L11^-T), n <= 256
// Per row r of B the oracle's order (DESIGN Q6) is, for
// i = 0 .. n-1:  x_i = b_i (/) L_ii,  then  b_j <- b_j (-) x_i (x) L_ji  for
// every j > i  -- each element receives its updates one at a time in
// ascending i, each (x), (-) and (/) one correctly rounded posit operation.
// This kernel runs exactly that loop.  A row is held by a half-warp, lane c
// owning columns c + 16 u (u = 0..15) as exact binary64 values in registers
// (the u loop is unrolled, so the row never touches shared memory); the lane
// owning column i divides (D-MAC division below), the quotient is broadcast
// by a shuffle, and every lane advances its later columns with the binary64
// MAC of gemm_d.cuh (L staged negated as binary64 in 32-column blocks, one
// copy per CTA of 32 rows).  Range contract as the GEMM's: operands (L, x)
// nonzero with |E| <= 37, every accumulator |E| <= 91 at each 16-step check.
// A warp whose rows leave it stops at that step, keeps its state, and after
// the loop finishes the row with the generic pattern operations from the same
// state (same bits).
constexpr int RD_ROWS = 32;                           // rows per CTA (16 warps, two rows each)
constexpr int RD_KB = 32;                             // L columns staged per block
constexpr int RD_LD = FR_NMAX + 1;

struct RdSmem {
  double l[RD_KB][RD_LD];                             // -L[j][c0 + k] (binary64, exact) at [k][j]
  double dg[RD_KB];                                   // L[c0 + k][c0 + k]
  double rc[RD_KB];                                   // RN(1 / L[c0 + k][c0 + k])
  int bad[RD_KB];                                     // column c0 + k has a zero / NaR / |E| > 37 L value
  pgd::dtab_tt<pgd::T64_GEMM> tab[pgd::DT_SIZE];
};

// the D-MAC division: pld::div_r (lanes_d.cuh)
__global__ void __launch_bounds__(RD_ROWS * 16, 2) k_trsm_rltn_d(const uint32_t* L, int64_t ldl, uint32_t* B,
                                                                  int64_t ldb, int64_t m, int64_t n,
                                                                  const int32_t* stop) {
  constexpr int NT = RD_ROWS * 16;
  extern __shared__ __align__(16) unsigned char rd_raw[];
  RdSmem& S = *reinterpret_cast<RdSmem*>(rd_raw);
  if (stop != nullptr && *stop != 0) return;
  const int tid = threadIdx.x, lane = tid & 31;
  const int c = lane & 15, hbase = lane & 16;          // column lane within the row; the row's first lane
  const int64_t r = (int64_t)blockIdx.x * RD_ROWS + (tid >> 4);
  const bool act = r < m;
  const int nn = (int)n;
  for (int i = tid; i < pgd::DT_SIZE; i += NT) S.tab[i] = pgd::dtab_fill<pgd::T64_GEMM>(i);
  const uint32_t tab0 = (uint32_t)__cvta_generic_to_shared(S.tab);

  // the row: b[u] = B[r][c + 16 u] as its exact binary64 value
  double b[16];
  bool okrow = true;
  uint32_t narm = 0u;                                   // NaR has no binary64 image: kept as a mask (a NaR
                                                        // makes the row slow from step 0, so b[] is never advanced)
#pragma unroll
  for (int u = 0; u < 16; u++) {
    const int j = c + 16 * u;
    const uint32_t x = (act && j < nn) ? B[r * ldb + j] : 0x40000000u;   // 1.0 in unused slots
    okrow &= pgd::d_decode(x, b[u]) && !pgd::d_above(b[u], pg::E_ACC_SLAB);
    if (x == p32::NAR) narm |= 1u << u;
  }
  bool slow = __any_sync(0xFFFFFFFFu, act && !okrow);
  int i_slow = 0;                                       // first step the generic path redoes

#pragma unroll
  for (int t = 0; t < 16; t++) {
    if (16 * t >= nn) continue;                         // CTA-uniform
    if (t % 2 == 0) {                                   // stage L's columns [c0, c0 + 32)
      const int c0 = 16 * t;
      __syncthreads();
      if (tid < RD_KB) S.bad[tid] = 0;
      __syncthreads();
      const int rows_l = nn - c0;
      for (int e = tid; e < RD_KB * rows_l; e += NT) {
        const int j = c0 + e / RD_KB, k = e % RD_KB;
        if (c0 + k >= nn) continue;
        const uint32_t x = L[(int64_t)j * ldl + c0 + k];
        if (j > c0 + k) {
          uint32_t sp = 0u;
          S.l[k][j] = pgd::stage_decode_d(x, 1u, sp);
          if (sp) atomicOr(&S.bad[k], 1);
        } else if (j == c0 + k) {
          uint32_t sp = 0u;
          const double d = pgd::stage_decode_d(x, 0u, sp);
          S.dg[k] = d;
          S.rc[k] = sp ? 0.0 : __drcp_rn(d);
          if (sp) atomicOr(&S.bad[k], 1);
        }
      }
      __syncthreads();
    }
    if (!slow && t > 0) {                               // accumulator range check every 16 steps
      bool hi = false;
#pragma unroll
      for (int u = t; u < 16; u++) hi |= pgd::d_above(b[u], pg::E_ACC_SLAB);
      if (__any_sync(0xFFFFFFFFu, act && hi)) { slow = true; i_slow = 16 * t; }
    }
    if (!slow) {
      const int iend = (nn - 16 * t) < 16 ? (nn - 16 * t) : 16;
      for (int ii = 0; ii < iend; ii++) {
        const int i = 16 * t + ii, k = i & (RD_KB - 1);
        double xo = 0.0;
        bool ok = S.bad[k] == 0;
        if (c == ii && ok) ok = pld::div_r(b[t], S.dg[k], S.rc[k], xo);
        if (__any_sync(0xFFFFFFFFu, act && !ok)) { slow = true; i_slow = i; break; }
        const double x = __shfl_sync(0xFFFFFFFFu, xo, hbase + ii);
        if (c == ii) b[t] = x;
        if (c > ii && c + 16 * t < nn) b[t] = pgd::dmac<pgd::T64_GEMM>(b[t], x, S.l[k][c + 16 * t], tab0);
#pragma unroll
        for (int u = t + 1; u < 16; u++)
          if (c + 16 * u < nn) b[u] = pgd::dmac<pgd::T64_GEMM>(b[u], x, S.l[k][c + 16 * u], tab0);
      }
    }
  }
  if (!slow) {
#pragma unroll
    for (int u = 0; u < 16; u++)
      if (act && c + 16 * u < nn) B[r * ldb + c + 16 * u] = pgd::d_encode(b[u]);
    return;
  }
  // generic path from step i_slow on (state: columns < i_slow final, the rest
  // updated by x_0 .. x_{i_slow - 1})
#pragma unroll
  for (int u = 0; u < 16; u++)
    if (act && c + 16 * u < nn) B[r * ldb + c + 16 * u] = ((narm >> u) & 1u) ? p32::NAR : pgd::d_encode(b[u]);
  __syncwarp();
  for (int i = i_slow; i < nn; i++) {
    const int o = i & 15;
    uint32_t xo = 0u;
    if (c == o && act) {
      xo = p32::div(B[r * ldb + i], L[(int64_t)i * ldl + i]);
      B[r * ldb + i] = xo;
    }
    const uint32_t x = __shfl_sync(0xFFFFFFFFu, xo, hbase + o);
    if (act)
      for (int j = c + 16 * ((i + 1 - c + 15) / 16); j < nn; j += 16)
        if (j > i) B[r * ldb + j] = p32::sub(B[r * ldb + j], p32::mul(x, L[(int64_t)j * ldl + i]));
  }
}

// ---- left TRSM on the D-MAC, element-right-looking (LU U12 = L11^-1 A12, unit diagonal), m <= 256
// Per column of B the oracle's order (DESIGN Q6): for k = 0 .. m-1,
// x_k = b_k is final, then b_i <- b_i (-) L_ik (x) x_k for every i > k
// (ascending k per element, each operation one rounded posit op).  Same
// machinery as k_trsm_rltn_d with rows and columns exchanged: a column of B
// is held by a half-warp, lane c owning rows c + 16 u as binary64 registers;
// 32 columns per CTA, staged in and out through shared memory (B is
// row-major, so the column tile is read and written with coalesced rows);
// -L[i][c0 + k] staged as binary64 at [k][i] in 32-column blocks.  No
// division (unit diagonal).  A warp leaving the range contract stops at that
// step and finishes with the generic pattern operations on the shared tile.
constexpr int LD_COLS = 32;                           // columns of B per CTA (16 warps, two columns each)

struct LdSmem {
  union {
    double l[RD_KB][RD_LD];                           // -L[i][c0 + k] at [k][i]
    uint32_t t[FR_NMAX][LD_COLS + 1];                 // the CTA's columns of B (patterns), row-major
  } u;
  int bad[RD_KB];
  pgd::dtab_tt<pgd::T64_GEMM> tab[pgd::DT_SIZE];
};

__global__ void __launch_bounds__(LD_COLS * 16, 2) k_trsm_llnu_d(const uint32_t* L, int64_t ldl, uint32_t* B,
                                                                  int64_t ldb, int64_t m, int64_t n) {
  constexpr int NT = LD_COLS * 16;
  extern __shared__ __align__(16) unsigned char ld_raw[];
  LdSmem& S = *reinterpret_cast<LdSmem*>(ld_raw);
  const int tid = threadIdx.x, lane = tid & 31;
  const int c = lane & 15, hbase = lane & 16;          // row lane within the column; the column's first lane
  const int cl = tid >> 4;                             // the CTA's column of this half-warp
  const int64_t col0 = (int64_t)blockIdx.x * LD_COLS;
  const int ncols = (n - col0) < LD_COLS ? (int)(n - col0) : LD_COLS;
  const bool act = cl < ncols;
  const int mm = (int)m;
  for (int i = tid; i < pgd::DT_SIZE; i += NT) S.tab[i] = pgd::dtab_fill<pgd::T64_GEMM>(i);
  const uint32_t tab0 = (uint32_t)__cvta_generic_to_shared(S.tab);
  for (int e = tid; e < mm * LD_COLS; e += NT) {
    const int i = e / LD_COLS, q = e % LD_COLS;
    S.u.t[i][q] = q < ncols ? B[(int64_t)i * ldb + col0 + q] : 0x40000000u;
  }
  __syncthreads();
  double b[16];
  bool okcol = true;
  uint32_t narm = 0u;                                   // NaR has no binary64 image: kept as a mask (a NaR
                                                        // makes the column slow from step 0, so b[] is never advanced)
#pragma unroll
  for (int u = 0; u < 16; u++) {
    const int i = c + 16 * u;
    const uint32_t x = i < mm ? S.u.t[i][cl] : 0x40000000u;
    okcol &= pgd::d_decode(x, b[u]) && !pgd::d_above(b[u], pg::E_ACC_SLAB);
    if (x == p32::NAR) narm |= 1u << u;
  }
  bool slow = __any_sync(0xFFFFFFFFu, act && !okcol);
  int k_slow = 0;

#pragma unroll
  for (int t = 0; t < 16; t++) {
    if (16 * t >= mm) continue;                         // CTA-uniform
    if (t % 2 == 0) {                                   // stage L's columns [c0, c0 + 32), rows below them
      const int c0 = 16 * t;
      __syncthreads();
      if (tid < RD_KB) S.bad[tid] = 0;
      __syncthreads();
      const int rows_l = mm - c0;
      for (int e = tid; e < RD_KB * rows_l; e += NT) {
        const int i = c0 + e / RD_KB, k = e % RD_KB;
        if (c0 + k >= mm || i <= c0 + k) continue;
        uint32_t sp = 0u;
        S.u.l[k][i] = pgd::stage_decode_d(L[(int64_t)i * ldl + c0 + k], 1u, sp);
        if (sp) atomicOr(&S.bad[k], 1);
      }
      __syncthreads();
    }
    if (!slow && t > 0) {
      bool hi = false;
#pragma unroll
      for (int u = t; u < 16; u++) hi |= pgd::d_above(b[u], pg::E_ACC_SLAB);
      if (__any_sync(0xFFFFFFFFu, act && hi)) { slow = true; k_slow = 16 * t; }
    }
    if (!slow) {
      const int kend = (mm - 16 * t) < 16 ? (mm - 16 * t) : 16;
      for (int ii = 0; ii < kend; ii++) {
        const int k = 16 * t + ii, kl = k & (RD_KB - 1);
        const bool ok = S.bad[kl] == 0 && (c != ii || pld::op_fast(b[t]));
        if (__any_sync(0xFFFFFFFFu, act && !ok)) { slow = true; k_slow = k; break; }
        const double x = __shfl_sync(0xFFFFFFFFu, b[t], hbase + ii);
        if (c > ii && c + 16 * t < mm) b[t] = pgd::dmac<pgd::T64_GEMM>(b[t], x, S.u.l[kl][c + 16 * t], tab0);
#pragma unroll
        for (int u = t + 1; u < 16; u++)
          if (c + 16 * u < mm) b[u] = pgd::dmac<pgd::T64_GEMM>(b[u], x, S.u.l[kl][c + 16 * u], tab0);
      }
    }
  }
  __syncthreads();                                      // L staging done: the union holds B's tile again
#pragma unroll
  for (int u = 0; u < 16; u++)
    if (act && c + 16 * u < mm) S.u.t[c + 16 * u][cl] = ((narm >> u) & 1u) ? p32::NAR : pgd::d_encode(b[u]);
  if (slow) {
    // generic path from step k_slow on (rows < k_slow final, the rest updated by x_0 .. x_{k_slow - 1});
    // lane c reads and writes only its own rows, row k reaches the others by a shuffle
    for (int k = k_slow; k < mm; k++) {
      const uint32_t xo = (act && c == (k & 15)) ? S.u.t[k][cl] : 0u;
      const uint32_t x = __shfl_sync(0xFFFFFFFFu, xo, hbase + (k & 15));
      if (act)
        for (int i = c + 16 * ((k + 1 - c + 15) / 16); i < mm; i += 16)
          if (i > k) S.u.t[i][cl] = p32::sub(S.u.t[i][cl], p32::mul(L[(int64_t)i * ldl + k], x));
    }
  }
  __syncthreads();
  for (int e = tid; e < mm * LD_COLS; e += NT) {
    const int i = e / LD_COLS, q = e % LD_COLS;
    if (q < ncols) B[(int64_t)i * ldb + col0 + q] = S.u.t[i][q];
  }
}

}  // namespace pl

using namespace pl;

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
  const int use_col = col_env >= 0 ? col_env : (n > (int64_t)pb_num_sms() * TB ? 4 : 0);
  static const int blk_env = [] {                 // warp-per-column CTA width: 8 (default) or 32 columns
    const char* e = getenv("POSIT_LLNU_BLK");
    return e ? atoi(e) : 8;
  }();
  static const int g8_env = [] {                  // POSIT_LLNU_G8=0: the integer-MAC in-block kernels
    const char* e = getenv("POSIT_LLNU_G8");
    return e ? atoi(e) : 1;
  }();
  const bool g8 = pb_dpath() && g8_env != 0;
  static const int d_env = [] {                   // POSIT_LLNU_D=0: the blocked kernels (in-block solves + GEMMs)
    const char* e = getenv("POSIT_LLNU_D");
    return e ? atoi(e) : 1;   // default since r2m: C5 178.1 -> 172.8 ms, C4 1134 -> 1126 ms, digests equal
  }();
  if (pb_dpath() && d_env != 0 && m <= FR_NMAX) {
    static PbOncePerDevice attrs;
    pb_once_per_device(attrs, [] {
      cudaFuncSetAttribute(k_trsm_llnu_d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LdSmem));
    });
    pb_count_launch();
    k_trsm_llnu_d<<<(unsigned)((n + LD_COLS - 1) / LD_COLS), LD_COLS * 16, sizeof(LdSmem), st>>>(L, ldl, B, ldb, m, n);
    return last_launch();
  }
  for (int64_t i0 = 0; i0 < m; i0 += TB) {
    const int64_t ib = (m - i0) < TB ? (m - i0) : TB;
    if (ib > 1) {
      pb_count_launch();
      if (g8)
        k_trsm_llnu_g8<<<(unsigned)((n + G8_COLS - 1) / G8_COLS), 256, 0, st>>>(L, ldl, B, ldb, i0, ib, n);
      else if (use_col == 8)
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
    // variant: W lanes per row x FR_ROWS rows per CTA [x L staged in chunks of CH columns]:
    // env POSIT_RLTN = "W,ROWS[,CH]"; CH = 128 fits three CTAs per SM
    static const int var = [] {
      const char* e = getenv("POSIT_RLTN");
      int w = 16, r = 16, ch = 256;
      if (e) sscanf(e, "%d,%d,%d", &w, &r, &ch);
      return (ch == 128 ? 100000 : 0) + w * 100 + r;
    }();
    static PbOncePerDevice attrs;
    pb_once_per_device(attrs, [] {
      cudaFuncSetAttribute(k_trsm_rltn_fused<16, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(FrSmem<16, 16>));
      cudaFuncSetAttribute(k_trsm_rltn_fused<16, 16, 128, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(FrSmem<16, 16, 128>));
      cudaFuncSetAttribute(k_trsm_rltn_fused<16, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(FrSmem<16, 32>));
      cudaFuncSetAttribute(k_trsm_rltn_fused<8, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(FrSmem<8, 16>));
      cudaFuncSetAttribute(k_trsm_rltn_fused<8, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(FrSmem<8, 32>));
      cudaFuncSetAttribute(k_trsm_rltn_fused<16, 16, FR_NMAX, 3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(FrSmem<16, 16, FR_NMAX, true>));
      cudaFuncSetAttribute(k_trsm_rltn_d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RdSmem));
    });
    static const int rd_env = [] {                 // POSIT_RLTN_D=0: the blocked fused kernel on the D-MAC path
      const char* e = getenv("POSIT_RLTN_D");
      return e ? atoi(e) : 1;   // default since r2m: C3 89.7 -> 86.9 ms, digest equal
    }();
    pb_count_launch();
#define PB_RLTN(W_, R_, ...)                                                                                         \
  k_trsm_rltn_fused<W_, R_, ##__VA_ARGS__><<<(unsigned)((m + R_ - 1) / R_), R_ * W_,                              \
                                              sizeof(FrSmem<W_, R_, ##__VA_ARGS__>), st>>>(L, ldl, B, ldb, m, n, stop, 1)
    if (pb_dpath() && var == 1616 && rd_env != 0)
      k_trsm_rltn_d<<<(unsigned)((m + RD_ROWS - 1) / RD_ROWS), RD_ROWS * 16, sizeof(RdSmem), st>>>(L, ldl, B, ldb, m,
                                                                                                 n, stop);
    else if (pb_dpath() && var == 1616)
      k_trsm_rltn_fused<16, 16, FR_NMAX, 3, true><<<(unsigned)((m + 15) / 16), 256, sizeof(FrSmem<16, 16, FR_NMAX, true>),
                                                    st>>>(L, ldl, B, ldb, m, n, stop, 1);
    else if (var == 1632) PB_RLTN(16, 32);
    else if (var == 816) PB_RLTN(8, 16);
    else if (var == 832) PB_RLTN(8, 32);
    else if (var == 101616) k_trsm_rltn_fused<16, 16, 128, 3><<<(unsigned)((m + 15) / 16), 256,
                                                               sizeof(FrSmem<16, 16, 128>), st>>>(L, ldl, B, ldb, m,
                                                                                                  n, stop, 1);
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
