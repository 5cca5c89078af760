// leaf.cu -- the LU panel: pivot search by signed compare of
// patterns, row swap, posit division, in-panel update.  The 32-column leaf is
// one cooperative launch with one grid sync per column; the panel is the
// recursive getrf2 traversal around it; the fused tail factors a whole
// trailing block the same way.
#include "lanes.cuh"
#include "lanes_d.cuh"

namespace pl {

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

// DM: the in-panel update on the binary64-pipe MAC (gemm_d.cuh), the pivot row
// staged as exact binary64 numbers (negated) with a fast flag
template <int WMAX, bool DM = false>
__global__ void __launch_bounds__(1024) k_leaf_coop1(uint32_t* A, int64_t lda, int64_t m, int64_t w,
                                                     int64_t rows_per_cta, int32_t* ipiv, int32_t* info,
                                                     int64_t row_base, LeafWs* ws, uint32_t* cand, uint32_t* jrow,
                                                     int ddiv) {
  extern __shared__ uint32_t tile[];                  // [rows_per_cta][w]
  __shared__ unsigned long long red[32];
  __shared__ unsigned long long cbest;                // this CTA's best candidate key (next column)
  __shared__ uint32_t srow[2 * WMAX];                 // the published rows p and j of the current column
  __shared__ uint4 urow[DM ? 1 : WMAX];               // the pivot row as decoded B operands {M, E, sg, fast}
  __shared__ uint32_t urowp[WMAX];                    // ... and as patterns
  __shared__ double urowd[DM ? WMAX : 1];             // DM: -(pivot row) in binary64
  __shared__ uint8_t urowf[DM ? WMAX : 1];            // DM: fast-operand flags
  __shared__ pgd::dtab_t dtab[DM ? pgd::DT_SIZE : 1];
  __shared__ uint4 tp[pg::TSIZE], tx[pg::TSIZE];      // the MAC's constant tables
  const int NT = blockDim.x;
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x;
  pg::fill_tables(tp, tx, tid, NT);
  if constexpr (DM)
    for (int i = tid; i < pgd::DT_SIZE; i += NT) dtab[i] = pgd::dtab_fill(i);
  const uint32_t dtab0 = (uint32_t)__cvta_generic_to_shared(dtab);
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
      const uint32_t x = srow[usrc + c];
      if constexpr (DM) {
        uint32_t sp = 0u;
        urowd[c] = pgd::stage_decode_d(x, 1u, sp);     // negated: c (-) l u = c (+) l (-u)
        urowf[c] = sp == 0u ? 1 : 0;
      } else {
        LaneVal t;
        lv_load(t, x);
        urow[c] = make_uint4(t.a.M, (uint32_t)t.a.E, (uint32_t)t.a.sg, lv_operand(t) ? 1u : 0u);
      }
      urowp[c] = x;
    }
    __syncthreads();
    const int i0 = (int)((j + 1 > rb ? j + 1 : rb) - rb);
    if (v != 0u) {                                    // Q8 (one division each); skipped for a zero pivot (Q11)
      pg::Acc dv;
      const bool dok = pg::acc_decode(v, dv) && v != 0x80000000u && dv.E <= 37 && dv.E >= -37;
      const double rcp = dok ? __drcp_rn((double)dv.M) * 4294967296.0 : 0.0;
      // DM && ddiv: the column scale on the binary64 pipe (pld::div_r), else the integer-path division
      double vd = 0.0, vr = 0.0;
      bool vfast = false;
      if constexpr (DM) {
        if (ddiv & 1) {
          uint32_t sp = 0u;
          vd = pgd::stage_decode_d(v, 0u, sp);
          vfast = sp == 0u;
          vr = vfast ? __drcp_rn(vd) : 0.0;
        }
      }
      for (int i = i0 + tid; i < nr; i += NT) {
        const uint32_t x = tile[i * W + (int)j];
        if constexpr (DM) {
          double xv, q;
          if (vfast && pgd::d_decode(x, xv) && !pgd::d_above(xv, pg::E_ACC_SLAB) && pld::div_r(xv, vd, vr, q)) {
            tile[i * W + (int)j] = pgd::d_encode(q);
            continue;
          }
        }
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
      uint32_t cnt = nr > i0 ? (uint32_t)(nr - i0) * (uint32_t)wq : 0u;
      if constexpr (DM) {
        // Row mode (ddiv & 2; tall CTAs: at least half the threads own a row): a thread takes whole
        // rows, so the multiplier l_ij is decoded once per row and there is no element -> (row, column)
        // division; lanes walk the columns in a rotated order (lane + t mod wq), which spreads one
        // column's rows (stride W words: one bank) over the banks.  Same single update per element.
        if ((ddiv & 2) && (nr - i0) * 2 >= NT) {
          const int start = (int)((uint32_t)(tid & 31) % (uint32_t)wq);
          for (int i = i0 + tid; i < nr; i += NT) {
            const uint32_t lp = tile[i * W + (int)j];
            uint32_t sp = 0u;
            const double l = pgd::stage_decode_d(lp, 0u, sp);
            int qq = start;
            for (int t = 0; t < wq; t++) {
              const int q = (int)j + 1 + qq;
              qq = qq + 1 == wq ? 0 : qq + 1;
              const uint32_t cx = tile[i * W + q];
              double cv;
              const bool cd = pgd::d_decode(cx, cv) && pld::in_lane_range(cv);
              const uint32_t nv = (sp == 0u && urowf[q] != 0 && cd)
                                      ? pgd::d_encode(pgd::dmac(cv, l, urowd[q], dtab0))
                                      : sub(cx, mul(lp, urowp[q]));
              tile[i * W + q] = nv;
              if (q == (int)j + 1) {
                const unsigned long long k = piv_key(nv, rb + i);
                best = k > best ? k : best;
              }
            }
          }
          cnt = 0u;
        }
      }
      for (uint32_t e = tid; e < cnt; e += NT) {
        const uint32_t ii = e / (uint32_t)wq;
        const int i = i0 + (int)ii;
        const int q = (int)j + 1 + (int)(e - ii * (uint32_t)wq);
        const uint32_t lp = tile[i * W + (int)j];
        uint32_t nv;
        if constexpr (DM) {
          uint32_t sp = 0u;
          const double l = pgd::stage_decode_d(lp, 0u, sp);
          const uint32_t cx = tile[i * W + q];
          double cv;
          const bool cd = pgd::d_decode(cx, cv) && pld::in_lane_range(cv);
          nv = (sp == 0u && urowf[q] != 0 && cd) ? pgd::d_encode(pgd::dmac(cv, l, urowd[q], dtab0))
                                                 : sub(cx, mul(lp, urowp[q]));
        } else {
          uint4 ad;
          const bool af = fast_a(lp, ad);
          const uint4 ub = urow[q];
          LaneVal c;
          lv_load(c, tile[i * W + q]);
          lv_fms_t(c, lp, af, ad, ub.x, (int32_t)ub.y, (int32_t)ub.z, ub.w != 0u, urowp[q], K);
          nv = lv_pattern(c);
        }
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

}  // namespace pl

using namespace pl;

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
  static const int coop_env = [] {
    const char* e = getenv("POSIT_LEAF_COOP");
    return e ? atoi(e) : 1;
  }();
  static PbOncePerDevice attrs;
  pb_once_per_device(attrs, [] {
    cudaFuncSetAttribute(k_leaf_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(k_leaf_coop1<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(k_leaf_coop1<TAIL_WMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(k_leaf_coop1<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    cudaFuncSetAttribute(k_leaf_coop1<TAIL_WMAX, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  });
  const int coop = pb_coop_supported() ? coop_env : 0, nsm = pb_num_sms();
  // on the caller's stream: one CTA of 256 threads per SM; on a side stream
  // (lookahead, sharing the SMs with the trailing GEMM): a few CTAs of 1024
  static const int force = [] {                 // POSIT_LEAF_CTAS = 16 / 148: force one configuration (tests, sweeps)
    const char* e = getenv("POSIT_LEAF_CTAS");
    return e ? atoi(e) : 0;
  }();
  const bool wide = force ? force > 16 : allow_coop;
  static const int side_env = [] {               // side-stream leaf CTAs (1024 threads each); 0: auto
    const char* e = getenv("POSIT_SIDE_LEAF_CTAS");
    const int v = e ? atoi(e) : 0;
    return v > 0 ? v : 0;
  }();
  // auto: 1024 rows per CTA, 8 to 16 CTAs (fewer CTAs leave more SMs to the
  // concurrent trailing update; r06e: C5 343.1 -> 342.2 ms with 8, and 16 at
  // m = 16384, where 8 would not fit the leaf in shared memory)
  const int64_t side_auto = (m + 1023) / 1024 < 8 ? 8 : ((m + 1023) / 1024 > 16 ? 16 : (m + 1023) / 1024);
  const int side_ctas = side_env > 0 ? side_env : (int)side_auto;
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
    static const int ddiv_env = [] {                // POSIT_LEAF_DDIV=1: the column scale by pld::div_r (D-MAC path)
      const char* e = getenv("POSIT_LEAF_DDIV");
      return e ? atoi(e) : 1;   // measured: see DESIGN.md section 8
    }();
    static const int rows_env = [] {                // POSIT_LEAF_ROWS=1: a thread per row in the update of tall CTAs
      const char* e = getenv("POSIT_LEAF_ROWS");
      return e ? atoi(e) : 0;   // opt-in until measured on the GPU
    }();
    int ddiv = (ddiv_env ? 1 : 0) | (rows_env ? 2 : 0);
    void* args[] = {&A, &ld, &mm, &ww, &rr, &ipiv, &info, &rbase, &ws, &cand, &jrow, &ddiv};
    const unsigned grid = (unsigned)((m + rpc - 1) / rpc);
    // coop 1: one grid sync per column (default); coop 2: two (publish after the pivot is known; w <= 64)
    const void* kfn = nullptr;
    if (grid <= (unsigned)LEAF_MAXCTA && (coop != 2 || wide_w))
      kfn = pb_dpath() ? (wide_w ? (const void*)k_leaf_coop1<TAIL_WMAX, true> : (const void*)k_leaf_coop1<64, true>)
                       : (wide_w ? (const void*)k_leaf_coop1<TAIL_WMAX> : (const void*)k_leaf_coop1<64>);
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
  const int nsm = pb_num_sms();
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

