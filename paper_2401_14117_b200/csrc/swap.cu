// swap.cu -- row interchanges (laswp) and the distributed
// panel's pivot key (posit_iamax_key).
#include "lanes.cuh"

namespace pl {

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

}  // namespace pl

using namespace pl;

int pb_laswp(int64_t ncols, uint32_t* A, int64_t lda, int64_t k1, int64_t k2, const int32_t* ipiv, int64_t ipiv_base,
             cudaStream_t st) {
  if (ncols <= 0 || k2 <= k1) return 0;
  constexpr size_t smem = 2 * SWP_MAX * SWP_COLS * sizeof(uint32_t);
  static PbOncePerDevice attrs;
  pb_once_per_device(attrs, [] {
    cudaFuncSetAttribute(k_laswp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  pb_count_launch();
  k_laswp<<<(unsigned)((ncols + SWP_COLS - 1) / SWP_COLS), 256, smem, st>>>(A, lda, ncols, k1, k2, ipiv, ipiv_base);
  return last_launch();
}

int pb_iamax_key(int64_t m, const uint32_t* col, int64_t stride, const int32_t* grow, int64_t row_min, long long* out,
                 cudaStream_t st) {
  pb_count_launch();
  k_iamax_key<<<1, 1024, 0, st>>>(m, col, stride, grow, row_min, out);
  return last_launch();
}

