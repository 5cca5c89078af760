// misc.cu -- the accuracy solves (Rgetrs / Rpotrs), elementwise
// posit ops, the Eq.2 epilogue (axpby) and the binary64 conversions (a0).
#include "lanes.cuh"

namespace pl {

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

}  // namespace pl

using namespace pl;

int pb_solve(bool chol, int64_t n, const uint32_t* A, int64_t lda, const int32_t* ipiv, uint32_t* b, cudaStream_t st) {
  if (n <= 0) return 0;
  const size_t smem = (size_t)n * sizeof(uint32_t);
  if (smem > 200 * 1024) return POSIT_ENOTSUP;
  static PbOncePerDevice attrs;
  pb_once_per_device(attrs, [] {
    cudaFuncSetAttribute(k_getrs, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_potrs, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
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

