// capi.cu -- the C ABI of libposit_b200.so (include/posit_b200.h): argument
// validation, the blocked getrf / potrf drivers, and the HOST-buffer GEMM.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <atomic>
#include <stdlib.h>
#include "gemm.cuh"
#include "internal.h"

static thread_local char g_last_error[256] = "";
static std::atomic<unsigned long long> g_launches{0};

void pb_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

bool pb_dpath() {
  static const bool v = [] {
    const char* e = getenv("POSIT_GEMM_PATH");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}

int pb_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0) { (void)cudaGetLastError(); d = 0; }
  return d;
}

// per-device caches (0 = not yet queried)
static std::atomic<int> g_nsm[PB_MAX_DEVICES];
static std::atomic<int> g_coop[PB_MAX_DEVICES];

int pb_num_sms() {
  const int d = pb_device() % PB_MAX_DEVICES;
  int v = g_nsm[d].load(std::memory_order_relaxed);
  if (v <= 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, pb_device()) != cudaSuccess || v <= 0) {
      (void)cudaGetLastError();
      v = 148;                                   // B200 (sm_100a); only if the query itself fails
    }
    g_nsm[d].store(v, std::memory_order_relaxed);
  }
  return v;
}

bool pb_coop_supported() {
  const int d = pb_device() % PB_MAX_DEVICES;
  int v = g_coop[d].load(std::memory_order_relaxed);
  if (v == 0) {
    int ok = 0;
    if (cudaDeviceGetAttribute(&ok, cudaDevAttrCooperativeLaunch, pb_device()) != cudaSuccess) {
      (void)cudaGetLastError();
      ok = 0;
    }
    v = ok ? 1 : -1;
    g_coop[d].store(v, std::memory_order_relaxed);
  }
  return v > 0;
}

static int cuda_check(cudaError_t e) {
  if (e == cudaSuccess) return 0;
  strncpy(g_last_error, cudaGetErrorString(e), sizeof(g_last_error) - 1);
  return POSIT_ECUDA;
}

static int launch_check(int rc) {
  if (rc == POSIT_ECUDA) {
    const cudaError_t e = cudaGetLastError();
    strncpy(g_last_error, cudaGetErrorString(e), sizeof(g_last_error) - 1);
  }
  return rc;
}

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int posit_abi_version(void) { return POSIT_ABI_VERSION; }

uint64_t posit_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

const char* posit_strerror(int code) {
  if (code == POSIT_OK) return "ok";
  if (code == POSIT_ENOTSUP) return "unsupported option";
  if (code == POSIT_ECUDA) return "CUDA error (see posit_last_error)";
  if (code < 0 && code > -100) return "invalid argument";
  return "unknown";
}

const char* posit_last_error(void) { return g_last_error; }

static int gemm_common(char transa, char transb, int64_t m, int64_t n, int64_t k, uint32_t alpha, const uint32_t* A,
                       int64_t lda, const uint32_t* B, int64_t ldb, uint32_t beta, uint32_t* C, int64_t ldc,
                       void* stream, bool naive) {
  if (transa != 'N' && transa != 'T') return -1;
  if (transb != 'N' && transb != 'T') return -2;
  if (m < 0) return -3;
  if (n < 0) return -4;
  if (k < 0) return -5;
  if (alpha != POSIT_ONE && alpha != POSIT_MONE) return -6;
  const int64_t acols = transa == 'N' ? k : m;       // A is m x k ('N') or k x m ('T'), row-major
  if (lda < (acols > 1 ? acols : 1)) return -8;
  if (ldb < ((transb == 'N' ? n : k) > 1 ? (transb == 'N' ? n : k) : 1)) return -10;
  if (beta != 0u && beta != POSIT_ONE) return -11;
  if (ldc < (n > 1 ? n : 1)) return -13;
  if (m == 0 || n == 0) return 0;
  if ((k > 0 && (A == nullptr || B == nullptr)) || C == nullptr) return -7;
  pg::Params P{m, n, k, A, lda, B, ldb, C, ldc, alpha == POSIT_MONE ? 1 : 0, beta == POSIT_ONE ? 1 : 0, nullptr};
  P.transa = transa == 'T' ? 1 : 0;
  const int rc = naive ? pb_launch_gemm_naive(P, transb == 'T', false, S(stream))
                       : pb_launch_gemm(P, transb == 'T', false, S(stream));
  if (rc) return launch_check(rc);
  return cuda_check(cudaPeekAtLastError());
}

int posit_gemm(char transa, char transb, int64_t m, int64_t n, int64_t k, uint32_t alpha, const uint32_t* A,
               int64_t lda, const uint32_t* B, int64_t ldb, uint32_t beta, uint32_t* C, int64_t ldc, void* stream) {
  return gemm_common(transa, transb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, stream, false);
}

int posit_gemm_naive(char transa, char transb, int64_t m, int64_t n, int64_t k, uint32_t alpha, const uint32_t* A,
                     int64_t lda, const uint32_t* B, int64_t ldb, uint32_t beta, uint32_t* C, int64_t ldc,
                     void* stream) {
  return gemm_common(transa, transb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, stream, true);
}

size_t posit_gemm_eq2_work_bytes(int64_t m, int64_t n) {
  if (m < 0 || n < 0) return 0;
  return (size_t)4 * (size_t)(m * n);
}

int posit_gemm_eq2(char transa, char transb, int64_t m, int64_t n, int64_t k, uint32_t alpha, const uint32_t* A,
                   int64_t lda, const uint32_t* B, int64_t ldb, uint32_t beta, uint32_t* C, int64_t ldc, void* work,
                   size_t work_bytes, void* stream) {
  if (transa != 'N' && transa != 'T') return -1;
  if (transb != 'N' && transb != 'T') return -2;
  if (m < 0) return -3;
  if (n < 0) return -4;
  if (k < 0) return -5;
  const int64_t acols = transa == 'N' ? k : m;
  if (lda < (acols > 1 ? acols : 1)) return -8;
  if (ldb < ((transb == 'N' ? n : k) > 1 ? (transb == 'N' ? n : k) : 1)) return -10;
  if (ldc < (n > 1 ? n : 1)) return -13;
  if (m == 0 || n == 0) return 0;
  if (work == nullptr || work_bytes < posit_gemm_eq2_work_bytes(m, n)) return -15;
  if ((k > 0 && (A == nullptr || B == nullptr)) || C == nullptr) return -7;
  uint32_t* T = static_cast<uint32_t*>(work);
  // t = sum of products from 0 (the fast kernel with alpha = +1, beta = 0), then the epilogue
  int rc;
  if (k > 0) {
    pg::Params P{m, n, k, A, lda, B, ldb, T, n, 0, 0, nullptr};
    P.transa = transa == 'T' ? 1 : 0;
    if ((rc = pb_launch_gemm(P, transb == 'T', false, S(stream)))) return launch_check(rc);
  } else if ((rc = cuda_check(cudaMemsetAsync(T, 0, posit_gemm_eq2_work_bytes(m, n), S(stream))))) {
    return rc;
  }
  return launch_check(pb_axpby(alpha, T, n, beta, C, ldc, m, n, S(stream)));
}

size_t posit_gemm_host_work_bytes(int64_t m, int64_t n, int64_t k) {
  if (m < 0 || n < 0 || k < 0) return 0;
  return (size_t)4 * (size_t)(m * k + k * n + m * n) + 256;
}

// Pipelined host GEMM (transa = 'N'): C's rows in chunks; chunk i's A rows
// and C rows go up on a copy stream while chunk i-1 computes (two compute
// streams, so one chunk's last wave overlaps the next chunk's first) and chunk
// i-2's C comes back on a third stream.  B goes up first, once.  Row chunks
// are independent outputs with unchanged per-element order, so the bits equal
// the one-launch GEMM.  POSIT_HOST_PIPELINE=0 forces the serial schedule.
static constexpr int64_t HOST_CHUNK_MIN = 512;
static int host_pipeline_env() {
  static const int v = [] {
    const char* e = getenv("POSIT_HOST_PIPELINE");
    return e ? atoi(e) : 1;
  }();
  return v;
}

static int gemm_host_pipelined(char transb, int64_t m, int64_t n, int64_t k, uint32_t alpha, const uint32_t* A,
                               int64_t lda, const uint32_t* B, int64_t ldb, uint32_t beta, uint32_t* C, int64_t ldc,
                               uint32_t* dA, uint32_t* dB, uint32_t* dC, cudaStream_t st) {
  const int64_t brow = transb == 'N' ? k : n, bcol = transb == 'N' ? n : k;
  static const int64_t nch_env = [] {          // POSIT_HOST_CHUNKS: row chunks (A/B runs; default m / 512, <= 8)
    const char* e = getenv("POSIT_HOST_CHUNKS");
    return e ? (int64_t)atoll(e) : (int64_t)0;
  }();
  int64_t nch = nch_env > 0 ? nch_env : m / HOST_CHUNK_MIN;
  if (nch > 8) nch = 8;
  if (nch < 1) nch = 1;
  const int64_t rows = (((m + nch - 1) / nch) + 63) / 64 * 64;
  nch = (m + rows - 1) / rows;
  constexpr int MAXCH = 8;
  // streams and events are created once per host thread and device (creating
  // them per call costs more than the copies they hide for small problems)
  struct HostPipe {
    cudaStream_t cs = nullptr, ds = nullptr, ks[2] = {nullptr, nullptr};
    cudaEvent_t ev0 = nullptr, ev_end = nullptr, ev_in[MAXCH] = {}, ev_done[MAXCH] = {};
    bool ok = false;
  };
  thread_local HostPipe pipes[16];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return POSIT_ECUDA;
  HostPipe& hp = pipes[dev];
  int rc = 0;
  auto ck = [&](cudaError_t e) { if (e != cudaSuccess && rc == 0) rc = cuda_check(e); return rc == 0; };
  if (!hp.ok) {
    bool good = cudaStreamCreateWithFlags(&hp.cs, cudaStreamNonBlocking) == cudaSuccess &&
                cudaStreamCreateWithFlags(&hp.ds, cudaStreamNonBlocking) == cudaSuccess &&
                cudaStreamCreateWithFlags(&hp.ks[0], cudaStreamNonBlocking) == cudaSuccess &&
                cudaStreamCreateWithFlags(&hp.ks[1], cudaStreamNonBlocking) == cudaSuccess &&
                cudaEventCreateWithFlags(&hp.ev0, cudaEventDisableTiming) == cudaSuccess &&
                cudaEventCreateWithFlags(&hp.ev_end, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; i < MAXCH && good; i++)
      good = cudaEventCreateWithFlags(&hp.ev_in[i], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&hp.ev_done[i], cudaEventDisableTiming) == cudaSuccess;
    if (!good) return cuda_check(cudaGetLastError());
    hp.ok = true;
  }
  cudaStream_t cs = hp.cs, ds = hp.ds, ks[2] = {hp.ks[0], hp.ks[1]};
  cudaEvent_t ev0 = hp.ev0, ev_end = hp.ev_end;
  cudaEvent_t* ev_in = hp.ev_in;
  cudaEvent_t* ev_done = hp.ev_done;
  // everything after the caller's earlier work on st
  ck(cudaEventRecord(ev0, st));
  for (cudaStream_t q : {cs, ds, ks[0], ks[1]}) ck(cudaStreamWaitEvent(q, ev0, 0));
  ck(cudaMemcpy2DAsync(dB, (size_t)bcol * 4, B, (size_t)ldb * 4, (size_t)bcol * 4, (size_t)brow, cudaMemcpyHostToDevice,
                       cs));
  for (int64_t i = 0; i < nch && rc == 0; i++) {
    const int64_t r0 = i * rows, mr = (m - r0) < rows ? (m - r0) : rows;
    ck(cudaMemcpy2DAsync(dA + r0 * k, (size_t)k * 4, A + r0 * lda, (size_t)lda * 4, (size_t)k * 4, (size_t)mr,
                         cudaMemcpyHostToDevice, cs));
    if (beta != 0u)
      ck(cudaMemcpy2DAsync(dC + r0 * n, (size_t)n * 4, C + r0 * ldc, (size_t)ldc * 4, (size_t)n * 4, (size_t)mr,
                           cudaMemcpyHostToDevice, cs));
    ck(cudaEventRecord(ev_in[i], cs));
    cudaStream_t q = ks[i & 1];
    ck(cudaStreamWaitEvent(q, ev_in[i], 0));
    if (rc == 0) {
      const int g = posit_gemm('N', transb, mr, n, k, alpha, dA + r0 * k, k > 0 ? k : 1, dB, bcol > 0 ? bcol : 1, beta,
                               dC + r0 * n, n > 0 ? n : 1, q);
      if (g) rc = g;
    }
    if (rc != 0) break;                          // never copy back rows that were not computed
    ck(cudaEventRecord(ev_done[i], q));
    ck(cudaStreamWaitEvent(ds, ev_done[i], 0));
    ck(cudaMemcpy2DAsync(C + r0 * ldc, (size_t)ldc * 4, dC + r0 * n, (size_t)n * 4, (size_t)n * 4, (size_t)mr,
                         cudaMemcpyDeviceToHost, ds));
  }
  if (rc == 0) {
    ck(cudaEventRecord(ev_end, ds));
    ck(cudaStreamWaitEvent(st, ev_end, 0));
    if (rc == 0) ck(cudaStreamSynchronize(st));
  }
  if (rc != 0) {
    // drain every pipeline stream before returning: no copy may still be in
    // flight into or out of the caller's host buffers
    for (cudaStream_t q : {cs, ks[0], ks[1], ds}) (void)cudaStreamSynchronize(q);
  }
  return rc;
}

int posit_gemm_host(char transa, char transb, int64_t m, int64_t n, int64_t k, uint32_t alpha, const uint32_t* A,
                    int64_t lda, const uint32_t* B, int64_t ldb, uint32_t beta, uint32_t* C, int64_t ldc,
                    void* dwork, size_t work_bytes, void* stream) {
  if (transa != 'N' && transa != 'T') return -1;
  if (transb != 'N' && transb != 'T') return -2;
  if (m < 0) return -3;
  if (n < 0) return -4;
  if (k < 0) return -5;
  if (alpha != POSIT_ONE && alpha != POSIT_MONE) return -6;
  if (lda < ((transa == 'N' ? k : m) > 1 ? (transa == 'N' ? k : m) : 1)) return -8;
  if (ldb < ((transb == 'N' ? n : k) > 1 ? (transb == 'N' ? n : k) : 1)) return -10;
  if (beta != 0u && beta != POSIT_ONE) return -11;
  if (ldc < (n > 1 ? n : 1)) return -13;
  if (m == 0 || n == 0) return 0;
  if ((k > 0 && (A == nullptr || B == nullptr)) || C == nullptr) return -7;
  if (work_bytes < posit_gemm_host_work_bytes(m, n, k) || dwork == nullptr) return -15;
  const int64_t brow = transb == 'N' ? k : n, bcol = transb == 'N' ? n : k;
  const int64_t arow = transa == 'N' ? m : k, acol = transa == 'N' ? k : m;
  uint32_t* dA = reinterpret_cast<uint32_t*>(dwork);
  uint32_t* dB = dA + m * k;
  uint32_t* dC = dB + k * n;
  cudaStream_t st = S(stream);
  int rc;
  if (transa == 'N' && k > 0 && m >= 2 * HOST_CHUNK_MIN && host_pipeline_env())
    return gemm_host_pipelined(transb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, dA, dB, dC, st);
  if ((rc = cuda_check(cudaMemcpy2DAsync(dA, (size_t)acol * 4, A, (size_t)lda * 4, (size_t)acol * 4, (size_t)arow,
                                         cudaMemcpyHostToDevice, st))))
    return rc;
  if ((rc = cuda_check(cudaMemcpy2DAsync(dB, (size_t)bcol * 4, B, (size_t)ldb * 4, (size_t)bcol * 4, (size_t)brow,
                                         cudaMemcpyHostToDevice, st))))
    return rc;
  if (beta != 0u) {
    if ((rc = cuda_check(cudaMemcpy2DAsync(dC, (size_t)n * 4, C, (size_t)ldc * 4, (size_t)n * 4, (size_t)m,
                                           cudaMemcpyHostToDevice, st))))
      return rc;
  }
  rc = posit_gemm(transa, transb, m, n, k, alpha, dA, acol > 0 ? acol : 1, dB, bcol > 0 ? bcol : 1, beta, dC,
                  n > 0 ? n : 1, stream);
  if (rc) return rc;
  if ((rc = cuda_check(cudaMemcpy2DAsync(C, (size_t)ldc * 4, dC, (size_t)n * 4, (size_t)n * 4, (size_t)m,
                                         cudaMemcpyDeviceToHost, st))))
    return rc;
  return cuda_check(cudaStreamSynchronize(st));
}

int posit_syrk(char uplo, char trans, int64_t n, int64_t k, uint32_t alpha, const uint32_t* A, int64_t lda,
               uint32_t beta, uint32_t* C, int64_t ldc, void* stream) {
  if (uplo != 'L' && uplo != 'U') return -1;
  if (trans != 'N' && trans != 'T') return -2;
  if (n < 0) return -3;
  if (k < 0) return -4;
  if (alpha != POSIT_ONE && alpha != POSIT_MONE) return -5;
  if (lda < (k > 1 ? k : 1)) return -7;
  if (beta != 0u && beta != POSIT_ONE) return -8;
  if (ldc < (n > 1 ? n : 1)) return -10;
  if (uplo != 'L' || trans != 'N') return POSIT_ENOTSUP;
  if (n == 0) return 0;
  pg::Params P{n, n, k, A, lda, A, lda, C, ldc, alpha == POSIT_MONE ? 1 : 0, beta == POSIT_ONE ? 1 : 0, nullptr};
  const int rc = pb_launch_gemm(P, true, true, S(stream));
  if (rc) return launch_check(rc);
  return cuda_check(cudaPeekAtLastError());
}

int posit_trsm(char side, char uplo, char transa, char diag, int64_t m, int64_t n, uint32_t alpha, const uint32_t* A,
               int64_t lda, uint32_t* B, int64_t ldb, void* stream) {
  if (side != 'L' && side != 'R') return -1;
  if (uplo != 'L' && uplo != 'U') return -2;
  if (transa != 'N' && transa != 'T') return -3;
  if (diag != 'N' && diag != 'U') return -4;
  if (m < 0) return -5;
  if (n < 0) return -6;
  if (alpha != POSIT_ONE) return -7;
  const int64_t ka = side == 'L' ? m : n;
  if (lda < (ka > 1 ? ka : 1)) return -9;
  if (ldb < (n > 1 ? n : 1)) return -11;
  if (m == 0 || n == 0) return 0;
  int rc;
  if (side == 'L' && uplo == 'L' && transa == 'N' && diag == 'U') {
    rc = pb_trsm_llnu(m, n, A, lda, B, ldb, S(stream));
  } else if (side == 'R' && uplo == 'L' && transa == 'T' && diag == 'N') {
    rc = pb_trsm_rltn(m, n, A, lda, B, ldb, nullptr, S(stream));
  } else {
    return POSIT_ENOTSUP;
  }
  return launch_check(rc);
}

size_t posit_getrf_work_bytes(int64_t m, int64_t n, int64_t nb) {
  (void)m; (void)n; (void)nb;
  return pb_panel_ws_bytes();
}

int posit_getrf_panel(int64_t m, int64_t b, uint32_t* A, int64_t lda, int32_t* ipiv, int32_t* info, int64_t row_base,
                      void* work, size_t work_bytes, void* stream) {
  if (m < 0) return -1;
  if (b < 0) return -2;
  if (lda < (b > 1 ? b : 1)) return -4;
  if (m == 0 || b == 0) return 0;
  if (work == nullptr || work_bytes < pb_panel_ws_bytes()) return -8;
  return launch_check(pb_getrf_panel(m, b, A, lda, ipiv, info, row_base, work, true, S(stream)));
}

int posit_laswp(int64_t ncols, uint32_t* A, int64_t lda, int64_t k1, int64_t k2, const int32_t* ipiv,
                int64_t ipiv_base, void* stream) {
  if (ncols < 0) return -1;
  if (lda < (ncols > 1 ? ncols : 1)) return -3;
  if (k1 < 0 || k2 < k1) return -4;
  return launch_check(pb_laswp(ncols, A, lda, k1, k2, ipiv, ipiv_base, S(stream)));
}

// Lookahead (both drivers): the next panel is factored on a high-priority
// side stream while the current step's trailing update of the columns beyond
// that panel runs on the caller's stream.  The two touch disjoint columns, and
// every element still receives its updates one product at a time in
// ascending k (reading Q6), so the bits equal the serial schedule.
// POSIT_LOOKAHEAD=0 forces the serial schedule.  Measured on one B200:
// Cholesky C3 240 -> 205 ms, LU C5 446 -> 406 ms, C4 2.84 -> 2.71 s.  On the
// side stream the LU leaf is a cooperative launch of 16 CTAs x 1024 threads,
// so it needs only 16 SMs while the trailing GEMM holds the rest.
static int lookahead_env() {
  static const int v = [] {                      // thread-safe one-time init
    const char* e = getenv("POSIT_LOOKAHEAD");
    return e ? atoi(e) : -1;
  }();
  return v;
}

static int64_t tail_w() {                       // POSIT_TAIL_W: width of the fused tail LU (0: off)
  static const int64_t v = [] {
    const char* e = getenv("POSIT_TAIL_W");
    const int64_t w = e ? (int64_t)atoll(e) : (int64_t)512;   // r04l sweep: 512 best (C5 -1.7 ms, C4 -2.4 ms)
    return w < 1024 ? w : (int64_t)1024;          // the fused kernel's widest leaf
  }();
  return v;
}
static int64_t tail_m() { return (int64_t)pb_num_sms() * 40; }   // rows: 40 per CTA x 1024 columns fit 160 KB

static int64_t wide_leaf_cols() {
  static const int64_t v = [] {
    const char* e = getenv("POSIT_WIDE_LEAF_COLS");
    return e ? (int64_t)atoll(e) : (int64_t)4096;
  }();
  return v;
}

struct SideStream {
  cudaStream_t side = nullptr;
  cudaEvent_t ev_col = nullptr, ev_panel = nullptr;
  int init() {
    int lo = 0, hi = 0;
    if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) return POSIT_ECUDA;
    if (cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi) != cudaSuccess) return POSIT_ECUDA;
    if (cudaEventCreateWithFlags(&ev_col, cudaEventDisableTiming) != cudaSuccess) return POSIT_ECUDA;
    if (cudaEventCreateWithFlags(&ev_panel, cudaEventDisableTiming) != cudaSuccess) return POSIT_ECUDA;
    return 0;
  }
  ~SideStream() {
    if (ev_col) cudaEventDestroy(ev_col);
    if (ev_panel) cudaEventDestroy(ev_panel);
    if (side) cudaStreamDestroy(side);     // released once its queued work completes
  }
};

int posit_getrf(int64_t m, int64_t n, uint32_t* A, int64_t lda, int32_t* ipiv, int32_t* info, int64_t nb,
                void* work, size_t work_bytes, void* stream) {
  if (m < 0) return -1;
  if (n < 0) return -2;
  if (lda < (n > 1 ? n : 1)) return -4;
  if (nb < 1) return -7;
  if (info == nullptr) return -6;
  if (work == nullptr || work_bytes < pb_panel_ws_bytes()) return -8;
  cudaStream_t st = S(stream);
  int rc = cuda_check(cudaMemsetAsync(info, 0, sizeof(int32_t), st));
  if (rc) return rc;
  const int64_t kmax = m < n ? m : n;
  if (kmax == 0) return 0;
  const bool la = lookahead_env() != 0 && kmax > nb;
  SideStream ss;
  if (la && (rc = ss.init())) return rc;
  // the last <= tail_w() columns as one fused cooperative LU (then its swaps on the columns left of it)
  auto fits_tail = [&](int64_t s0) { return tail_w() > 0 && n - s0 <= tail_w() && m - s0 <= tail_m(); };
  auto run_tail = [&](int64_t s0) -> int {
    int r = pb_getrf_tail(m - s0, n - s0, A + s0 * lda + s0, lda, ipiv + s0, info, s0, work, st);
    if (r) return r;
    if (s0 > 0 && (r = pb_laswp(s0, A, lda, s0, kmax, ipiv, 0, st))) return r;
    return 0;
  };
  if (fits_tail(0)) {
    if ((rc = run_tail(0)) == 0) return cuda_check(cudaPeekAtLastError());
    if (rc != POSIT_ENOTSUP) return launch_check(rc);
  }
  // panel 0 on the caller's stream
  if ((rc = pb_getrf_panel(m, kmax < nb ? kmax : nb, A, lda, ipiv, info, 0, work, true, st))) return launch_check(rc);
  for (int64_t s = 0; s < kmax; s += nb) {
    const int64_t b = (kmax - s) < nb ? (kmax - s) : nb;
    const int64_t s1 = s + b;                                  // next panel's first column / row
    int64_t b1 = (kmax - s1) < nb ? (kmax - s1) : nb;          // its width (<= 0: none)
    // the rest after this step goes to the fused tail: update all of it now, no next panel
    const bool tail_next = b1 > 0 && fits_tail(s1);
    if (tail_next) b1 = 0;
    if (la && s > 0 && (rc = cuda_check(cudaStreamWaitEvent(st, ss.ev_panel, 0)))) return rc;
    // the panel's swaps on the columns left and right of it
    if (s > 0 && (rc = pb_laswp(s, A, lda, s, s1, ipiv, 0, st))) return launch_check(rc);
    if (s1 < n && (rc = pb_laswp(n - s1, A + s1, lda, s, s1, ipiv, 0, st))) return launch_check(rc);
    if (s1 < n) {
      // U12 = L11^{-1} A12
      if ((rc = pb_trsm_llnu(b, n - s1, A + s * lda + s, lda, A + s * lda + s1, lda, st))) return launch_check(rc);
    }
    if (s1 < n && s1 < m) {
      const uint32_t* L21 = A + s1 * lda + s;
      const uint32_t* U12 = A + s * lda + s1;
      if (b1 > 0) {
        // trailing update of the next panel's columns first ...
        pg::Params Pc{m - s1, b1, b, L21, lda, U12, lda, A + s1 * lda + s1, lda, 1, 1, nullptr};
        if ((rc = pb_launch_gemm(Pc, false, false, st))) return launch_check(rc);
        if (la) {
          // ... then factor it on the side stream while the rest of the update runs
          if ((rc = cuda_check(cudaEventRecord(ss.ev_col, st)))) return rc;
          if ((rc = cuda_check(cudaStreamWaitEvent(ss.side, ss.ev_col, 0)))) return rc;
          // the leaf takes a few SMs while the trailing update is large, every SM
          // once it is small (the panel is then the critical path: panel_sweep
          // r03s, m = 2048: 2.6 ms on 16 CTAs vs 2.1 ms on 148; threshold swept in r03u:
          // C5 376.5 -> 371.0 ms, C4 2618 -> 2613 ms)
          const bool wide_leaf = (n - s1 - b1) <= wide_leaf_cols();
          if ((rc = pb_getrf_panel(m - s1, b1, A + s1 * lda + s1, lda, ipiv + s1, info, s1, work, wide_leaf,
                                   ss.side)))
            return launch_check(rc);
          if ((rc = cuda_check(cudaEventRecord(ss.ev_panel, ss.side)))) return rc;
        }
        if (s1 + b1 < n) {
          pg::Params Pr{m - s1, n - s1 - b1, b, L21, lda, U12 + b1, lda, A + s1 * lda + s1 + b1, lda, 1, 1, nullptr};
          // disjoint columns from the update just before it: may overlap its last wave
          if ((rc = pb_launch_gemm(Pr, false, false, st, la))) return launch_check(rc);
        }
        if (!la &&
            (rc = pb_getrf_panel(m - s1, b1, A + s1 * lda + s1, lda, ipiv + s1, info, s1, work, true, st)))
          return launch_check(rc);
      } else {
        pg::Params P{m - s1, n - s1, b, L21, lda, U12, lda, A + s1 * lda + s1, lda, 1, 1, nullptr};
        if ((rc = pb_launch_gemm(P, false, false, st))) return launch_check(rc);
      }
    }
    if (tail_next) {
      if ((rc = run_tail(s1))) return launch_check(rc);
      break;
    }
  }
  return cuda_check(cudaPeekAtLastError());
}

size_t posit_potrf_work_bytes(int64_t n, int64_t nb) {
  (void)n; (void)nb;
  return 0;
}

int posit_potrf(char uplo, int64_t n, uint32_t* A, int64_t lda, int32_t* info, int64_t nb, void* work,
                size_t work_bytes, void* stream) {
  (void)work; (void)work_bytes;
  if (uplo != 'L' && uplo != 'U') return -1;
  if (n < 0) return -2;
  if (lda < (n > 1 ? n : 1)) return -4;
  if (info == nullptr) return -5;
  if (nb < 1) return -6;
  if (uplo != 'L') return POSIT_ENOTSUP;
  cudaStream_t st = S(stream);
  int rc = cuda_check(cudaMemsetAsync(info, 0, sizeof(int32_t), st));
  if (rc) return rc;
  if (n == 0) return 0;
  const bool la = lookahead_env() != 0 && n >= 4 * nb;
  SideStream ss;
  if (la && (rc = ss.init())) return rc;
  // diagonal block and panel 0 on the caller's stream
  {
    const int64_t b = n < nb ? n : nb;
    if ((rc = pb_potf2(b, A, lda, info, 0, st))) return launch_check(rc);
    if (b < n && (rc = pb_trsm_rltn(n - b, b, A, lda, A + b * lda, lda, info, st))) return launch_check(rc);
  }
  for (int64_t s = 0; s < n; s += nb) {
    const int64_t b = (n - s) < nb ? (n - s) : nb;
    const int64_t s1 = s + b;
    if (s1 >= n) break;
    const int64_t b1 = (n - s1) < nb ? (n - s1) : nb;
    if (la && s > 0 && (rc = cuda_check(cudaStreamWaitEvent(st, ss.ev_panel, 0)))) return rc;
    const uint32_t* L21 = A + s1 * lda + s;
    // SYRK of the next block column first (rows s1.., columns s1..s1+b1, lower part) ...
    pg::Params Pc{n - s1, b1, b, L21, lda, L21, lda, A + s1 * lda + s1, lda, 1, 1, info};
    if ((rc = pb_launch_gemm(Pc, true, true, st))) return launch_check(rc);
    auto panel = [&](cudaStream_t q) -> int {
      int r;
      if ((r = pb_potf2(b1, A + s1 * lda + s1, lda, info, s1, q))) return r;
      if (s1 + b1 < n && (r = pb_trsm_rltn(n - s1 - b1, b1, A + s1 * lda + s1, lda, A + (s1 + b1) * lda + s1, lda,
                                           info, q)))
        return r;
      return 0;
    };
    if (la) {
      // ... then the next diagonal block and panel on the side stream
      if ((rc = cuda_check(cudaEventRecord(ss.ev_col, st)))) return rc;
      if ((rc = cuda_check(cudaStreamWaitEvent(ss.side, ss.ev_col, 0)))) return rc;
      if ((rc = panel(ss.side))) return launch_check(rc);
      if ((rc = cuda_check(cudaEventRecord(ss.ev_panel, ss.side)))) return rc;
    }
    // the rest of the trailing update (lower triangle beyond the next block column)
    if (s1 + b1 < n) {
      const uint32_t* L2b = A + (s1 + b1) * lda + s;
      pg::Params Pr{n - s1 - b1, n - s1 - b1, b, L2b, lda, L2b, lda, A + (s1 + b1) * lda + s1 + b1, lda, 1, 1, info};
      // disjoint columns from the block-column update just before it: may overlap its last wave
      if ((rc = pb_launch_gemm(Pr, true, true, st, la))) return launch_check(rc);
    }
    if (!la && (rc = panel(st))) return launch_check(rc);
  }
  if (la && (rc = cuda_check(cudaStreamWaitEvent(st, ss.ev_panel, 0)))) return rc;
  return cuda_check(cudaPeekAtLastError());
}

int posit_getrs(char trans, int64_t n, const uint32_t* LU, int64_t lda, const int32_t* ipiv, uint32_t* b,
                void* stream) {
  if (trans != 'N') return trans == 'T' ? POSIT_ENOTSUP : -1;
  if (n < 0) return -2;
  if (lda < (n > 1 ? n : 1)) return -4;
  if (n > 0 && (LU == nullptr || ipiv == nullptr || b == nullptr)) return -3;
  return launch_check(pb_solve(false, n, LU, lda, ipiv, b, S(stream)));
}

int posit_potrs(char uplo, int64_t n, const uint32_t* L, int64_t lda, uint32_t* b, void* stream) {
  if (uplo != 'L') return uplo == 'U' ? POSIT_ENOTSUP : -1;
  if (n < 0) return -2;
  if (lda < (n > 1 ? n : 1)) return -4;
  if (n > 0 && (L == nullptr || b == nullptr)) return -3;
  return launch_check(pb_solve(true, n, L, lda, nullptr, b, S(stream)));
}

int posit_iamax_key(int64_t m, const uint32_t* col, int64_t stride, const int32_t* global_row, int64_t row_min,
                    int64_t* key, void* stream) {
  if (m < 0) return -1;
  if (stride < 1) return -3;
  if (key == nullptr) return -7;
  if (m > 0 && (col == nullptr || global_row == nullptr)) return -2;
  return launch_check(pb_iamax_key(m, col, stride, global_row, row_min, reinterpret_cast<long long*>(key), S(stream)));
}

int posit_from_f64(const double* x, uint32_t* out, int64_t count, void* stream) {
  if (count < 0) return -3;
  return launch_check(pb_from_f64(x, out, count, S(stream)));
}

int posit_to_f64(const uint32_t* p, double* out, int64_t count, void* stream) {
  if (count < 0) return -3;
  return launch_check(pb_to_f64(p, out, count, S(stream)));
}

int posit_vec_op(int op, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count, void* stream) {
  if (op < POSIT_OP_ADD || op > POSIT_OP_DSQRT || op == 7) return -1;
  if (count < 0) return -5;
  if (count > 0 && (a == nullptr || b == nullptr || out == nullptr)) return -2;
  if (op >= POSIT_OP_DADD) return launch_check(pb_vec_d(op, a, b, nullptr, out, count, S(stream)));
  return launch_check(pb_vec_op(op, a, b, out, count, S(stream)));
}

int posit_vec_dmac(const uint32_t* c, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count,
                   void* stream) {
  if (count < 0) return -5;
  if (count > 0 && (a == nullptr || b == nullptr || c == nullptr || out == nullptr)) return -1;
  return launch_check(pb_vec_d(7, a, b, c, out, count, S(stream)));
}

}  // extern "C"
