// internal.h -- declarations shared by the .cu files of libposit_b200 (not public).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/posit_b200.h"

#define PB_ERR_TOO_LARGE POSIT_ENOTSUP

namespace pg { struct Params; }

// pdl: programmatic dependent launch after the previous kernel on st (only for
// an update that does not read that kernel's output)
int pb_launch_gemm(const pg::Params& P, bool transb, bool syrk, cudaStream_t st, bool pdl = false);
int pb_launch_gemm_d(const pg::Params& P, bool transb, bool syrk, cudaStream_t st, bool pdl, int variant);   // gemm_d.cu
int pb_vec_d(int op, const uint32_t* a, const uint32_t* b, const uint32_t* c, uint32_t* out, int64_t count,
             cudaStream_t st);
int pb_launch_gemm_naive(const pg::Params& P, bool transb, bool syrk, cudaStream_t st);
int pb_launch_gemm_tiny(const pg::Params& P, bool transb, bool syrk, cudaStream_t st);   // chol.cu

// leaf.cu, swap.cu, trsm.cu, chol.cu, misc.cu
int pb_getrf_panel(int64_t m, int64_t b, uint32_t* A, int64_t lda, int32_t* ipiv, int32_t* info,
                   int64_t row_base, void* ws, bool allow_coop, cudaStream_t st);
size_t pb_panel_ws_bytes();
int pb_getrf_tail(int64_t m, int64_t w, uint32_t* A, int64_t lda, int32_t* ipiv, int32_t* info, int64_t row_base,
                  void* ws, cudaStream_t st);
int pb_laswp(int64_t ncols, uint32_t* A, int64_t lda, int64_t k1, int64_t k2, const int32_t* ipiv,
             int64_t ipiv_base, cudaStream_t st);
int pb_trsm_llnu(int64_t m, int64_t n, const uint32_t* L, int64_t ldl, uint32_t* B, int64_t ldb, cudaStream_t st);
int pb_trsm_rltn(int64_t m, int64_t n, const uint32_t* L, int64_t ldl, uint32_t* B, int64_t ldb,
                 const int32_t* stop_flag, cudaStream_t st);
int pb_potf2(int64_t b, uint32_t* A, int64_t lda, int32_t* info, int64_t row_base, cudaStream_t st);
int pb_solve(bool chol, int64_t n, const uint32_t* A, int64_t lda, const int32_t* ipiv, uint32_t* b, cudaStream_t st);
int pb_axpby(uint32_t alpha, const uint32_t* T, int64_t ldt, uint32_t beta, uint32_t* C, int64_t ldc, int64_t m,
             int64_t n, cudaStream_t st);
int pb_iamax_key(int64_t m, const uint32_t* col, int64_t stride, const int32_t* grow, int64_t row_min, long long* out,
                 cudaStream_t st);
int pb_vec_op(int op, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count, cudaStream_t st);
int pb_from_f64(const double* x, uint32_t* out, int64_t count, cudaStream_t st);
int pb_to_f64(const uint32_t* p, double* out, int64_t count, cudaStream_t st);
int pb_gemm_guarded(const pg::Params& P, bool transb, bool syrk, const int32_t* stop_flag, cudaStream_t st);

// POSIT_GEMM_PATH: 1 (default) = the binary64-pipe MAC (gemm_d.cuh, lanes_d.cuh)
// in every kernel that has it, 0 = the integer MAC everywhere (same bits)
bool pb_dpath();

// number of kernels this library has launched (posit_kernel_launches)
void pb_count_launch();

// Per-device facts and one-time init.  Kernel attributes (dynamic shared
// memory limits) and the SM count belong to a device, so everything cached is
// keyed by the current device (capi.cu), never by a process-wide static.
#include <mutex>
#include <utility>
constexpr int PB_MAX_DEVICES = 64;
int pb_device();             // current CUDA device (0 if the query fails)
int pb_num_sms();            // multiprocessor count of the current device (cached per device)
bool pb_coop_supported();    // cooperative launch support of the current device (cached per device)
struct PbOncePerDevice { std::once_flag flag[PB_MAX_DEVICES]; };
template <class F>
inline void pb_once_per_device(PbOncePerDevice& once, F&& fn) {
  const int d = pb_device();
  std::call_once(once.flag[d < PB_MAX_DEVICES ? d : PB_MAX_DEVICES - 1], std::forward<F>(fn));
}
