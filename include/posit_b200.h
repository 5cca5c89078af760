/*
 * posit_b200.h -- C ABI of libposit_b200.so: the Posit(32,2) hot path of the
 * paper's posit-accelerated dense LU and Cholesky (arxiv 2401.14117,
 * "Evaluation of POSIT Arithmetic with Accelerators") on NVIDIA B200 (sm_100a).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (LaTeX source), S:n = SPEC.md
 * line n; "Q<k>" = the reading of an ambiguous passage listed in DESIGN.md.
 *
 * Data.  Matrices are ROW-MAJOR arrays of uint32_t Posit(32,2) bit patterns
 * (Eq.1; 0x00000000 = 0, 0x80000000 = NaR, 0x40000000 = 1) with a
 * leading dimension ld >= number of columns (reading Q13: the paper's
 * MPLAPACK is column-major; BASELINE config 2 fixes row-major).  Element (i,j)
 * of X is X[i*ldx + j].  Pivot vectors are int32_t, 1-based (LAPACK).
 *
 * Arithmetic.  Every multiply and every add is one correctly rounded
 * Posit(32,2) operation: round to nearest, ties to even on the encoding (Q1),
 * saturating at +-maxpos / +-minpos (Q2), NaR absorbing, x/0 = NaR,
 * sqrt(x<0) = NaR (Q3).  There is no quire.  Order contract (Q6): every
 * output element receives its products one at a time in ascending k,
 *     c <- c (+/-) (a_ik (x) b_kj),
 * so blocked, tiled and distributed executions are bit-identical to the
 * textbook unblocked loops.
 *
 * Memory and streams.  Unless a function says HOST, every pointer is DEVICE
 * memory allocated and owned by the caller; the library keeps no hidden
 * persistent allocations.  `stream` is a cudaStream_t (NULL = legacy default
 * stream).  All work is enqueued asynchronously on `stream`; no function
 * synchronises the device except the *_host variants.  Results (including
 * *info and ipiv) are valid once the stream has reached the enqueued work.
 *
 * Return codes.  0 = enqueued successfully.  -i = the i-th argument is invalid
 * (LAPACK xerbla style).  POSIT_ENOTSUP = an unsupported option.  POSIT_ECUDA =
 * a CUDA launch/API error (text via posit_last_error()).  Numerical failure
 * (zero pivot, non-positive-definite minor) is never a return code: it is
 * written to *info on the device.  NaR inputs are legal and propagate.
 */
#ifndef POSIT_B200_H
#define POSIT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define POSIT_ABI_VERSION 2
#define POSIT_OK 0
#define POSIT_ENOTSUP (-100)
#define POSIT_ECUDA (-101)

#define POSIT_ONE 0x40000000u   /* +1 */
#define POSIT_MONE 0xC0000000u  /* -1 */
#define POSIT_NAR 0x80000000u

/* Library version (POSIT_ABI_VERSION). */
int posit_abi_version(void);

/* Number of CUDA kernels this library has launched in this process so far
 * (all entry points, all threads; a monotone counter for launch accounting). */
uint64_t posit_kernel_launches(void);

/* Static description of a return code. */
const char* posit_strerror(int code);

/* Text of the last CUDA error seen by this thread ("" if none). */
const char* posit_last_error(void);

/*
 * posit_gemm -- Eq.2: C <- alpha*op(A)*op(B) + beta*C in
 * Posit(32,2), op(X) = X ('N') or X^T ('T').  op(A) is m x k, op(B) is k x n,
 * C is m x n.  Per element: c <- (beta == 0 ? 0 : C_ij); for l = 0..k-1:
 * c <- c (+) (+/-(op(A)_il (x) op(B)_lj)), sign = sign(alpha); C_ij <- c.
 * With alpha = -1, beta = +1 this is the trailing-matrix update of the blocked
 * LU, the hot path.
 *   alpha  must be POSIT_ONE or POSIT_MONE (else -6); beta must be 0 or
 *          POSIT_ONE (else -11) (reading Q7).
 *   transa, transb 'N' or 'T' (the paper's four transpose variants):
 *   A is stored m x k ('N') or k x m ('T'), B k x n ('N') or n x k ('T').
 *   lda >= k ('N') or >= m ('T'), ldb >= n ('N') or >= k ('T'), ldc >= n.
 * C must not overlap A or B.
 */
int posit_gemm(char transa, char transb, int64_t m, int64_t n, int64_t k, uint32_t alpha,
               const uint32_t* A, int64_t lda, const uint32_t* B, int64_t ldb, uint32_t beta,
               uint32_t* C, int64_t ldc, void* stream);

/*
 * posit_gemm_eq2 -- Eq.2 for ANY alpha, beta in the order SPEC S:200 states:
 *   t = sum_l op(A)_il (x) op(B)_lj   accumulated from 0 in ascending l,
 *   C_ij <- (alpha (x) t) (+) (beta (x) C_ij)   (mul, mul, add),
 * every operation one correctly rounded Posit(32,2) op.  (posit_gemm keeps the
 * path's order, reading Q6: c <- c (-) a (x) b from C_ij; for alpha = -1,
 * beta = 1 the two orders round differently.)  work: DEVICE buffer of
 * posit_gemm_eq2_work_bytes(m, n) bytes for t (else -15).  Arguments and
 * layouts as posit_gemm.
 */
size_t posit_gemm_eq2_work_bytes(int64_t m, int64_t n);
int posit_gemm_eq2(char transa, char transb, int64_t m, int64_t n, int64_t k, uint32_t alpha,
                   const uint32_t* A, int64_t lda, const uint32_t* B, int64_t ldb, uint32_t beta,
                   uint32_t* C, int64_t ldc, void* work, size_t work_bytes, void* stream);

/* Same contract and result as posit_gemm, computed by a one-thread-per-output
 * kernel with the generic per-operation path (a parity cross-check; slow). */
int posit_gemm_naive(char transa, char transb, int64_t m, int64_t n, int64_t k, uint32_t alpha,
                     const uint32_t* A, int64_t lda, const uint32_t* B, int64_t ldb, uint32_t beta,
                     uint32_t* C, int64_t ldc, void* stream);

/* HOST variant of posit_gemm (end-to-end path): A, B, C are HOST arrays
 * (pinned memory recommended); `dwork` is a DEVICE workspace of at least
 * posit_gemm_host_work_bytes(m, n, k) bytes.  Copies A, B, C to the device,
 * runs posit_gemm, copies C back and synchronises `stream`.  With transa = 'N'
 * and m >= 1024 the work is pipelined in row chunks of C (internal streams and
 * events; B first, then each chunk's A and C rows up while the previous chunk
 * computes and the one before comes back); the result is bit-identical (row
 * chunks are independent outputs, Q6).  Returns after the copies complete.
 * The pipeline's four streams and events are created on first use per host
 * thread and device and kept for the process (no memory is held). */
size_t posit_gemm_host_work_bytes(int64_t m, int64_t n, int64_t k);
int posit_gemm_host(char transa, char transb, int64_t m, int64_t n, int64_t k, uint32_t alpha,
                    const uint32_t* A, int64_t lda, const uint32_t* B, int64_t ldb, uint32_t beta,
                    uint32_t* C, int64_t ldc, void* dwork, size_t work_bytes, void* stream);

/*
 * posit_syrk -- lower triangle of C (n x n) <- alpha*A*A^T + beta*C, A n x k
 * (uplo = 'L', trans = 'N' only), same per-element order as posit_gemm.  The
 * Cholesky trailing update.  The strict upper triangle of C is
 * neither read nor written.  alpha/beta as posit_gemm (-5 / -8).
 */
int posit_syrk(char uplo, char trans, int64_t n, int64_t k, uint32_t alpha, const uint32_t* A, int64_t lda,
               uint32_t beta, uint32_t* C, int64_t ldc, void* stream);

/*
 * posit_trsm -- triangular solve with multiple right-hand sides
 * (S:206-214), alpha must be POSIT_ONE (else -7).  Supported:
 *   side='L', uplo='L', transa='N', diag='U':  B (m x n) <- L^{-1} B, L m x m
 *       unit lower: b_ij <- b_ij (-) l_ik (x) b_kj, k = 0..i-1 ascending.
 *       (LU: U12 = L11^{-1} A12.)
 *   side='R', uplo='L', transa='T', diag='N':  B (m x n) <- B L^{-T}, L n x n
 *       lower: b_ij <- b_ij (-) b_ik (x) l_jk, k = 0..j-1 ascending, then
 *       b_ij <- b_ij (/) l_jj.  (Cholesky: L21 = A21 L11^{-T}.)
 * Other combinations return POSIT_ENOTSUP.  Only the referenced triangle of
 * A is read.
 */
int posit_trsm(char side, char uplo, char transa, char diag, int64_t m, int64_t n, uint32_t alpha,
               const uint32_t* A, int64_t lda, uint32_t* B, int64_t ldb, void* stream);

/*
 * posit_getrf -- blocked right-looking LU with partial pivoting of the m x n
 * matrix A, block size nb.  Result bit-identical
 * to the textbook kij loop: for k: p = argmax_{i>=k} abs(a_ik) by signed
 * compare of patterns, ties -> smallest i (Q10); ipiv[k] = p+1; if a_pk != 0
 * swap rows k and p across the full width and set a_ik <- a_ik (/) a_kk
 * (one posit division, Q8) for i > k, else *info = first such k+1 (Q11, the
 * factorisation continues); a_ij <- a_ij (-) a_ik (x) a_kj for i,j > k.
 * On exit A holds L (unit, strictly lower) and U; ipiv (length min(m,n)) and
 * info are DEVICE int32.  work is a DEVICE workspace of at least
 * posit_getrf_work_bytes(m, n, nb) bytes (pivot keys of the panel), owned by
 * the caller and not used concurrently by another call (else -8).
 */
size_t posit_getrf_work_bytes(int64_t m, int64_t n, int64_t nb);
int posit_getrf(int64_t m, int64_t n, uint32_t* A, int64_t lda, int32_t* ipiv, int32_t* info, int64_t nb,
                void* work, size_t work_bytes, void* stream);

/*
 * posit_getrf_panel -- unblocked LU with partial pivoting of the m x b panel
 * A (the panel step of posit_getrf; used by the multi-GPU driver).  The same
 * per-column operations as posit_getrf (pivot by signed compare of abs
 * patterns, Q10; one posit division per multiplier, Q8; zero pivot -> info,
 * Q11), i.e. LAPACK's getf2 step that MPLAPACK's Rgetrf runs on the host in
 * the paper.  Row swaps are applied inside the
 * panel only.  ipiv[j] receives row_base + p + 1
 * (1-based, offset by row_base); *info, if still 0, receives row_base + j + 1
 * at the first zero pivot.  work: DEVICE workspace of posit_getrf_work_bytes()
 * bytes (else -8).
 */
int posit_getrf_panel(int64_t m, int64_t b, uint32_t* A, int64_t lda, int32_t* ipiv, int32_t* info,
                      int64_t row_base, void* work, size_t work_bytes, void* stream);

/*
 * posit_laswp -- apply the row interchanges ipiv[k1..k2) in order to columns
 * [0, ncols) of A: for k = k1..k2-1, swap rows k and ipiv[k]-1-ipiv_base
 * (LAPACK laswp, the row-interchange step of the blocked Rgetrf, P:157,
 * P:505-516; "swap rows k and p across the full width").  Pure
 * data movement (bit copies, no arithmetic).  ipiv is DEVICE int32 with at
 * least k2 entries; rows k1..k2-1 and every ipiv[k]-1-ipiv_base must lie in
 * [0, number of rows of A).  Returns -i for a bad i-th argument.
 */
int posit_laswp(int64_t ncols, uint32_t* A, int64_t lda, int64_t k1, int64_t k2, const int32_t* ipiv,
                int64_t ipiv_base, void* stream);

/*
 * posit_potrf -- blocked right-looking Cholesky A = L L^T of the n x n SPD
 * matrix (uplo = 'L' only), block size nb.
 * Bit-identical to the textbook loop: for k: if signed(a_kk) <= 0 then
 * *info = k+1 and stop (Q9); a_kk <- sqrt(a_kk); a_ik <- a_ik (/) a_kk;
 * a_ij <- a_ij (-) a_ik (x) a_jk for k < j <= i.  The strict upper triangle is
 * not referenced.  After a failure only *info and the columns of the blocks
 * before the failing block are defined.
 */
size_t posit_potrf_work_bytes(int64_t n, int64_t nb);
int posit_potrf(char uplo, int64_t n, uint32_t* A, int64_t lda, int32_t* info, int64_t nb, void* work,
                size_t work_bytes, void* stream);

/*
 * posit_getrs / posit_potrs -- one right-hand side b (length n, DEVICE,
 * overwritten by x) solved with the factors of posit_getrf / posit_potrf:
 * the Rgetrs / Rpotrs of the paper's accuracy study.
 * getrs: b <- P b, L y = b (unit lower), U x = y.  potrs: L y = b, L^T x = y.
 * Order (reading Q21, reference-BLAS trsv): forward substitution gives each
 * element its updates in ascending k, back substitution in descending k;
 * every multiply, subtract and divide is one correctly rounded posit op.
 * trans must be 'N' / uplo 'L' (else POSIT_ENOTSUP); n <= 51200 (shared
 * memory, else POSIT_ENOTSUP).  Latency-bound single-CTA kernels: a report
 * tool, not the hot path.
 */
int posit_getrs(char trans, int64_t n, const uint32_t* LU, int64_t lda, const int32_t* ipiv, uint32_t* b,
                void* stream);
int posit_potrs(char uplo, int64_t n, const uint32_t* L, int64_t lda, uint32_t* b, void* stream);

/*
 * posit_iamax_key -- pivot search over m entries col[i * stride] whose rows
 * have global indices global_row[i] (DEVICE int32; the rows a rank owns in a
 * 2D block-cyclic layout): *key (DEVICE int64) <- max over i with
 * global_row[i] >= row_min of ((abs(col_i) + 2^31) << 31) | (2^31 - 1 -
 * global_row[i]), abs by two's complement compared as a signed int (reading
 * Q10: larger abs first, ties -> smaller row; NaR the minimum), 0 if none.
 * Non-negative, so a MAX all-reduce over ranks yields the global pivot.
 */
int posit_iamax_key(int64_t m, const uint32_t* col, int64_t stride, const int32_t* global_row, int64_t row_min,
                    int64_t* key, void* stream);

/* Conversions: binary64 -> posit rounds once (RNE), NaN/Inf -> NaR,
 * -0 -> 0, subnormals -> +-minpos; posit -> binary64 is exact (NaR -> NaN). */
int posit_from_f64(const double* x, uint32_t* out, int64_t count, void* stream);
int posit_to_f64(const uint32_t* p, double* out, int64_t count, void* stream);

/* Elementwise ops (Table tabrandom's Add/Mul/Div/Sqrt kernels):
 * out[i] = a[i] op b[i]; op: 0 add, 1 sub, 2 mul, 3 div, 4 sqrt (b unused). */
#define POSIT_OP_ADD 0
#define POSIT_OP_SUB 1
#define POSIT_OP_MUL 2
#define POSIT_OP_DIV 3
#define POSIT_OP_SQRT 4
/* The same add and mul computed by the binary64-pipe MAC's steps (the D-MAC,
 * DESIGN.md section 6): 5 = add (operands |scale| <= 75, else the generic add),
 * 6 = mul (operands |scale| <= 37, else the generic mul).  Same bits as 0 / 2:
 * they exist so the D-MAC's rounding can be checked against the oracle one
 * operation at a time (every product and every sum rounded). */
#define POSIT_OP_DADD 5
#define POSIT_OP_DMUL 6
/* The panel kernels' division and square root on the binary64 pipe (S:206-214:
 * the Cholesky column scale l_ik = a_ik (/) l_kk and l_kk = sqrt(a_kk)), for the
 * same one-operation check: 8 = div (dividend |scale| <= 91, divisor
 * |scale| <= 37: faithful quotient + exact residual -> round to odd -> lattice;
 * else the generic div), 9 = sqrt (a > 0, |scale| <= 75: correctly rounded root
 * + exact residual -> round to odd -> lattice; else the generic sqrt; b unused).
 * Same bits as 3 / 4.  (7 is posit_vec_dmac's internal code.) */
#define POSIT_OP_DDIV 8
#define POSIT_OP_DSQRT 9
int posit_vec_op(int op, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count, void* stream);

/* out[i] = c[i] (+) (a[i] (x) b[i]): one step of the trailing update's chain
 * (reading Q6), through the D-MAC when |Ea|, |Eb| <= 37 and
 * |Ec| <= 91 (nonzero operands), else the generic mul and add (same bits).
 * Device pointers, count elements each; stream-ordered. */
int posit_vec_dmac(const uint32_t* c, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count,
                   void* stream);

#ifdef __cplusplus
}
#endif

#endif /* POSIT_B200_H */
