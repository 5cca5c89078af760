/*
 * posit_oracle.c -- the CPU ORACLE for the Posit(32,2) hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path
 * (paper_2401_14117_b200/csrc); neither side includes the other.
 *
 * What it computes, and where the paper says so (P:n = /root/reference/PAPER.md
 * line n, S:n = SPEC.md line n, "SURVEY 8(c)" = the readings in SURVEY.md
 * section 8(c), repeated in DESIGN.md "Readings"):
 *
 *   value of a posit        Eq.1, P:123-138 (regime run k(r), u = 2^(2^es)),
 *                           exact fraction budget per S:39-45 (reading Q5).
 *   encode + rounding       P:146-151 ("the fraction is rounded using the new
 *                           f_s"); round-to-nearest-even on the ENCODING,
 *                           saturating at maxpos/minpos, S:67-75 (Q1, Q2).
 *   add / sub / mul         P:183, P:190 (SoftPosit add/mul ported); each is
 *                           the exact rational result rounded once.
 *   div / sqrt              Table tabrandom "Div"/"Sqrt";
 *                           exact result rounded once (Q3).
 *   from_f64 / to_f64       S:121-129.
 *   GEMM (Eq.2)  c <- (beta==0 ? 0 : C_ij); for l ascending:
 *                           c <- c (+/-) (a_il (x) b_lj)   (order contract Q6).
 *   SYRK (lower)            same per-element order, lower triangle only.
 *   TRSM                    forward/back substitution, ascending k.
 *   getrf                   textbook right-looking kij LU, partial pivoting,
 *                           one posit division per multiplier (Q8, Q10, Q11),
 *                           P:157.
 *   potrf (lower)           textbook right-looking Cholesky (Q9),
 *                           P:158.
 *
 * How it computes (deliberately unlike the GPU path): patterns are decoded by
 * a bit-by-bit regime scan (the sequential loop of P:150); every
 * operation forms the exact result as an integer N times 2^X in 128-bit
 * arithmetic and rounds by writing out the posit bit string
 * regime || exponent || fraction and applying RNE to its first n-1 bits
 * (SURVEY 8(c) c2).  Width-generic (n <= 32, es <= 3) so that posit(8,0) can
 * be checked exhaustively against the exact-rational checker (checker.py).
 *
 * Parallelism: OpenMP over independent output elements only, so each
 * element's operation sequence is exactly the serial one.
 */
#include <stdint.h>
#include <math.h>
#include <string.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

#define K_ZERO 0
#define K_NAR 1
#define K_NUM 2

typedef struct {
    int kind;      /* K_ZERO, K_NAR or K_NUM */
    int sign;      /* 1 if negative */
    int scale;     /* k * 2^es + e */
    int fbits;     /* fraction bits f_s actually present in the pattern */
    uint64_t sig;  /* (1 << fbits) | f   -> value = sig * 2^(scale - fbits) */
} pdec;

static uint32_t mask_n(int n) { return n == 32 ? 0xFFFFFFFFu : ((1u << n) - 1u); }

static int bitlen_u128(u128 x) {
    uint64_t hi = (uint64_t)(x >> 64), lo = (uint64_t)x;
    if (hi) return 128 - __builtin_clzll(hi);
    if (lo) return 64 - __builtin_clzll(lo);
    return 0;
}

/* ---- c1: the value of a pattern (Eq.1) ------------- */
static pdec p_decode(uint32_t p, int n, int es) {
    pdec d;
    memset(&d, 0, sizeof d);
    const uint32_t m = mask_n(n);
    p &= m;
    if (p == 0) { d.kind = K_ZERO; return d; }
    if (p == (1u << (n - 1))) { d.kind = K_NAR; return d; }
    d.kind = K_NUM;
    d.sign = (int)((p >> (n - 1)) & 1u);
    if (d.sign) p = (~p + 1u) & m;              /* negate first (Q4) */
    int i = n - 2;                               /* first bit after the sign */
    const int r = (int)((p >> i) & 1u);
    int run = 0;
    while (i >= 0 && (int)((p >> i) & 1u) == r) { run++; i--; }   /* k(r) */
    const int k = r ? run - 1 : -run;
    if (i >= 0) i--;                             /* the terminating bit */
    int e = 0;
    for (int j = 0; j < es; j++) {               /* missing exponent bits read as 0 */
        e <<= 1;
        if (i >= 0) { e |= (int)((p >> i) & 1u); i--; }
    }
    const int fs = i + 1;                        /* remaining bits are the fraction */
    const uint64_t f = fs > 0 ? (uint64_t)(p & (uint32_t)((1ull << fs) - 1ull)) : 0;
    d.scale = k * (1 << es) + e;
    d.fbits = fs;
    d.sig = (1ull << fs) | f;
    return d;
}

/* ---- c2: round an exact nonzero value (-1)^sign * N * 2^X to posit(n,es) --
 * Writes the unbounded bit string regime || e || fraction ("the size
 * of the exponent ... is encoded in the regime, and the fraction is rounded
 * using the new f_s"), keeps n-1 bits, round-to-nearest-even on the
 * encoding (Q1), saturates (Q2). */
typedef struct { u128 acc; int pos; int lost; } bitstr;

static void bs_append(bitstr* b, u128 bits, int len) {
    if (len <= 0) return;
    if (len <= b->pos) {
        b->acc |= bits << (b->pos - len);
        b->pos -= len;
    } else {
        const int drop = len - b->pos;
        if (b->pos > 0) b->acc |= bits >> drop;
        if (drop >= 128 ? bits != 0 : (bits & ((((u128)1) << drop) - 1)) != 0) b->lost = 1;
        b->pos = 0;
    }
}

static uint32_t p_encode(int sign, u128 N, int X, int n, int es) {
    const uint32_t m = mask_n(n);
    const int bl = bitlen_u128(N);
    const int scale = X + bl - 1;                /* floor(log2 |x|) */
    const int maxscale = (n - 2) << es;          /* maxpos = useed^(n-2) */
    const int is_pow2 = (N & (N - 1)) == 0;
    uint32_t p;
    if (scale >= maxscale) {
        p = m >> 1;                              /* |x| >= maxpos -> maxpos */
    } else if (scale < -maxscale || (scale == -maxscale && is_pow2)) {
        p = 1;                                   /* 0 < |x| <= minpos -> minpos */
    } else {
        const int useed_log = 1 << es;
        const int k = scale >> es;               /* floor(scale / 2^es) */
        const int e = scale - k * useed_log;
        bitstr b = {0, 128, 0};
        if (k >= 0) bs_append(&b, ((((u128)1) << (k + 1)) - 1) << 1, k + 2);  /* 1..1 0 */
        else        bs_append(&b, 1, -k + 1);                                  /* 0..0 1 */
        bs_append(&b, (u128)e, es);
        bs_append(&b, N & ((((u128)1) << (bl - 1)) - 1), bl - 1);              /* fraction */
        p = (uint32_t)(b.acc >> (128 - (n - 1)));
        const int guard = (int)((b.acc >> (128 - n)) & 1);
        const int sticky = b.lost || ((b.acc << n) != 0);
        if (guard && (sticky || (p & 1u))) p++;
    }
    return sign ? ((~p + 1u) & m) : p;
}

/* ---- c3: operations ------------------------------------------------------ */
static uint32_t nar_of(int n) { return 1u << (n - 1); }

uint32_t or_neg(uint32_t a, int n, int es) { (void)es; return (~a + 1u) & mask_n(n); }

uint32_t or_add(uint32_t a, uint32_t b, int n, int es) {
    const pdec x = p_decode(a, n, es), y = p_decode(b, n, es);
    if (x.kind == K_NAR || y.kind == K_NAR) return nar_of(n);
    if (x.kind == K_ZERO) return b & mask_n(n);
    if (y.kind == K_ZERO) return a & mask_n(n);
    const int Xx = x.scale - x.fbits, Xy = y.scale - y.fbits;
    if (Xx - Xy > 90 || Xy - Xx > 90) {
        /* One operand lies entirely more than 60 binades below the other.
         * Every rounding boundary (lattice point or midpoint) next to the
         * larger value B is a multiple of 2^(scale(B)-31) away from it, so the
         * exact sum B +/- |small| and the representative B +/- 2^(X_B-90) lie
         * strictly inside the same boundary-free interval: same rounding. */
        const pdec* B = (Xx > Xy) ? &x : &y;
        const pdec* S = (Xx > Xy) ? &y : &x;
        const u128 NB = ((u128)B->sig) << 90;
        const u128 N = (B->sign == S->sign) ? NB + 1 : NB - 1;
        return p_encode(B->sign, N, (Xx > Xy ? Xx : Xy) - 90, n, es);
    }
    const int X = Xx < Xy ? Xx : Xy;
    const u128 Nx = ((u128)x.sig) << (Xx - X);
    const u128 Ny = ((u128)y.sig) << (Xy - X);
    int sign;
    u128 N;
    if (x.sign == y.sign) { N = Nx + Ny; sign = x.sign; }
    else if (Nx >= Ny)    { N = Nx - Ny; sign = x.sign; }
    else                  { N = Ny - Nx; sign = y.sign; }
    if (N == 0) return 0;                        /* exact cancellation: the only zero */
    return p_encode(sign, N, X, n, es);
}

uint32_t or_sub(uint32_t a, uint32_t b, int n, int es) { return or_add(a, or_neg(b, n, es), n, es); }

uint32_t or_mul(uint32_t a, uint32_t b, int n, int es) {
    const pdec x = p_decode(a, n, es), y = p_decode(b, n, es);
    if (x.kind == K_NAR || y.kind == K_NAR) return nar_of(n);
    if (x.kind == K_ZERO || y.kind == K_ZERO) return 0;
    const u128 N = (u128)x.sig * (u128)y.sig;    /* exact, <= 62 bits */
    return p_encode(x.sign ^ y.sign, N, (x.scale - x.fbits) + (y.scale - y.fbits), n, es);
}

uint32_t or_div(uint32_t a, uint32_t b, int n, int es) {
    const pdec x = p_decode(a, n, es), y = p_decode(b, n, es);
    if (x.kind == K_NAR || y.kind == K_NAR || y.kind == K_ZERO) return nar_of(n);  /* Q3 */
    if (x.kind == K_ZERO) return 0;
    /* q = sig_x * 2^64 / sig_y has >= 34 integer bits; a nonzero remainder is
     * represented by the half-way point of (Q, Q+1), which holds no rounding
     * boundary because boundaries sit at integer multiples of >= 2^4 here. */
    const u128 num = ((u128)x.sig) << 64;
    const u128 Q = num / (u128)y.sig, R = num % (u128)y.sig;
    const u128 N = (Q << 1) | (R != 0);
    const int X = (x.scale - x.fbits) - (y.scale - y.fbits) - 64 - 1;
    return p_encode(x.sign ^ y.sign, N, X, n, es);
}

static u128 isqrt_u128(u128 v) {               /* largest r with r*r <= v, by bisection */
    u128 lo = 0, hi = ((u128)1) << 64;         /* v < 2^128 -> sqrt < 2^64 */
    while (hi - lo > 1) {
        const u128 mid = lo + ((hi - lo) >> 1);
        if (mid * mid <= v) lo = mid; else hi = mid;
    }
    return lo;
}

uint32_t or_sqrt(uint32_t a, int n, int es) {
    const pdec x = p_decode(a, n, es);
    if (x.kind == K_NAR || (x.kind == K_NUM && x.sign)) return nar_of(n);    /* Q3 */
    if (x.kind == K_ZERO) return 0;
    u128 S = x.sig;
    int X = x.scale - x.fbits;
    if (X & 1) { S <<= 1; X -= 1; }               /* make the exponent even */
    const u128 T = S << 80;                      /* S < 2^33 -> T < 2^113 */
    const u128 r = isqrt_u128(T);                /* >= 40 significant bits */
    const u128 N = (r << 1) | (r * r != T);      /* remainder -> half-way representative */
    return p_encode(0, N, X / 2 - 40 - 1, n, es);
}

uint32_t or_from_f64(double v, int n, int es) {
    if (isnan(v) || isinf(v)) return nar_of(n);
    if (v == 0.0) return 0;                      /* also -0.0 */
    int e;
    const double f = frexp(fabs(v), &e);          /* |v| = f * 2^e, f in [0.5, 1) */
    const uint64_t M = (uint64_t)ldexp(f, 53);    /* exact 53-bit integer */
    return p_encode(v < 0, (u128)M, e - 53, n, es);
}

double or_to_f64(uint32_t a, int n, int es) {
    const pdec x = p_decode(a, n, es);
    if (x.kind == K_NAR) return NAN;
    if (x.kind == K_ZERO) return 0.0;
    const double v = ldexp((double)x.sig, x.scale - x.fbits);
    return x.sign ? -v : v;
}

/* f_s of a pattern (for the paper's P:283-285 facts); -1 for zero/NaR */
int or_fraction_bits(uint32_t a, int n, int es) {
    const pdec x = p_decode(a, n, es);
    return x.kind == K_NUM ? x.fbits : -1;
}

int or_scale(uint32_t a, int n, int es) {
    const pdec x = p_decode(a, n, es);
    return x.kind == K_NUM ? x.scale : -100000;
}

/* ---- array helpers (tests and input conversion) ------------------------- */
int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void or_from_f64_array(const double* v, uint32_t* out, int64_t count, int n, int es) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; i++) out[i] = or_from_f64(v[i], n, es);
}

void or_to_f64_array(const uint32_t* p, double* out, int64_t count, int n, int es) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; i++) out[i] = or_to_f64(p[i], n, es);
}

/* op: 0 add, 1 sub, 2 mul, 3 div, 4 sqrt (b ignored), 5 neg (b ignored) */
void or_vec_op(int op, const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t count, int n, int es) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; i++) {
        switch (op) {
            case 0: out[i] = or_add(a[i], b[i], n, es); break;
            case 1: out[i] = or_sub(a[i], b[i], n, es); break;
            case 2: out[i] = or_mul(a[i], b[i], n, es); break;
            case 3: out[i] = or_div(a[i], b[i], n, es); break;
            case 4: out[i] = or_sqrt(a[i], n, es); break;
            default: out[i] = or_neg(a[i], n, es); break;
        }
    }
}

/* Exhaustive round trip over all 2^32 Posit(32,2) patterns:
 * returns the number of patterns p (other than NaR) with
 * from_f64(to_f64(p)) != p, plus the number of adjacent pairs whose values
 * are out of signed-integer order.  NaR must map to NaN and back. */
int64_t or_roundtrip_all32(int64_t* order_violations) {
    int64_t bad = 0, unordered = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad, unordered)
    for (int64_t i = 0; i < (1ll << 32); i++) {
        const uint32_t p = (uint32_t)i;
        const double v = or_to_f64(p, 32, 2);
        if (p == 0x80000000u) { if (!isnan(v) || or_from_f64(v, 32, 2) != p) bad++; continue; }
        if (or_from_f64(v, 32, 2) != p) bad++;
        const uint32_t q = p + 1u;                        /* next pattern in signed order */
        if (q != 0x80000000u && p != 0x7FFFFFFFu) {
            if (!(or_to_f64(q, 32, 2) > v)) unordered++;
        }
    }
    if (order_violations) *order_violations = unordered;
    return bad;
}

/* ---- c4: linear algebra in Posit(32,2), row-major, the order contract ---- */
#define P32_ONE 0x40000000u
#define P32_MONE 0xC0000000u
static inline uint32_t padd(uint32_t a, uint32_t b) { return or_add(a, b, 32, 2); }
static inline uint32_t psub(uint32_t a, uint32_t b) { return or_sub(a, b, 32, 2); }
static inline uint32_t pmul(uint32_t a, uint32_t b) { return or_mul(a, b, 32, 2); }
static inline uint32_t pdiv(uint32_t a, uint32_t b) { return or_div(a, b, 32, 2); }

/* Eq.2 with alpha in {+1,-1}, beta in {0,1} (Q7).  Returns 0, or -i for a bad
 * i-th argument (LAPACK style). */
int or_gemm(char transa, char transb, int64_t m, int64_t n, int64_t k, uint32_t alpha,
            const uint32_t* A, int64_t lda, const uint32_t* B, int64_t ldb, uint32_t beta,
            uint32_t* C, int64_t ldc) {
    if (transa != 'N' && transa != 'T') return -1;
    if (transb != 'N' && transb != 'T') return -2;
    if (m < 0) return -3;
    if (n < 0) return -4;
    if (k < 0) return -5;
    if (alpha != P32_ONE && alpha != P32_MONE) return -6;
    if (beta != 0u && beta != P32_ONE) return -11;
    const int neg = (alpha == P32_MONE);
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t i = 0; i < m; i++) {
        for (int64_t j = 0; j < n; j++) {
            uint32_t c = beta ? C[i * ldc + j] : 0u;
            for (int64_t l = 0; l < k; l++) {
                const uint32_t a = transa == 'N' ? A[i * lda + l] : A[l * lda + i];
                const uint32_t b = transb == 'N' ? B[l * ldb + j] : B[j * ldb + l];
                const uint32_t t = pmul(a, b);
                c = neg ? psub(c, t) : padd(c, t);
            }
            C[i * ldc + j] = c;
        }
    }
    return 0;
}

/* C_lower <- beta*C + alpha * A * A^T (trans 'N': A is n x k).  Upper untouched. */
/* Eq.2 in the order SPEC S:200 states for general alpha, beta:
 *   t = sum_l op(A)_il (x) op(B)_lj   accumulated from 0 in ascending l,
 *   C_ij <- (alpha (x) t) (+) (beta (x) C_ij)   (mul, mul, add; the beta term last).
 * (posit_gemm's path contract, Q6, is the other order: c <- c (-) a (x) b.) */
int or_gemm_eq2(char transa, char transb, int64_t m, int64_t n, int64_t k, uint32_t alpha,
                const uint32_t* A, int64_t lda, const uint32_t* B, int64_t ldb, uint32_t beta,
                uint32_t* C, int64_t ldc) {
    if (transa != 'N' && transa != 'T') return -1;
    if (transb != 'N' && transb != 'T') return -2;
    if (m < 0) return -3;
    if (n < 0) return -4;
    if (k < 0) return -5;
#pragma omp parallel for collapse(2) schedule(static)
    for (int64_t i = 0; i < m; i++) {
        for (int64_t j = 0; j < n; j++) {
            uint32_t t = 0u;
            for (int64_t l = 0; l < k; l++) {
                const uint32_t a = transa == 'N' ? A[i * lda + l] : A[l * lda + i];
                const uint32_t b = transb == 'N' ? B[l * ldb + j] : B[j * ldb + l];
                t = padd(t, pmul(a, b));
            }
            C[i * ldc + j] = padd(pmul(alpha, t), pmul(beta, C[i * ldc + j]));
        }
    }
    return 0;
}

int or_syrk_lower(int64_t n, int64_t k, uint32_t alpha, const uint32_t* A, int64_t lda,
                  uint32_t beta, uint32_t* C, int64_t ldc) {
    if (n < 0) return -3;
    if (k < 0) return -4;
    if (alpha != P32_ONE && alpha != P32_MONE) return -5;
    if (beta != 0u && beta != P32_ONE) return -8;
    const int neg = (alpha == P32_MONE);
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t i = 0; i < n; i++) {
        for (int64_t j = 0; j <= i; j++) {
            uint32_t c = beta ? C[i * ldc + j] : 0u;
            for (int64_t l = 0; l < k; l++) {
                const uint32_t t = pmul(A[i * lda + l], A[j * lda + l]);
                c = neg ? psub(c, t) : padd(c, t);
            }
            C[i * ldc + j] = c;
        }
    }
    return 0;
}

/* side L, lower, no transpose, unit diagonal: B (m x n) <- L^{-1} B, L m x m.
 * b_ij <- b_ij (-) l_ik (x) b_kj for k = 0..i-1 ascending (forward substitution). */
int or_trsm_llnu(int64_t m, int64_t n, const uint32_t* L, int64_t ldl, uint32_t* B, int64_t ldb) {
    if (m < 0) return -5;
    if (n < 0) return -6;
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; j++) {
        for (int64_t i = 0; i < m; i++) {
            uint32_t b = B[i * ldb + j];
            for (int64_t k = 0; k < i; k++) b = psub(b, pmul(L[i * ldl + k], B[k * ldb + j]));
            B[i * ldb + j] = b;
        }
    }
    return 0;
}

/* side R, lower, transpose, non-unit: B (m x n) <- B L^{-T}, L n x n.
 * b_ij <- b_ij (-) b_ik (x) l_jk for k = 0..j-1 ascending, then b_ij <- b_ij (/) l_jj. */
int or_trsm_rltn(int64_t m, int64_t n, const uint32_t* L, int64_t ldl, uint32_t* B, int64_t ldb) {
    if (m < 0) return -5;
    if (n < 0) return -6;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; i++) {
        for (int64_t j = 0; j < n; j++) {
            uint32_t b = B[i * ldb + j];
            for (int64_t k = 0; k < j; k++) b = psub(b, pmul(B[i * ldb + k], L[j * ldl + k]));
            B[i * ldb + j] = pdiv(b, L[j * ldl + j]);
        }
    }
    return 0;
}

static inline int32_t pabs_key(uint32_t a) {    /* abs by negation; compared as signed ints */
    const int32_t s = (int32_t)a;
    return s < 0 ? (int32_t)(~a + 1u) : s;       /* NaR stays INT32_MIN (the minimum) */
}

/* Textbook right-looking LU with partial pivoting, SURVEY 8(c) c4:
 *   p = argmax_{i>=k} abs(a_ik) (signed compare of patterns, ties -> smallest i)
 *   ipiv_k = p+1; if a_pk != 0: swap rows k,p (full width), a_ik <- a_ik (/) a_kk
 *   else info <- info or k+1
 *   a_ij <- a_ij (-) a_ik (x) a_kj for i > k, j > k                      */
/* or_getrf_steps runs this loop's steps k in [k0, k1) only, so that a long run
 * (configs[3], n = 16384) can be checkpointed between steps (A, ipiv, info)
 * and resumed; or_getrf is all steps from a zeroed info.  Same arithmetic. */
int or_getrf_steps(int64_t m, int64_t n, uint32_t* A, int64_t lda, int32_t* ipiv, int32_t* info, int64_t k0,
                   int64_t k1) {
    if (m < 0) return -1;
    if (n < 0) return -2;
    const int64_t kmax = m < n ? m : n;
    if (k1 > kmax) k1 = kmax;
    for (int64_t k = k0; k < k1; k++) {
        int64_t p = k;
        int32_t best = pabs_key(A[k * lda + k]);
        for (int64_t i = k + 1; i < m; i++) {
            const int32_t v = pabs_key(A[i * lda + k]);
            if (v > best) { best = v; p = i; }
        }
        ipiv[k] = (int32_t)(p + 1);
        if (A[p * lda + k] != 0u) {
            if (p != k) {
                for (int64_t j = 0; j < n; j++) {
                    const uint32_t t = A[k * lda + j]; A[k * lda + j] = A[p * lda + j]; A[p * lda + j] = t;
                }
            }
            const uint32_t piv = A[k * lda + k];
            for (int64_t i = k + 1; i < m; i++) A[i * lda + k] = pdiv(A[i * lda + k], piv);
        } else if (*info == 0) {
            *info = (int32_t)(k + 1);
        }
#pragma omp parallel for schedule(static)
        for (int64_t i = k + 1; i < m; i++) {
            const uint32_t l = A[i * lda + k];
            for (int64_t j = k + 1; j < n; j++) A[i * lda + j] = psub(A[i * lda + j], pmul(l, A[k * lda + j]));
        }
    }
    return 0;
}

int or_getrf(int64_t m, int64_t n, uint32_t* A, int64_t lda, int32_t* ipiv, int32_t* info) {
    if (m < 0) return -1;
    if (n < 0) return -2;
    *info = 0;
    return or_getrf_steps(m, n, A, lda, ipiv, info, 0, m < n ? m : n);
}

/* Textbook right-looking Cholesky, lower, SURVEY 8(c) c4 / Q9:
 *   if signed(a_kk) <= 0: info = k+1, stop;  a_kk <- sqrt(a_kk);
 *   a_ik <- a_ik (/) a_kk (i > k);  a_ij <- a_ij (-) a_ik (x) a_jk (k < j <= i). */
int or_potrf_lower(int64_t n, uint32_t* A, int64_t lda, int32_t* info) {
    if (n < 0) return -2;
    *info = 0;
    for (int64_t k = 0; k < n; k++) {
        if ((int32_t)A[k * lda + k] <= 0) { *info = (int32_t)(k + 1); return 0; }
        const uint32_t d = or_sqrt(A[k * lda + k], 32, 2);
        A[k * lda + k] = d;
        for (int64_t i = k + 1; i < n; i++) A[i * lda + k] = pdiv(A[i * lda + k], d);
#pragma omp parallel for schedule(dynamic, 16)
        for (int64_t i = k + 1; i < n; i++) {
            const uint32_t lik = A[i * lda + k];
            for (int64_t j = k + 1; j <= i; j++) A[i * lda + j] = psub(A[i * lda + j], pmul(lik, A[j * lda + k]));
        }
    }
    return 0;
}

/* Solves for the accuracy report (Rgetrs / Rpotrs), one RHS, in
 * Posit(32,2), in the loop order of the reference BLAS trsv that MPLAPACK's
 * Rtrsv follows (reading Q21): forward substitution receives its
 * updates in ascending k, back substitution in DESCENDING k (column-oriented
 * "x_j final, then update every x_i, i < j" for U x = y; the dot-product
 * form for L^T x = y, which runs i = n-1 .. j+1).  Written as the plain
 * per-element loops. */
int or_getrs(int64_t n, const uint32_t* LU, int64_t lda, const int32_t* ipiv, uint32_t* b) {
    for (int64_t k = 0; k < n; k++) {             /* apply P */
        const int64_t p = ipiv[k] - 1;
        if (p != k) { const uint32_t t = b[k]; b[k] = b[p]; b[p] = t; }
    }
    for (int64_t i = 0; i < n; i++)               /* L y = Pb, unit lower */
        for (int64_t k = 0; k < i; k++) b[i] = psub(b[i], pmul(LU[i * lda + k], b[k]));
    for (int64_t i = n - 1; i >= 0; i--) {        /* U x = y */
        for (int64_t k = n - 1; k > i; k--) b[i] = psub(b[i], pmul(LU[i * lda + k], b[k]));
        b[i] = pdiv(b[i], LU[i * lda + i]);
    }
    return 0;
}

int or_potrs_lower(int64_t n, const uint32_t* L, int64_t lda, uint32_t* b) {
    for (int64_t i = 0; i < n; i++) {             /* L y = b */
        for (int64_t k = 0; k < i; k++) b[i] = psub(b[i], pmul(L[i * lda + k], b[k]));
        b[i] = pdiv(b[i], L[i * lda + i]);
    }
    for (int64_t i = n - 1; i >= 0; i--) {        /* L^T x = y */
        for (int64_t k = n - 1; k > i; k--) b[i] = psub(b[i], pmul(L[k * lda + i], b[k]));
        b[i] = pdiv(b[i], L[i * lda + i]);
    }
    return 0;
}
