/*
 * checker_wide.c -- the exact-rational checker of oracle/checker.py, restated
 * in C with exact wide-integer comparisons, so that S:443's ">= 1e7 random
 * pairs" can be checked in seconds instead of days.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  It shares no code,
 * header, table or constant with the C oracle (posit_oracle.c) or with the
 * CUDA path, and it uses a different method from both:
 *
 *   value(p)   Eq.1 of the paper: sign, the regime run read bit by
 *              bit, es exponent bits (missing bits read as 0), the remaining
 *              bits as the fraction (reading Q5) -> an exact pair
 *              (M, X) with value = M * 2^X.
 *   rounding   the definition of checker.round_to_posit (reading Q1/Q2,
 *              SURVEY 8(c) c2), without any bit-string encoder: bisection
 *              over the signed order of patterns for the largest p
 *              with value(p) <= |x|; the midpoint between p and p+1 is the
 *              value of pattern 2p+1 read as a Posit(n+1, es); below -> p,
 *              above -> p+1, equal -> the even one.  |x| >= maxpos ->
 *              maxpos, 0 < |x| <= minpos -> minpos.
 *   ops        add / sub / mul / div: every comparison of a candidate value
 *              with the EXACT result is an exact integer comparison on
 *              768-bit integers (a + b, a * b, c * b <= a for the quotient);
 *              sqrt: c^2 <= a and m^2 <= a, also exact.
 *
 * Validated against checker.py (exact Fractions) in tests/test_oracle_wide.py
 * before it is used to pin the oracle.
 */
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NL 12                      /* 12 x 64 = 768-bit unsigned integers */
typedef struct { uint64_t w[NL]; } big;

static void big_set(big* r, uint64_t lo, uint64_t hi) { memset(r, 0, sizeof *r); r->w[0] = lo; r->w[1] = hi; }

static void big_shl(big* r, int s) {           /* r <<= s, 0 <= s < 640 */
    const int q = s / 64, b = s % 64;
    for (int i = NL - 1; i >= 0; i--) {
        uint64_t v = 0;
        if (i - q >= 0) v = r->w[i - q] << b;
        if (b && i - q - 1 >= 0) v |= r->w[i - q - 1] >> (64 - b);
        r->w[i] = v;
    }
}

static int big_cmp(const big* a, const big* b) {
    for (int i = NL - 1; i >= 0; i--)
        if (a->w[i] != b->w[i]) return a->w[i] < b->w[i] ? -1 : 1;
    return 0;
}

static void big_add(big* r, const big* a, const big* b) {
    unsigned __int128 c = 0;
    for (int i = 0; i < NL; i++) { c += (unsigned __int128)a->w[i] + b->w[i]; r->w[i] = (uint64_t)c; c >>= 64; }
}

static void big_sub(big* r, const big* a, const big* b) {     /* a >= b */
    uint64_t br = 0;
    for (int i = 0; i < NL; i++) {
        const uint64_t x = a->w[i], y = b->w[i];
        const uint64_t d = x - y - br;
        br = (x < y) || (x - y < br);
        r->w[i] = d;
    }
}

/* value = M * 2^X as the 768-bit integer M << (X - base) */
static void big_from(big* r, unsigned __int128 M, int X, int base) {
    big_set(r, (uint64_t)M, (uint64_t)(M >> 64));
    big_shl(r, X - base);
}

/* ---- Eq.1: the value of a posit(n, es) pattern, literally ---------------- */
enum { CW_ZERO = 0, CW_NAR = 1, CW_NUM = 2 };
typedef struct { int kind, sign; uint64_t M; int X; } val;

static val value(uint64_t p, int n, int es) {
    val v = {CW_NUM, 0, 0, 0};
    const uint64_t mask = (n == 64) ? ~0ull : ((1ull << n) - 1);
    p &= mask;
    if (p == 0) { v.kind = CW_ZERO; return v; }
    if (p == (1ull << (n - 1))) { v.kind = CW_NAR; return v; }
    v.sign = (int)(p >> (n - 1));
    if (v.sign) p = (0 - p) & mask;
    int bits[64], nb = 0;
    for (int i = n - 2; i >= 0; i--) bits[nb++] = (int)((p >> i) & 1);   /* after the sign, MSB first */
    const int r = bits[0];
    int m = 0;
    while (m < nb && bits[m] == r) m++;
    const int k = r ? m - 1 : -m;
    int j = m + 1;                                   /* skip the terminating bit, if any */
    int e = 0;
    for (int q = 0; q < es; q++) { e = 2 * e + (j < nb ? bits[j] : 0); j++; }
    uint64_t f = 0;
    int fb = 0;
    for (; j < nb; j++) { f = 2 * f + (uint64_t)bits[j]; fb++; }
    v.M = (1ull << fb) + f;                          /* 1.f scaled by 2^fb */
    v.X = k * (1 << es) + e - fb;
    return v;
}

/* ---- the exact target and "value(c) ? target" ----------------------------- */
enum { T_SUM = 0, T_PROD = 1, T_QUOT = 2, T_ROOT = 3 };
typedef struct {
    int type;
    /* T_SUM: |sa*A + sb*B|, A = Ma 2^Xa, B = Mb 2^Xb (held as S 2^base) */
    big S; int base;
    /* T_PROD: Ma*Mb 2^(Xa+Xb); T_QUOT: (Ma 2^Xa) / (Mb 2^Xb); T_ROOT: sqrt(Ma 2^Xa) */
    uint64_t Ma, Mb; int Xa, Xb;
} target;

#define BASE (-300)              /* below every exponent that occurs: X >= -242 (products, squares); X <= 240 */

/* sign of value(c) - target, for c = M 2^X (M > 0) */
static int cmp_target(uint64_t M, int X, const target* t) {
    big c, r;
    switch (t->type) {
        case T_SUM:
            big_from(&c, M, X, t->base);
            return big_cmp(&c, &t->S);
        case T_PROD:
            big_from(&c, M, X, BASE);
            big_from(&r, (unsigned __int128)t->Ma * t->Mb, t->Xa + t->Xb, BASE);
            return big_cmp(&c, &r);
        case T_QUOT:                                 /* c ? a / b  <=>  c * b ? a */
            big_from(&c, (unsigned __int128)M * t->Mb, X + t->Xb, BASE);
            big_from(&r, t->Ma, t->Xa, BASE);
            return big_cmp(&c, &r);
        default:                                     /* c ? sqrt(a)  <=>  c^2 ? a */
            big_from(&c, (unsigned __int128)M * M, 2 * X, BASE);
            big_from(&r, t->Ma, t->Xa, BASE);
            return big_cmp(&c, &r);
    }
}

/* checker.round_to_posit for a nonzero exact target of sign `sign` */
static uint64_t round_target(const target* t, int sign, int n, int es) {
    const uint64_t mask = (1ull << n) - 1, mp = (1ull << (n - 1)) - 1;
    const val vmax = value(mp, n, es), vmin = value(1, n, es);
    uint64_t p;
    if (cmp_target(vmax.M, vmax.X, t) <= 0) {
        p = mp;                                      /* |x| >= maxpos */
    } else if (cmp_target(vmin.M, vmin.X, t) >= 0) {
        p = 1;                                       /* 0 < |x| <= minpos */
    } else {
        uint64_t lo = 1, hi = mp;                    /* value(lo) < |x| < value(hi) */
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) / 2;
            const val vm = value(mid, n, es);
            if (cmp_target(vm.M, vm.X, t) <= 0) lo = mid; else hi = mid;
        }
        p = lo;
        const val vp = value(p, n, es);
        if (cmp_target(vp.M, vp.X, t) != 0) {
            const val md = value(2 * p + 1, n + 1, es);  /* the midpoint, read as Posit(n+1, es) */
            const int c = cmp_target(md.M, md.X, t);     /* midpoint ? |x| */
            if (c < 0 || (c == 0 && (p & 1))) p = p + 1;
        }
    }
    return sign ? ((0 - p) & mask) : p;
}

/* ---- the operations (checker.py add / sub / mul / div / sqrt) ------------- */
static uint64_t cw_add_signed(uint64_t a, uint64_t b, int negb, int n, int es) {
    const uint64_t nar = 1ull << (n - 1);
    const val x = value(a, n, es), y = value(b, n, es);
    if (x.kind == CW_NAR || y.kind == CW_NAR) return nar;
    const int sy = y.sign ^ negb;
    if (x.kind == CW_ZERO && y.kind == CW_ZERO) return 0;
    target t;
    memset(&t, 0, sizeof t);
    t.type = T_SUM;
    t.base = BASE;
    big A, B;
    if (x.kind == CW_ZERO) big_set(&A, 0, 0); else big_from(&A, x.M, x.X, BASE);
    if (y.kind == CW_ZERO) big_set(&B, 0, 0); else big_from(&B, y.M, y.X, BASE);
    int sign;
    if (x.sign == sy || x.kind == CW_ZERO || y.kind == CW_ZERO) {
        big_add(&t.S, &A, &B);
        sign = (x.kind == CW_ZERO) ? sy : x.sign;
    } else {
        const int c = big_cmp(&A, &B);
        if (c == 0) return 0;                        /* exact cancellation */
        if (c > 0) { big_sub(&t.S, &A, &B); sign = x.sign; } else { big_sub(&t.S, &B, &A); sign = sy; }
    }
    return round_target(&t, sign, n, es);
}

static uint64_t cw_mul(uint64_t a, uint64_t b, int n, int es) {
    const val x = value(a, n, es), y = value(b, n, es);
    if (x.kind == CW_NAR || y.kind == CW_NAR) return 1ull << (n - 1);
    if (x.kind == CW_ZERO || y.kind == CW_ZERO) return 0;
    target t = {T_PROD};
    t.Ma = x.M; t.Mb = y.M; t.Xa = x.X; t.Xb = y.X;
    return round_target(&t, x.sign ^ y.sign, n, es);
}

static uint64_t cw_div(uint64_t a, uint64_t b, int n, int es) {
    const val x = value(a, n, es), y = value(b, n, es);
    if (x.kind == CW_NAR || y.kind == CW_NAR || y.kind == CW_ZERO) return 1ull << (n - 1);
    if (x.kind == CW_ZERO) return 0;
    target t = {T_QUOT};
    t.Ma = x.M; t.Mb = y.M; t.Xa = x.X; t.Xb = y.X;
    return round_target(&t, x.sign ^ y.sign, n, es);
}

static uint64_t cw_sqrt(uint64_t a, int n, int es) {
    const val x = value(a, n, es);
    if (x.kind == CW_NAR || (x.kind == CW_NUM && x.sign)) return 1ull << (n - 1);
    if (x.kind == CW_ZERO) return 0;
    target t = {T_ROOT};
    t.Ma = x.M; t.Xa = x.X;
    return round_target(&t, 0, n, es);
}

uint64_t cw_op1(int op, uint64_t a, uint64_t b, int n, int es) {
    switch (op) {
        case 0: return cw_add_signed(a, b, 0, n, es);
        case 1: return cw_add_signed(a, b, 1, n, es);
        case 2: return cw_mul(a, b, n, es);
        case 3: return cw_div(a, b, n, es);
        default: return cw_sqrt(a, n, es);
    }
}

/* expected results for count pairs (op codes as or_vec_op: 0 add, 1 sub,
 * 2 mul, 3 div, 4 sqrt): want[i]; returns the number of i with
 * want[i] != got[i] */
int64_t cw_check(int op, const uint32_t* a, const uint32_t* b, const uint32_t* got, uint32_t* want, int64_t count,
                 int n, int es) {
    int64_t nbad = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : nbad)
    for (int64_t i = 0; i < count; i++) {
        want[i] = (uint32_t)cw_op1(op, a[i], b ? b[i] : 0u, n, es);
        nbad += want[i] != got[i];
    }
    return nbad;
}

int cw_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
