/*
 * mdoracle.c — the CPU ORACLE for mdps_eval_diff.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load or call this
 * library.  It shares no code, header, table or helper with the CUDA path
 * (paper_2012_06607_b200/), and the CUDA path never calls it.
 *
 * What it computes (PAPER.md, arXiv 2012.06607):
 *   - multiple-double numbers: an unevaluated sum of L hardware doubles
 *     (§2), L <= MDO_MAXL;
 *   - every operation is computed EXACTLY in integer arithmetic (a
 *     "superaccumulator": a fixed-point integer in base 2^32 digits wide
 *     enough for any product of two doubles) and then rounded GREEDILY to L
 *     limbs: limb_0 = RN(X), limb_1 = RN(X - limb_0), ..., RN = IEEE
 *     round-to-nearest-even.  This is the plain definition of "X in L-fold
 *     double precision"; no error-free transformation of the GPU path is used;
 *   - the truncated power-series product z_k = sum_{i<=k} x_i y_{k-i},
 *     k = 0..d (§3), each coefficient formed exactly then
 *     rounded to L limbs; complex product re = ac - bd, im = ad + bc
 *     (reading R5);
 *   - the polynomial system with series coefficients f_i(x) and its Jacobian
 *     (§4) by the PLAIN definition: each
 *     monomial, and each exponent-weighted monomial quotient a_l x^(a-e_l),
 *     multiplied out left to right in ascending variable order (repeated
 *     factors for exponents), every series product rounded to L limbs; the
 *     sum over monomials exact, rounded once (readings R1-R4);
 *   - md division (long division, L+2 quotient digits) and square root (L+2
 *     correction steps) — used only by pins (series inverse, PAPER.md:172-175;
 *     the 2-norm example).
 *   - multitasking over output entries with the paper's job queue: a counter
 *     guarded by a binary semaphore (§5, Fig. 1).
 *
 * Pins: tests/test_oracle_*.py (exact rationals, closed forms, invariants,
 * the paper's worked examples).  See DESIGN.md "Oracle".
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define MDO_MAXL 16

typedef __int128 i128;
typedef unsigned __int128 u128;

/* ---------------------------------------------------------------------------
 * Superaccumulator: value = sum_j c[j] * 2^(32*(j - SA_BIAS)).
 * Range 2^-2688 .. 2^2688 covers any product of two finite doubles.
 * Cells are int64 holding (signed) sums of 32-bit chunks; normalisation
 * propagates carries so that all but the top cell lie in [0, 2^32).
 * ------------------------------------------------------------------------- */
#define SA_N 168
#define SA_BIAS 84

typedef struct {
    int64_t c[SA_N];
    int lo, hi; /* touched range; lo > hi means zero */
} sa_t;

static __thread int g_err; /* sticky range error flag (per thread) */

static void sa_init(sa_t *s) {
    memset(s->c, 0, sizeof s->c);
    s->lo = SA_N;
    s->hi = -1;
}

static void sa_reset(sa_t *s) {
    if (s->hi >= s->lo) memset(&s->c[s->lo], 0, sizeof(int64_t) * (size_t)(s->hi - s->lo + 1));
    s->lo = SA_N;
    s->hi = -1;
}

/* add (neg ? -1 : 1) * mag * 2^e exactly */
static void sa_dep(sa_t *s, int neg, u128 mag, int e) {
    if (!mag) return;
    int p = e + 32 * SA_BIAS;
    if (p < 0) { g_err = 1; return; }
    int j = p >> 5, sh = p & 31, t = 0;
    if (j + 6 >= SA_N) { g_err = 1; return; }
    while (mag) {
        uint64_t chunk = ((uint64_t)(mag & 0xffffffffu)) << sh; /* < 2^63 */
        int64_t lo = (int64_t)(chunk & 0xffffffffu), hi = (int64_t)(chunk >> 32);
        if (neg) { lo = -lo; hi = -hi; }
        s->c[j + t] += lo;
        s->c[j + t + 1] += hi;
        mag >>= 32;
        t++;
    }
    if (j < s->lo) s->lo = j;
    if (j + t > s->hi) s->hi = j + t;
}

/* a double as sign, 53-bit integer mantissa and exponent: |v| = m * 2^e */
static void dec(double v, int *neg, uint64_t *m, int *e) {
    int ex;
    double f = frexp(fabs(v), &ex);
    *m = (uint64_t)ldexp(f, 53);
    *e = ex - 53;
    *neg = v < 0;
}

static void sa_add_double(sa_t *s, double v) {
    if (v == 0.0) return;
    int neg, e;
    uint64_t m;
    dec(v, &neg, &m, &e);
    sa_dep(s, neg, m, e);
}

/* w * a * b exactly (w a small integer, |w| < 2^20) */
static void sa_add_prod(sa_t *s, double a, double b, int64_t w) {
    if (a == 0.0 || b == 0.0 || w == 0) return;
    int na, nb, ea, eb;
    uint64_t ma, mb;
    dec(a, &na, &ma, &ea);
    dec(b, &nb, &mb, &eb);
    int neg = na ^ nb ^ (w < 0);
    u128 mag = (u128)ma * mb * (u128)(w < 0 ? -w : w);
    sa_dep(s, neg, mag, ea + eb);
}

/* carry propagation; returns sign of the value (-1, 0, +1) */
static int sa_norm(sa_t *s) {
    if (s->hi < s->lo) return 0;
    for (int j = s->lo; j < s->hi; j++) {
        int64_t v = s->c[j];
        int64_t carry = v >> 32; /* floor(v / 2^32) (arithmetic shift) */
        s->c[j] = v - carry * 4294967296LL;
        s->c[j + 1] += carry;
    }
    while (s->c[s->hi] >= 4294967296LL || s->c[s->hi] < -4294967296LL) {
        if (s->hi + 1 >= SA_N) { g_err = 1; break; }
        int64_t v = s->c[s->hi];
        int64_t carry = v >> 32;
        s->c[s->hi] = v - carry * 4294967296LL;
        s->c[s->hi + 1] += carry;
        s->hi++;
    }
    while (s->hi >= s->lo && s->c[s->hi] == 0) s->hi--;
    while (s->lo <= s->hi && s->c[s->lo] == 0) s->lo++;
    if (s->hi < s->lo) { s->lo = SA_N; s->hi = -1; return 0; }
    return s->c[s->hi] < 0 ? -1 : 1;
}

/* magnitude digits of a normalised accumulator into d[] (uint32), range lo..hi */
static int sa_mag(const sa_t *s, int sign, uint32_t *d, int *lo, int *hi) {
    *lo = s->lo;
    *hi = s->hi;
    if (sign >= 0) {
        for (int j = s->lo; j <= s->hi; j++) d[j] = (uint32_t)s->c[j];
        return 0;
    }
    int64_t borrow = 0; /* digits of -X */
    for (int j = s->lo; j <= s->hi; j++) {
        int64_t v = -s->c[j] - borrow;
        borrow = 0;
        while (v < 0) { v += 4294967296LL; borrow++; }
        d[j] = (uint32_t)v;
    }
    while (*hi >= *lo && d[*hi] == 0) (*hi)--;
    return 1;
}

static inline uint64_t dcell(const uint32_t *d, int lo, int hi, int j) {
    return (j < lo || j > hi) ? 0 : (uint64_t)d[j];
}

/* RN(X) for the accumulated value X (ties to even); normalises s */
static double sa_rn(sa_t *s) {
    int sign = sa_norm(s);
    if (!sign) return 0.0;
    uint32_t d[SA_N];
    int lo, hi;
    int neg = sa_mag(s, sign, d, &lo, &hi);
    if (hi < lo) return 0.0;
    int top = 31 - __builtin_clz(d[hi]);
    int P = 32 * (hi - SA_BIAS) + top; /* MSB weight 2^P */
    int q = P - 52;
    if (q < -1074) q = -1074;
    if (P > 1023) { g_err = 1; return neg ? -INFINITY : INFINITY; }
    /* M = bits [q, P] */
    int pos = q + 32 * SA_BIAS;
    int j = pos >> 5, sh = pos & 31;
    uint64_t w = dcell(d, lo, hi, j) >> sh;
    w |= dcell(d, lo, hi, j + 1) << (32 - sh);
    if (sh) w |= dcell(d, lo, hi, j + 2) << (64 - sh);
    int nb = P - q + 1;
    uint64_t M = nb >= 64 ? w : (w & ((1ULL << nb) - 1));
    /* round bit (q-1) and sticky (below q-1) */
    int rpos = pos - 1;
    int rj = rpos >> 5, rsh = rpos & 31;
    int rbit = (int)((dcell(d, lo, hi, rj) >> rsh) & 1);
    int sticky = 0;
    if (rsh && (dcell(d, lo, hi, rj) & ((1ULL << rsh) - 1))) sticky = 1;
    for (int t = lo; !sticky && t < rj; t++)
        if (d[t]) sticky = 1;
    if (rbit && (sticky || (M & 1))) M++;
    double r = ldexp((double)M, q);
    return neg ? -r : r;
}

/* greedy rounding of the accumulated value to L limbs; consumes s */
static void sa_round_limbs(sa_t *s, int L, double *out, int stride) {
    for (int l = 0; l < L; l++) {
        double limb = sa_rn(s);
        out[l * stride] = limb;
        if (limb == 0.0) {
            for (int t = l + 1; t < L; t++) out[t * stride] = 0.0;
            break;
        }
        sa_add_double(s, -limb);
    }
    sa_reset(s);
}

/* ---------------------------------------------------------------------------
 * Multiple-double numbers (real): arrays of L doubles, limb 0 first.
 * ------------------------------------------------------------------------- */

/* greedy L-limb rounding of the exact sum of v[0..n) */
int mdo_round(const double *v, int n, int L, double *out) {
    sa_t s;
    sa_init(&s);
    g_err = 0;
    for (int i = 0; i < n; i++) sa_add_double(&s, v[i]);
    sa_round_limbs(&s, L, out, 1);
    return g_err ? -1 : 0;
}

int mdo_add(const double *a, const double *b, int L, double *out) {
    sa_t s;
    sa_init(&s);
    g_err = 0;
    for (int i = 0; i < L; i++) { sa_add_double(&s, a[i]); sa_add_double(&s, b[i]); }
    sa_round_limbs(&s, L, out, 1);
    return g_err ? -1 : 0;
}

int mdo_mul(const double *a, const double *b, int L, double *out) {
    sa_t s;
    sa_init(&s);
    g_err = 0;
    for (int p = 0; p < L; p++)
        for (int q = 0; q < L; q++) sa_add_prod(&s, a[p], b[q], 1);
    sa_round_limbs(&s, L, out, 1);
    return g_err ? -1 : 0;
}

/* long division: L+2 quotient digits q_j = RN(remainder) / b_0, each followed
 * by the exact update remainder -= q_j * b; the quotient is the exact sum of
 * the q_j rounded to L limbs.  a has La limbs, b has Lb limbs. */
static int md_div_gen(const double *a, int La, const double *b, int Lb, int L, double *out) {
    if (b[0] == 0.0) return -2;
    sa_t r, qs;
    sa_init(&r);
    sa_init(&qs);
    for (int i = 0; i < La; i++) sa_add_double(&r, a[i]);
    for (int j = 0; j < L + 2; j++) {
        double r0 = sa_rn(&r);
        if (r0 == 0.0) break;
        double qj = r0 / b[0];
        sa_add_double(&qs, qj);
        for (int p = 0; p < Lb; p++) sa_add_prod(&r, qj, b[p], -1);
    }
    sa_round_limbs(&qs, L, out, 1);
    return 0;
}

int mdo_div(const double *a, const double *b, int L, double *out) {
    g_err = 0;
    int rc = md_div_gen(a, L, b, L, L, out);
    return rc ? rc : (g_err ? -1 : 0);
}

/* square root: s_0 = sqrt(a_0); then L+1 corrections c = RN(a - S^2) / (2 s_0),
 * each residual formed exactly; result = RN_L(sum of the corrections) */
static int md_sqrt_gen(const double *a, int La, int L, double *out) {
    if (a[0] < 0.0) return -2;
    if (a[0] == 0.0) { for (int l = 0; l < L; l++) out[l] = 0.0; return 0; }
    double S[MDO_MAXL + 4];
    int ns = 0;
    S[ns++] = sqrt(a[0]);
    sa_t r;
    sa_init(&r);
    for (int j = 0; j < L + 1; j++) {
        sa_reset(&r);
        for (int i = 0; i < La; i++) sa_add_double(&r, a[i]);
        for (int p = 0; p < ns; p++)
            for (int q = 0; q < ns; q++) sa_add_prod(&r, S[p], S[q], -1);
        double r0 = sa_rn(&r);
        if (r0 == 0.0) break;
        S[ns++] = r0 / (2.0 * S[0]);
    }
    sa_t t;
    sa_init(&t);
    for (int p = 0; p < ns; p++) sa_add_double(&t, S[p]);
    sa_round_limbs(&t, L, out, 1);
    return 0;
}

int mdo_sqrt(const double *a, int L, double *out) {
    g_err = 0;
    int rc = md_sqrt_gen(a, L, L, out);
    return rc ? rc : (g_err ? -1 : 0);
}

/* 2-norm of a complex md vector v[count][2][L]: the sum of
 * squares is formed exactly, rounded to L+2 limbs, then square-rooted. */
int mdo_norm2(const double *v, int count, int L, double *out) {
    g_err = 0;
    sa_t s;
    sa_init(&s);
    for (int i = 0; i < count; i++)
        for (int part = 0; part < 2; part++) {
            const double *x = v + ((size_t)i * 2 + part) * L;
            for (int p = 0; p < L; p++)
                for (int q = 0; q < L; q++) sa_add_prod(&s, x[p], x[q], 1);
        }
    double sq[MDO_MAXL + 2];
    sa_round_limbs(&s, L + 2, sq, 1);
    int rc = md_sqrt_gen(sq, L + 2, L, out);
    return rc ? rc : (g_err ? -1 : 0);
}

/* ---------------------------------------------------------------------------
 * Truncated power series, layout [2][L][D] (part, limb, coefficient).
 * ------------------------------------------------------------------------- */
#define SIDX(part, limb, k, L, D) (((size_t)(part) * (L) + (limb)) * (D) + (k))

/* a series with every limb pre-split into signed 53-bit mantissa and exponent */
typedef struct { int64_t *m; int *e; } dser_t;

static void dser_fill(dser_t *d, const double *x, size_t count) {
    for (size_t t = 0; t < count; t++) {
        int neg, e;
        uint64_t m;
        if (x[t] == 0.0) { d->m[t] = 0; d->e[t] = 0; continue; }
        dec(x[t], &neg, &m, &e);
        d->m[t] = neg ? -(int64_t)m : (int64_t)m;
        d->e[t] = e;
    }
}

static inline void sa_dep_mm(sa_t *s, int64_t ma, int ea, int64_t mb, int eb, int negate) {
    if (!ma || !mb) return;
    i128 p = (i128)ma * (i128)mb;
    int neg = (p < 0) ^ negate;
    u128 mag = (u128)(p < 0 ? -p : p);
    sa_dep(s, neg, mag, ea + eb);
}

/* z = x * y mod t^D.  counts (optional): [0] += complex
 * md multiplications x_i*y_{k-i}, [1] += complex md additions — (d+2)(d+1)/2
 * and (d+1)d/2 per product.  z may alias neither input.
 * dx, dy: scratch of 2*L*D entries each. */
static void series_mul(const double *x, const double *y, int D, int L, double *z,
                       long long *counts, sa_t *sr, sa_t *si, dser_t *dx, dser_t *dy) {
    size_t SS = (size_t)2 * L * D;
    dser_fill(dx, x, SS);
    dser_fill(dy, y, SS);
    for (int k = 0; k < D; k++) {
        for (int i = 0; i <= k; i++) {
            int j = k - i;
            for (int p = 0; p < L; p++) {
                size_t xr = SIDX(0, p, i, L, D), xi = SIDX(1, p, i, L, D);
                for (int q = 0; q < L; q++) {
                    size_t yr = SIDX(0, q, j, L, D), yi = SIDX(1, q, j, L, D);
                    sa_dep_mm(sr, dx->m[xr], dx->e[xr], dy->m[yr], dy->e[yr], 0); /* re += a c */
                    sa_dep_mm(sr, dx->m[xi], dx->e[xi], dy->m[yi], dy->e[yi], 1); /* re -= b d */
                    sa_dep_mm(si, dx->m[xr], dx->e[xr], dy->m[yi], dy->e[yi], 0); /* im += a d */
                    sa_dep_mm(si, dx->m[xi], dx->e[xi], dy->m[yr], dy->e[yr], 0); /* im += b c */
                }
            }
            if (counts) {
                counts[0] += 1;
                if (i > 0) counts[1] += 1;
            }
        }
        sa_round_limbs(sr, L, &z[SIDX(0, 0, k, L, D)], D);
        sa_round_limbs(si, L, &z[SIDX(1, 0, k, L, D)], D);
    }
}

static int dser_alloc(dser_t *d, size_t count) {
    d->m = (int64_t *)malloc(count * sizeof(int64_t));
    d->e = (int *)malloc(count * sizeof(int));
    return (d->m && d->e) ? 0 : -1;
}
static void dser_free(dser_t *d) { free(d->m); free(d->e); }

int mdo_series_mul(const double *x, const double *y, int D, int L, double *z, long long *counts) {
    g_err = 0;
    sa_t *s = (sa_t *)malloc(2 * sizeof(sa_t));
    dser_t dx, dy;
    size_t SS = (size_t)2 * L * D;
    dser_alloc(&dx, SS);
    dser_alloc(&dy, SS);
    sa_init(&s[0]);
    sa_init(&s[1]);
    series_mul(x, y, D, L, z, counts, &s[0], &s[1], &dx, &dy);
    dser_free(&dx);
    dser_free(&dy);
    free(s);
    return g_err ? -1 : 0;
}

/* z = x + y */
int mdo_series_add(const double *x, const double *y, int D, int L, double *z) {
    g_err = 0;
    sa_t s;
    sa_init(&s);
    for (int part = 0; part < 2; part++)
        for (int k = 0; k < D; k++) {
            for (int p = 0; p < L; p++) {
                sa_add_double(&s, x[SIDX(part, p, k, L, D)]);
                sa_add_double(&s, y[SIDX(part, p, k, L, D)]);
            }
            sa_round_limbs(&s, L, &z[SIDX(part, 0, k, L, D)], D);
        }
    return g_err ? -1 : 0;
}

/* complex md division (ar + i ai) / (br + i bi), operands contiguous with
 * La and Lb limbs: (a * conj(b)) / |b|^2, numerator parts and |b|^2 formed
 * exactly and rounded to L+3 limbs, then two real long divisions to L limbs. */
#define BUF (MDO_MAXL + 16)
static int cdiv(const double *ar, const double *ai, int La, const double *br, const double *bi, int Lb,
                int L, double *qr, double *qi) {
    sa_t s;
    sa_init(&s);
    int L3 = L + 3;
    double nr[BUF], ni[BUF], den[BUF];
    for (int p = 0; p < Lb; p++)
        for (int q = 0; q < Lb; q++) {
            sa_add_prod(&s, br[p], br[q], 1);
            sa_add_prod(&s, bi[p], bi[q], 1);
        }
    sa_round_limbs(&s, L3, den, 1);
    for (int p = 0; p < La; p++)
        for (int q = 0; q < Lb; q++) {
            sa_add_prod(&s, ar[p], br[q], 1);
            sa_add_prod(&s, ai[p], bi[q], 1);
        }
    sa_round_limbs(&s, L3, nr, 1);
    for (int p = 0; p < La; p++)
        for (int q = 0; q < Lb; q++) {
            sa_add_prod(&s, ai[p], br[q], 1);
            sa_add_prod(&s, ar[p], bi[q], -1);
        }
    sa_round_limbs(&s, L3, ni, 1);
    int rc = md_div_gen(nr, L3, den, L3, L, qr);
    if (rc) return rc;
    return md_div_gen(ni, L3, den, L3, L, qi);
}

/* y = 1/x mod t^D (exists when x_0 != 0):
 * y_0 = 1/x_0, y_k = -(sum_{i=1..k} x_i y_{k-i}) / x_0, the sum formed
 * exactly and rounded to L+3 limbs before the division. */
int mdo_series_inv(const double *x, int D, int L, double *y) {
    g_err = 0;
    if (L > MDO_MAXL) return -3;
    double x0r[BUF], x0i[BUF], one[BUF] = {1.0}, zero[BUF] = {0.0}, qr[BUF], qi[BUF];
    for (int p = 0; p < L; p++) { x0r[p] = x[SIDX(0, p, 0, L, D)]; x0i[p] = x[SIDX(1, p, 0, L, D)]; }
    if (x0r[0] == 0.0 && x0i[0] == 0.0) return -2;
    int rc = cdiv(one, zero, 1, x0r, x0i, L, L, qr, qi);
    if (rc) return rc;
    for (int p = 0; p < L; p++) { y[SIDX(0, p, 0, L, D)] = qr[p]; y[SIDX(1, p, 0, L, D)] = qi[p]; }
    sa_t sr, si;
    sa_init(&sr);
    sa_init(&si);
    for (int k = 1; k < D; k++) {
        for (int i = 1; i <= k; i++)
            for (int p = 0; p < L; p++)
                for (int q = 0; q < L; q++) {
                    double xr = x[SIDX(0, p, i, L, D)], xi = x[SIDX(1, p, i, L, D)];
                    double yr = y[SIDX(0, q, k - i, L, D)], yi = y[SIDX(1, q, k - i, L, D)];
                    sa_add_prod(&sr, xr, yr, -1);
                    sa_add_prod(&sr, xi, yi, 1);
                    sa_add_prod(&si, xr, yi, -1);
                    sa_add_prod(&si, xi, yr, -1);
                }
        double nr[BUF], ni[BUF];
        sa_round_limbs(&sr, L + 3, nr, 1);
        sa_round_limbs(&si, L + 3, ni, 1);
        rc = cdiv(nr, ni, L + 3, x0r, x0i, L, L, qr, qi);
        if (rc) return rc;
        for (int p = 0; p < L; p++) { y[SIDX(0, p, k, L, D)] = qr[p]; y[SIDX(1, p, k, L, D)] = qi[p]; }
    }
    return g_err ? -1 : 0;
}

/* ---------------------------------------------------------------------------
 * Evaluation and differentiation of a polynomial system with series
 * coefficients, by the plain definition.
 *
 * System: poly i has monomials r in [poly_ptr[i], poly_ptr[i+1]); monomial r
 * has variables vars[mono_ptr[r] .. mono_ptr[r+1]) with exponents exps[..]
 * (any order; multiplied in ascending variable order), coefficient series
 * coeffs[r] ([2][L][D]).  x: [n][2][L][D].
 *
 * Entry (i, j): j = -1 -> value f_i(x); j >= 0 -> J_ij = df_i/dx_j;
 * j = -2 -> the degree-weighted value g_i(x) of Euler's identity for
 * polynomials, sum_j x_j df_i/dx_j = sum_r deg(r) c_r x^{a_r} (every monomial
 * is homogeneous of its own degree deg(r) = sum_l a_l), used to check whole
 * Jacobian rows (mdo_euler_residual below).
 *   f_i  = RN_L( sum_r  c_r * prod_l x_{v_l}^{a_l} )
 *   g_i  = RN_L( sum_r  deg(r) * (c_r * prod_l x_{v_l}^{a_l}) )
 *   J_ij = RN_L( sum_{r : j in r}  a_j * c_r * x^{a_r - e_j} )
 * with every series product in the chains rounded to L limbs.
 * ------------------------------------------------------------------------- */
typedef struct {
    int n_polys, n, D, L;
    const int *poly_ptr, *mono_ptr, *vars, *exps;
    const double *coeffs, *x;
    int n_entries;
    const int *rows, *cols;
    double *out; /* [n_entries][2][L][D] */
    double *out_f; /* optional, for (i, -2) entries: f_i from the same chains */
    /* job queue: counter guarded by a binary semaphore */
    pthread_mutex_t lock;
    int next;
    int err;
    long long products;
} job_t;

/* ascending order of the variables of monomial r (insertion sort of indices) */
static int mono_order(const job_t *J, int r, int *idx) {
    int a = J->mono_ptr[r], b = J->mono_ptr[r + 1], m = b - a;
    for (int t = 0; t < m; t++) idx[t] = a + t;
    for (int t = 1; t < m; t++) {
        int v = idx[t], u = t - 1;
        while (u >= 0 && J->vars[idx[u]] > J->vars[v]) { idx[u + 1] = idx[u]; u--; }
        idx[u + 1] = v;
    }
    return m;
}

static void run_entry(job_t *J, int e, double *t0, double *t1, sa_t *acc, sa_t *sr, sa_t *si,
                      dser_t *dx, dser_t *dy, sa_t *acc_f) {
    int i = J->rows[e], jcol = J->cols[e], D = J->D, L = J->L;
    size_t SS = (size_t)2 * L * D;
    long long prods = 0;
    int idx[4096];
    for (int r = J->poly_ptr[i]; r < J->poly_ptr[i + 1]; r++) {
        int m = mono_order(J, r, idx);
        int weight = 1;
        if (jcol >= 0) {
            int found = 0;
            for (int t = 0; t < m; t++)
                if (J->vars[idx[t]] == jcol) { found = 1; weight = J->exps[idx[t]]; }
            if (!found) continue;
        } else if (jcol == -2) {
            weight = 0;
            for (int t = 0; t < m; t++) weight += J->exps[idx[t]];
            if (weight == 0 && !J->out_f) continue; /* a constant term has degree 0 (but is part of f) */
        }
        /* chain: t = c_r; then multiply by each factor left to right */
        memcpy(t0, J->coeffs + (size_t)r * SS, SS * sizeof(double));
        for (int t = 0; t < m; t++) {
            int v = J->vars[idx[t]];
            int a = J->exps[idx[t]] - ((jcol >= 0 && v == jcol) ? 1 : 0);
            for (int rep = 0; rep < a; rep++) {
                series_mul(t0, J->x + (size_t)v * SS, D, L, t1, NULL, sr, si, dx, dy);
                double *sw = t0; t0 = t1; t1 = sw;
                prods++;
            }
        }
        /* exact accumulation of weight * t into the entry accumulators */
        for (int part = 0; part < 2; part++)
            for (int k = 0; k < D; k++)
                for (int p = 0; p < L; p++) {
                    double v = t0[SIDX(part, p, k, L, D)];
                    if (v != 0.0) {
                        int neg, ex;
                        uint64_t mm;
                        dec(v, &neg, &mm, &ex);
                        if (weight) sa_dep(&acc[part * D + k], neg, (u128)mm * (u128)weight, ex);
                        if (jcol == -2 && J->out_f) sa_dep(&acc_f[part * D + k], neg, (u128)mm, ex);
                    }
                }
    }
    double *o = J->out + (size_t)e * SS;
    for (int part = 0; part < 2; part++)
        for (int k = 0; k < D; k++) sa_round_limbs(&acc[part * D + k], L, &o[SIDX(part, 0, k, L, D)], D);
    if (jcol == -2 && J->out_f) {
        double *of = J->out_f + (size_t)e * SS;
        for (int part = 0; part < 2; part++)
            for (int k = 0; k < D; k++) sa_round_limbs(&acc_f[part * D + k], L, &of[SIDX(part, 0, k, L, D)], D);
    }
    pthread_mutex_lock(&J->lock);
    J->products += prods;
    pthread_mutex_unlock(&J->lock);
}

static void *worker(void *arg) {
    job_t *J = (job_t *)arg;
    size_t SS = (size_t)2 * J->L * J->D;
    double *t0 = (double *)malloc(SS * sizeof(double));
    double *t1 = (double *)malloc(SS * sizeof(double));
    sa_t *acc = (sa_t *)malloc(sizeof(sa_t) * (size_t)(4 * J->D + 2));
    for (int t = 0; t < 4 * J->D + 2; t++) sa_init(&acc[t]);
    dser_t dx, dy;
    dser_alloc(&dx, SS);
    dser_alloc(&dy, SS);
    g_err = 0;
    for (;;) {
        pthread_mutex_lock(&J->lock); /* request entry to the semaphore */
        int e = J->next++;            /* take the next job */
        pthread_mutex_unlock(&J->lock);
        if (e >= J->n_entries) break;
        run_entry(J, e, t0, t1, acc, &acc[2 * J->D], &acc[2 * J->D + 1], &dx, &dy, &acc[2 * J->D + 2]);
    }
    if (g_err) {
        pthread_mutex_lock(&J->lock);
        J->err = 1;
        pthread_mutex_unlock(&J->lock);
    }
    dser_free(&dx);
    dser_free(&dy);
    free(t0);
    free(t1);
    free(acc);
    return NULL;
}

static int eval_entries_impl(int n_polys, int n, const int *poly_ptr, const int *mono_ptr, const int *vars,
                             const int *exps, const double *coeffs, const double *x, int degree, int L,
                             int n_entries, const int *rows, const int *cols, double *out, double *out_f,
                             int nthreads, long long *products) {
    if (L < 1 || L > MDO_MAXL || degree < 0 || n < 1) return -3;
    for (int e = 0; e < n_entries; e++)
        if (rows[e] < 0 || rows[e] >= n_polys || cols[e] >= n || cols[e] < -2) return -3;
    for (int r = 0; r < poly_ptr[n_polys]; r++)
        if (mono_ptr[r + 1] - mono_ptr[r] > 4096) return -3;
    job_t J;
    memset(&J, 0, sizeof J);
    J.n_polys = n_polys; J.n = n; J.D = degree + 1; J.L = L;
    J.poly_ptr = poly_ptr; J.mono_ptr = mono_ptr; J.vars = vars; J.exps = exps;
    J.coeffs = coeffs; J.x = x; J.n_entries = n_entries; J.rows = rows; J.cols = cols; J.out = out;
    J.out_f = out_f;
    pthread_mutex_init(&J.lock, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > n_entries) nthreads = n_entries > 0 ? n_entries : 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, worker, &J);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&J.lock);
    if (products) *products = J.products;
    return J.err ? -1 : 0;
}

/* returns 0, or <0 on error; *products (optional) = series products computed */
int mdo_eval_entries(int n_polys, int n, const int *poly_ptr, const int *mono_ptr, const int *vars,
                     const int *exps, const double *coeffs, const double *x, int degree, int L,
                     int n_entries, const int *rows, const int *cols, double *out, int nthreads,
                     long long *products) {
    return eval_entries_impl(n_polys, n, poly_ptr, mono_ptr, vars, exps, coeffs, x, degree, L, n_entries, rows,
                             cols, out, NULL, nthreads, products);
}

/* both f_i and g_i of the given rows from ONE set of monomial chains (the
 * Euler check of non-homogeneous systems): out_g[e] = entry (rows[e], -2),
 * out_f[e] = entry (rows[e], -1), bit for bit. */
int mdo_eval_values_weighted(int n_polys, int n, const int *poly_ptr, const int *mono_ptr, const int *vars,
                             const int *exps, const double *coeffs, const double *x, int degree, int L,
                             int count, const int *rows, double *out_g, double *out_f, int nthreads,
                             long long *products) {
    int *cols = (int *)malloc(sizeof(int) * (size_t)(count > 0 ? count : 1));
    if (!cols) return -2;
    for (int e = 0; e < count; e++) cols[e] = -2;
    int rc = eval_entries_impl(n_polys, n, poly_ptr, mono_ptr, vars, exps, coeffs, x, degree, L, count, rows, cols,
                               out_g, out_f, nthreads, products);
    free(cols);
    return rc;
}

/* ---------------------------------------------------------------------------
 * Test metric: per output series s,
 *   e_s = max_k |a_{s,k} - b_{s,k}| / max(max_k |b_{s,k}|, 1)
 * with the complex difference of each coefficient formed EXACTLY and then
 * rounded to one double per part.  a, b: [count][2][L][D].  err: [count].
 * ------------------------------------------------------------------------- */
int mdo_series_err(const double *a, const double *b, int count, int D, int L, double *err) {
    g_err = 0;
    sa_t s;
    sa_init(&s);
    size_t SS = (size_t)2 * L * D;
    for (int c = 0; c < count; c++) {
        const double *A = a + (size_t)c * SS, *B = b + (size_t)c * SS;
        double maxd = 0.0, maxb = 0.0;
        for (int k = 0; k < D; k++) {
            double dd[2], bb[2];
            for (int part = 0; part < 2; part++) {
                for (int p = 0; p < L; p++) {
                    sa_add_double(&s, A[SIDX(part, p, k, L, D)]);
                    sa_add_double(&s, -B[SIDX(part, p, k, L, D)]);
                }
                dd[part] = sa_rn(&s);
                sa_reset(&s);
                for (int p = 0; p < L; p++) sa_add_double(&s, B[SIDX(part, p, k, L, D)]);
                bb[part] = sa_rn(&s);
                sa_reset(&s);
            }
            double md = hypot(dd[0], dd[1]), mb = hypot(bb[0], bb[1]);
            if (md > maxd) maxd = md;
            if (mb > maxb) maxb = mb;
        }
        err[c] = maxd / (maxb > 1.0 ? maxb : 1.0);
    }
    return g_err ? -1 : 0;
}

/* ---------------------------------------------------------------------------
 * Euler residual of a Jacobian row (test metric for full-size outputs;
 * SURVEY §8(c) C3 "eval/diff identities", R19).  For every
 * polynomial f, Euler's identity for the homogeneous parts gives
 *     sum_j x_j * df/dx_j = sum_r deg(r) c_r x^{a_r} =: g,
 * truncated at t^D like every product.  For row c:
 *     r_{c,k} = sum_j sum_{q<=k} x_{j,q} J_{c,j,k-q}  -  g_{c,k}
 * formed EXACTLY (every limb product in the superaccumulator), then rounded
 * to one double per part; res[c][k] = |r_{c,k}| (complex modulus).
 * x: [n][2][L][D]; J: [count][n][2][L][D]; g: [count][2][L][D];
 * res: [count][D].  Rows are jobs claimed from a counter (nthreads workers).
 * ------------------------------------------------------------------------- */
typedef struct {
    int count, n, D, L;
    const double *x, *J, *g;
    double *res;
    pthread_mutex_t lock;
    int next, err;
} euler_t;

static void *euler_worker(void *arg) {
    euler_t *E = (euler_t *)arg;
    int n = E->n, D = E->D, L = E->L;
    size_t SS = (size_t)2 * L * D;
    sa_t *acc = (sa_t *)malloc(sizeof(sa_t) * (size_t)(2 * D));
    dser_t dx, dj;
    int ok = acc && dser_alloc(&dx, SS * (size_t)n) == 0 && dser_alloc(&dj, SS * (size_t)n) == 0;
    g_err = 0;
    if (ok) dser_fill(&dx, E->x, SS * (size_t)n);
    for (;;) {
        pthread_mutex_lock(&E->lock);
        int c = E->next++;
        pthread_mutex_unlock(&E->lock);
        if (c >= E->count || !ok) break;
        for (int t = 0; t < 2 * D; t++) sa_init(&acc[t]);
        const double *Jc = E->J + (size_t)c * n * SS, *gc = E->g + (size_t)c * SS;
        dser_fill(&dj, Jc, SS * (size_t)n);
        for (int j = 0; j < n; j++) {
            size_t xo = (size_t)j * SS, jo = (size_t)j * SS;
            for (int k = 0; k < D; k++)
                for (int q = 0; q <= k; q++)
                    for (int p = 0; p < L; p++) {
                        size_t xr = xo + SIDX(0, p, q, L, D), xi = xo + SIDX(1, p, q, L, D);
                        for (int u = 0; u < L; u++) {
                            size_t yr = jo + SIDX(0, u, k - q, L, D), yi = jo + SIDX(1, u, k - q, L, D);
                            sa_dep_mm(&acc[k], dx.m[xr], dx.e[xr], dj.m[yr], dj.e[yr], 0);     /* re += a c */
                            sa_dep_mm(&acc[k], dx.m[xi], dx.e[xi], dj.m[yi], dj.e[yi], 1);     /* re -= b d */
                            sa_dep_mm(&acc[D + k], dx.m[xr], dx.e[xr], dj.m[yi], dj.e[yi], 0); /* im += a d */
                            sa_dep_mm(&acc[D + k], dx.m[xi], dx.e[xi], dj.m[yr], dj.e[yr], 0); /* im += b c */
                        }
                    }
        }
        for (int k = 0; k < D; k++) {
            double part[2];
            for (int pt = 0; pt < 2; pt++) {
                for (int p = 0; p < L; p++) sa_add_double(&acc[pt * D + k], -gc[SIDX(pt, p, k, L, D)]);
                part[pt] = sa_rn(&acc[pt * D + k]);
            }
            E->res[(size_t)c * D + k] = hypot(part[0], part[1]);
        }
    }
    if (g_err || !ok) {
        pthread_mutex_lock(&E->lock);
        E->err = 1;
        pthread_mutex_unlock(&E->lock);
    }
    if (ok) { dser_free(&dx); dser_free(&dj); }
    free(acc);
    return NULL;
}

int mdo_euler_residual(int count, int n, int D, int L, const double *x, const double *J, const double *g,
                       double *res, int nthreads) {
    if (count < 0 || n < 1 || D < 1 || L < 1 || L > MDO_MAXL) return -3;
    if (count == 0) return 0;
    euler_t E;
    memset(&E, 0, sizeof E);
    E.count = count; E.n = n; E.D = D; E.L = L; E.x = x; E.J = J; E.g = g; E.res = res;
    pthread_mutex_init(&E.lock, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > count) nthreads = count;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, euler_worker, &E);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&E.lock);
    return E.err ? -1 : 0;
}

/* ---------------------------------------------------------------------------
 * Block lower-triangular Toeplitz forward substitution (§4):
 *   (A_0 + A_1 t + ... + A_d t^d)(dx_0 + dx_1 t + ... + dx_d t^d) = b(t),
 * A_k = the coefficient-k matrix of the series matrix J (J[p][q] a series).
 * As the paper states it: factor A_0 once (LU with partial
 * pivoting for N = n), then for j = 0..d
 *     A_0 dx_j = b_j - sum_{i=1..j} A_i dx_{j-i}.
 * Readings (R9-R12):
 *   - pivot k = the row i >= k maximising |re_0(a_ik)| + |im_0(a_ik)| (leading
 *     limbs, one double rounding), lowest index on ties; rows swapped whole;
 *     a zero pivot column is "singular" (return -4);
 *   - multipliers l_ik = a_ik / a_kk correctly rounded (cdiv); every Schur
 *     update a_ij - l_ik u_kj formed exactly and rounded once;
 *   - r_j = b_j - sum_{i,q} A_i[p][q] dx_{j-i}[q]: every entry formed exactly,
 *     rounded once; forward substitution y_i = RN(r_i - sum_{q<i} l_iq y_q);
 *     back substitution dx_i = RN_{L+3}(y_i - sum_{q>i} u_iq dx_q) / u_ii.
 * J: [n][n][2][L][D] (row p, column q), b and dx: [n][2][L][D], piv: [n].
 * The right-hand sides of one j are independent jobs over p (PAPER.md:410-413:
 * "one job is the update of one right hand side vector"), run by nthreads
 * workers claiming rows from a counter guarded by a binary semaphore.
 * ------------------------------------------------------------------------- */
#define EIDX(p, q, part, limb, k, n, L, D) (((((size_t)(p) * (n) + (q)) * 2 + (part)) * (L) + (limb)) * (D) + (k))

typedef struct {
    int n, D, L, j;
    const double *J, *b;
    double *dx, *r; /* r: [n][2][L] right-hand side of step j */
    pthread_mutex_t lock;
    int next, err;
} ts_job_t;

static void *ts_rhs_worker(void *arg) {
    ts_job_t *T = (ts_job_t *)arg;
    int n = T->n, D = T->D, L = T->L, j = T->j;
    sa_t *s = (sa_t *)malloc(2 * sizeof(sa_t));
    sa_init(&s[0]);
    sa_init(&s[1]);
    g_err = 0;
    for (;;) {
        pthread_mutex_lock(&T->lock);
        int p = T->next++;
        pthread_mutex_unlock(&T->lock);
        if (p >= n) break;
        for (int part = 0; part < 2; part++)
            for (int l = 0; l < L; l++) sa_add_double(&s[part], T->b[SIDX(part, l, j, L, D) + (size_t)p * 2 * L * D]);
        for (int i = 1; i <= j; i++)
            for (int q = 0; q < n; q++)
                for (int u = 0; u < L; u++)
                    for (int v = 0; v < L; v++) {
                        double ar = T->J[EIDX(p, q, 0, u, i, n, L, D)], ai = T->J[EIDX(p, q, 1, u, i, n, L, D)];
                        const double *x = T->dx + (size_t)q * 2 * L * D;
                        double xr = x[SIDX(0, v, j - i, L, D)], xi = x[SIDX(1, v, j - i, L, D)];
                        sa_add_prod(&s[0], ar, xr, -1); /* re -= ar xr - ai xi */
                        sa_add_prod(&s[0], ai, xi, 1);
                        sa_add_prod(&s[1], ar, xi, -1); /* im -= ar xi + ai xr */
                        sa_add_prod(&s[1], ai, xr, -1);
                    }
        for (int part = 0; part < 2; part++) sa_round_limbs(&s[part], L, T->r + ((size_t)p * 2 + part) * L, 1);
    }
    if (g_err) {
        pthread_mutex_lock(&T->lock);
        T->err = 1;
        pthread_mutex_unlock(&T->lock);
    }
    free(s);
    return NULL;
}

/* pivot magnitude: |re_0| + |im_0| rounded once (the same double on every
 * implementation that adds the two absolute leading limbs) */
static double piv_mag(const double *re, const double *im) { return fabs(re[0]) + fabs(im[0]); }

int mdo_toeplitz_solve(int n, int D, int L, const double *J, const double *b, double *dx, int *piv,
                       int nthreads) {
    if (n < 1 || D < 1 || L < 1 || L > MDO_MAXL) return -3;
    g_err = 0;
    const size_t E = (size_t)2 * L; /* doubles per complex md element */
    double *lu = (double *)malloc(sizeof(double) * (size_t)n * n * E);
    double *r = (double *)malloc(sizeof(double) * (size_t)n * E);
    double *y = (double *)malloc(sizeof(double) * (size_t)n * E);
    sa_t *s = (sa_t *)malloc(2 * sizeof(sa_t));
    if (!lu || !r || !y || !s) return -5;
    sa_init(&s[0]);
    sa_init(&s[1]);
#define LU(i, q, part) (lu + (((size_t)(i) * n + (q)) * 2 + (part)) * L)
    for (int p = 0; p < n; p++)
        for (int q = 0; q < n; q++)
            for (int part = 0; part < 2; part++)
                for (int l = 0; l < L; l++) LU(p, q, part)[l] = J[EIDX(p, q, part, l, 0, n, L, D)];
    int rc = 0;
    /* LU with partial pivoting of A_0 (right-looking Gaussian elimination) */
    for (int k = 0; k < n && !rc; k++) {
        int best = k;
        double bm = piv_mag(LU(k, k, 0), LU(k, k, 1));
        for (int i = k + 1; i < n; i++) {
            double m = piv_mag(LU(i, k, 0), LU(i, k, 1));
            if (m > bm) { bm = m; best = i; }
        }
        piv[k] = best;
        if (bm == 0.0) { rc = -4; break; }
        if (best != k)
            for (int q = 0; q < n; q++)
                for (size_t t = 0; t < E; t++) {
                    double tmp = LU(k, q, 0)[t];
                    LU(k, q, 0)[t] = LU(best, q, 0)[t];
                    LU(best, q, 0)[t] = tmp;
                }
        for (int i = k + 1; i < n; i++) {
            double lr[BUF], li[BUF];
            rc = cdiv(LU(i, k, 0), LU(i, k, 1), L, LU(k, k, 0), LU(k, k, 1), L, L, lr, li);
            if (rc) break;
            memcpy(LU(i, k, 0), lr, sizeof(double) * L);
            memcpy(LU(i, k, 1), li, sizeof(double) * L);
            for (int q = k + 1; q < n; q++) {
                const double *ur = LU(k, q, 0), *ui = LU(k, q, 1);
                for (int l = 0; l < L; l++) {
                    sa_add_double(&s[0], LU(i, q, 0)[l]);
                    sa_add_double(&s[1], LU(i, q, 1)[l]);
                }
                for (int u = 0; u < L; u++)
                    for (int v = 0; v < L; v++) {
                        sa_add_prod(&s[0], lr[u], ur[v], -1);
                        sa_add_prod(&s[0], li[u], ui[v], 1);
                        sa_add_prod(&s[1], lr[u], ui[v], -1);
                        sa_add_prod(&s[1], li[u], ur[v], -1);
                    }
                sa_round_limbs(&s[0], L, LU(i, q, 0), 1);
                sa_round_limbs(&s[1], L, LU(i, q, 1), 1);
            }
        }
    }
    /* forward substitution over the coefficients j = 0..d */
    ts_job_t T;
    memset(&T, 0, sizeof T);
    T.n = n; T.D = D; T.L = L; T.J = J; T.b = b; T.dx = dx; T.r = r;
    pthread_mutex_init(&T.lock, NULL);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > n) nthreads = n;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int j = 0; j < D && !rc; j++) {
        T.j = j;
        T.next = 0;
        if (nthreads == 1) ts_rhs_worker(&T);
        else {
            for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, ts_rhs_worker, &T);
            for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
        }
        if (T.err) { rc = -1; break; }
#define RV(v, i, part) ((v) + ((size_t)(i) * 2 + (part)) * L)
        for (int k = 0; k < n; k++)
            if (piv[k] != k)
                for (size_t t = 0; t < E; t++) {
                    double tmp = RV(r, k, 0)[t];
                    RV(r, k, 0)[t] = RV(r, piv[k], 0)[t];
                    RV(r, piv[k], 0)[t] = tmp;
                }
        for (int i = 0; i < n; i++) { /* L y = P r, unit lower triangular */
            for (int l = 0; l < L; l++) {
                sa_add_double(&s[0], RV(r, i, 0)[l]);
                sa_add_double(&s[1], RV(r, i, 1)[l]);
            }
            for (int q = 0; q < i; q++) {
                const double *lr = LU(i, q, 0), *li = LU(i, q, 1), *yr = RV(y, q, 0), *yi = RV(y, q, 1);
                for (int u = 0; u < L; u++)
                    for (int v = 0; v < L; v++) {
                        sa_add_prod(&s[0], lr[u], yr[v], -1);
                        sa_add_prod(&s[0], li[u], yi[v], 1);
                        sa_add_prod(&s[1], lr[u], yi[v], -1);
                        sa_add_prod(&s[1], li[u], yr[v], -1);
                    }
            }
            sa_round_limbs(&s[0], L, RV(y, i, 0), 1);
            sa_round_limbs(&s[1], L, RV(y, i, 1), 1);
        }
        for (int i = n - 1; i >= 0; i--) { /* U dx_j = y */
            for (int l = 0; l < L; l++) {
                sa_add_double(&s[0], RV(y, i, 0)[l]);
                sa_add_double(&s[1], RV(y, i, 1)[l]);
            }
            for (int q = i + 1; q < n; q++) {
                const double *ur = LU(i, q, 0), *ui = LU(i, q, 1);
                const double *x = dx + (size_t)q * 2 * L * D;
                for (int u = 0; u < L; u++)
                    for (int v = 0; v < L; v++) {
                        double xr = x[SIDX(0, v, j, L, D)], xi = x[SIDX(1, v, j, L, D)];
                        sa_add_prod(&s[0], ur[u], xr, -1);
                        sa_add_prod(&s[0], ui[u], xi, 1);
                        sa_add_prod(&s[1], ur[u], xi, -1);
                        sa_add_prod(&s[1], ui[u], xr, -1);
                    }
            }
            double nr[BUF], ni[BUF], qr[BUF], qi[BUF];
            sa_round_limbs(&s[0], L + 3, nr, 1);
            sa_round_limbs(&s[1], L + 3, ni, 1);
            rc = cdiv(nr, ni, L + 3, LU(i, i, 0), LU(i, i, 1), L, L, qr, qi);
            if (rc) break;
            double *x = dx + (size_t)i * 2 * L * D;
            for (int l = 0; l < L; l++) { x[SIDX(0, l, j, L, D)] = qr[l]; x[SIDX(1, l, j, L, D)] = qi[l]; }
        }
    }
#undef RV
#undef LU
    pthread_mutex_destroy(&T.lock);
    free(th);
    free(lu); free(r); free(y); free(s);
    if (rc) return rc;
    return g_err ? -1 : 0;
}

/* ---------------------------------------------------------------------------
 * Least squares for N > n equations ("For N > n, the linear
 * systems are solved in the least squares sense").  With full column rank,
 * the least-squares solution of A_0 dx_j = r_j is the plain definition
 * dx_j = (A_0^H A_0)^-1 A_0^H r_j, and r_j = b_j - sum_{i>=1} A_i dx_{j-i}
 * turns the whole forward substitution into the square one for
 *     At_i = A_0^H A_i (n x n),  bt_j = A_0^H b_j,
 * At_0 = A_0^H A_0 (reading R18).  This routine forms every entry of
 * At and bt EXACTLY and rounds it to Lo limbs (Lo = L + 3 keeps the squared
 * condition number of the normal equations out of the result); the caller
 * solves the square system at Lo limbs and rounds to L.
 * J: [N][n][2][L][D], b: [N][2][L][D]; Jt: [n][n][2][Lo][D], bt: [n][2][Lo][D].
 * ------------------------------------------------------------------------- */
int mdo_toeplitz_normal(int N, int n, int D, int L, const double *J, const double *b, int Lo, double *Jt,
                        double *bt) {
    if (N < 1 || n < 1 || D < 1 || L < 1 || Lo < 1 || Lo > MDO_MAXL) return -3;
    g_err = 0;
    sa_t *s = (sa_t *)malloc(2 * sizeof(sa_t));
    if (!s) return -5;
    sa_init(&s[0]);
    sa_init(&s[1]);
    /* conj(a) * c: re = ar cr + ai ci, im = ar ci - ai cr */
    for (int p = 0; p < n; p++)
        for (int col = 0; col <= n; col++)  /* col == n: the right-hand side */
            for (int k = 0; k < D; k++) {
                for (int r = 0; r < N; r++)
                    for (int u = 0; u < L; u++)
                        for (int v = 0; v < L; v++) {
                            double ar = J[EIDX(r, p, 0, u, 0, n, L, D)], ai = J[EIDX(r, p, 1, u, 0, n, L, D)];
                            double cr, ci;
                            if (col < n) {
                                cr = J[EIDX(r, col, 0, v, k, n, L, D)];
                                ci = J[EIDX(r, col, 1, v, k, n, L, D)];
                            } else {
                                cr = b[SIDX(0, v, k, L, D) + (size_t)r * 2 * L * D];
                                ci = b[SIDX(1, v, k, L, D) + (size_t)r * 2 * L * D];
                            }
                            sa_add_prod(&s[0], ar, cr, 1);
                            sa_add_prod(&s[0], ai, ci, 1);
                            sa_add_prod(&s[1], ar, ci, 1);
                            sa_add_prod(&s[1], ai, cr, -1);
                        }
                double *out = col < n ? Jt + EIDX(p, col, 0, 0, k, n, Lo, D) : bt + SIDX(0, 0, k, Lo, D) + (size_t)p * 2 * Lo * D;
                sa_round_limbs(&s[0], Lo, out, D);
                sa_round_limbs(&s[1], Lo, out + (size_t)Lo * D, D);
            }
    free(s);
    return g_err ? -1 : 0;
}
