// kernels_dig.cuh — the B200-first product path (MDPS_ALGO_DIGITS).
//
// Why.  On sm_100a every FP64 instruction (DADD, DMUL, DFMA) costs one slot
// of the same 64-lane/SM pipe, so the cost of a complex md multiply-add is
// its FP64 instruction count.  The paper's md arithmetic (PAPER.md:76-80,
// Table 1) spends most of it on TwoSum cascades that keep every rounding
// error.  Here each real md coefficient is split ONCE into S signed digits of
// BETA = 23 bits on a radix-2^23 grid anchored at the coefficient's own
// exponent (an error-free split in the sense of Dekker/Veltkamp: every digit
// is an exact double).  A digit product is then exact (<= 44 bits), and the
// sum of a few hundred of them is exact too, so one DFMA per digit pair does
// the work of a TwoProd plus its TwoSum cascade.  The truncated convolution
// z_k = sum_{i<=k} x_i y_{k-i} is accumulated EXACTLY
// into S integer-valued digit accumulators per output coefficient; the only
// rounding is the truncation below digit S-1, which S is chosen to put more
// than 8 bits below the md precision 2^(-53 L).
//
// Representation (pool slot s): digits [S][D][2] doubles (digit, coefficient,
// part) and one radix exponent per complex coefficient [D] int32.  Part value
//     v = sum_j  digit_j * R^(e - 1 - j),   R = 2^BETA,  |v| < R^e / 2,
// every digit balanced (|digit_j| <= R/2 + 1, the top one included); both
// parts of a coefficient share e (the larger part's); a zero coefficient has
// e = ZERO_E.  Limb planes (the ABI layout) are converted to digits on
// entry (x every call, coefficients at create) and back to limbs only for
// values and Jacobian entries (the addition jobs), so the whole DAG runs on
// digits.
//
// Alignment across terms.  A term x_i y_{k-i} has exponent e_x + e_y; the
// accumulator of z_k is anchored at e_acc = max over its terms (a pre-pass
// over the exponents, integer work only), and a term with
// delta = e_acc - e_x - e_y is added delta digits lower.  The shift is
// applied through the shared-memory ADDRESS of the per-lane operand's digit
// planes (digit l reads plane l - delta, or a zero when l < delta), so the
// FMAs always hit statically indexed registers.
//
// This file shares no code with the CPU oracle (oracle/).
#pragma once
#include "md.cuh"

namespace mdps {

constexpr int BETA = 23;
constexpr double RADIX = 8388608.0;          // 2^23
constexpr double INV_RADIX = 1.0 / 8388608.0;
constexpr double MAGIC = 6755399441055744.0;  // 1.5 * 2^52: rounds |x| < 2^51 to an integer
constexpr int ZERO_E = -(1 << 24);

// digits per part for L limbs: (S-2)*BETA >= 53 L + 8 covers the worst case
// of both operands having a 1-bit top digit with 8 bits to spare.
__host__ __device__ constexpr int digits_for(int L) {
    int S = 2;
    while ((S - 2) * BETA < 53 * L + 8) S++;
    return S;
}
// terms between carry normalisations.  Stored digits satisfy |d_j| <= R/2 + 1,
// so one term adds at most 2 (t+1) (R/2+1)^2 <= 1.01 S R^2 / 2 to an
// accumulator digit t <= S-1 (two real products per part); a carry pass
// leaves |A_t| <= R/2 + 2^31, and accumulators must stay below 2^53:
// NORM * 1.01 S 2^45 < 2^53 - 2^32.  The top accumulator digit is never
// carried out of: it collects at most 2 D (R/2+1)^2 < 2^53 for D <= 128.
__host__ __device__ constexpr int norm_every(int S) { return 25600 / (S * 101) - 1; }

// doubles per digit-pool slot (one series: [S][D][2]) and ints per exponent
// slot (one per complex coefficient: [D])
__host__ __device__ constexpr size_t dig_slot_stride(int S, int D) { return (size_t)2 * S * D; }
__host__ __device__ constexpr size_t dig_exp_stride(int D) { return (size_t)D; }

// 2^(BETA*q) as a double: exact in the normal range, else formed by two
// scalings (rounds into the subnormal range / saturates)
__device__ __forceinline__ double radix_pow(int q) {
    int ex = BETA * q;
    if (ex >= -1022 && ex <= 1023) return __longlong_as_double((long long)(1023 + ex) << 52);
    ex = max(min(ex, 2046), -2044);
    const int a = ex / 2, b = ex - a;
    return __dmul_rn(__longlong_as_double((long long)(1023 + a) << 52),
                     __longlong_as_double((long long)(1023 + b) << 52));
}

__device__ __forceinline__ double rint_magic(double x) { return __dsub_rn(__dadd_rn(x, MAGIC), MAGIC); }

// One parallel carry pass (exact): every digit t >= 1 hands rint(A_t / R) to
// digit t-1 at once — S independent 4-instruction chains instead of one
// serial chain.  q = (A_t + 1.5 2^52 R) - 1.5 2^52 R is A_t rounded to the
// nearest multiple of R (ties to even; exact for |A_t| < 2^51 R), so the
// carry costs two additions, one subtraction and one FMA per digit.  From
// |A_t| < 2^53 one pass leaves |A_t| <= R/2 + 2^31, a second <= R/2 + 2^9, a
// third <= R/2 + 1.
template <int N>
__device__ __forceinline__ void carry_pass(double (&A)[N]) {
    constexpr double MAGIC_R = MAGIC * RADIX;
    double q[N];
#pragma unroll
    for (int t = N - 1; t >= 1; t--) q[t] = __dsub_rn(__dadd_rn(A[t], MAGIC_R), MAGIC_R);
#pragma unroll
    for (int t = N - 1; t >= 1; t--) {
        A[t] = __dsub_rn(A[t], q[t]);
        A[t - 1] = __fma_rn(q[t], INV_RADIX, A[t - 1]);
    }
}

// balance digits 1..N-1 into [-R/2 - 1, R/2 + 1], carrying into digit 0 (exact)
template <int N>
__device__ __forceinline__ void carry_normalize(double (&A)[N]) {
    carry_pass(A);
    carry_pass(A);
    carry_pass(A);
}

__device__ __forceinline__ int ceil_div(int a, int b) { return a >= 0 ? (a + b - 1) / b : -((-a) / b); }

// 2^k as a double for k in [-1022, 1023]
__device__ __forceinline__ double pow2i(int k) { return __longlong_as_double((long long)(1023 + k) << 52); }

// radix exponent of one real md number (L limbs, any overlap): the smallest
// e with |v| < R^e / 2 (a balanced top digit); ZERO_E for zero, 0 for NaN
template <int L>
__device__ __forceinline__ int limbs_exponent(const double (&v0)[L]) {
    double m = 0.0;
#pragma unroll
    for (int p = 0; p < L; p++) m = __dadd_ru(m, fabs(v0[p]));
    if (!(m > 0.0)) return m == 0.0 ? ZERO_E : 0;
    const int emin = ilogb(m) + 1;  // |v| <= m < 2^emin
    return ceil_div(emin + 1, BETA);
}

// one real md number -> S balanced digits on the grid of exponent e (e at
// least its own limbs_exponent; a larger e puts leading zero digits in
// front and rounds at digit S-1 of the larger grid).  The limbs are first
// scaled EXACTLY by 2^(-BETA (e-1)) (two power-of-two factors, each in
// range), so the digit grid is fixed — R^0 .. R^-(S-1) — whatever the
// magnitude: no weight under- or overflows for tiny values.
template <int L, int S>
__device__ __forceinline__ void limbs_to_digits_at(const double (&v0)[L], int e, double (&d)[S]) {
    const int sh = -BETA * (e - 1), s1 = sh / 2, s2 = sh - s1;
    const double f1 = pow2i(s1), f2 = pow2i(s2);
    double v[L];
#pragma unroll
    for (int p = 0; p < L; p++) v[p] = __dmul_rn(__dmul_rn(v0[p], f1), f2);  // |v| < R / 2
#pragma unroll
    for (int j = 0; j < S; j++) {
        const double C = MAGIC * pow2i(-BETA * j);  // rounds to multiples of R^-j
        double acc = 0.0;
#pragma unroll
        for (int p = 0; p < L; p++) {
            const double q = __dsub_rn(__dadd_rn(v[p], C), C);
            v[p] = __dsub_rn(v[p], q);
            acc = __dadd_rn(acc, q);
        }
        d[j] = __dmul_rn(acc, pow2i(BETA * j));
    }
    carry_normalize(d);
}

// one real md number (L limbs, any overlap) -> S balanced digits + exponent
// (its own grid; the solver's digit vectors)
template <int L, int S>
__device__ __forceinline__ int limbs_to_digits(const double (&v0)[L], double (&d)[S]) {
    const int e = limbs_exponent<L>(v0);
    if (e == ZERO_E || e == 0) {
        double m = 0.0;
#pragma unroll
        for (int p = 0; p < L; p++) m = __dadd_ru(m, fabs(v0[p]));
        if (!(m > 0.0)) {  // zero (or NaN: also mapped to the zero encoding's exponent)
#pragma unroll
            for (int j = 0; j < S; j++) d[j] = (m == 0.0) ? 0.0 : m;
            return m == 0.0 ? ZERO_E : 0;
        }
    }
    limbs_to_digits_at<L, S>(v0, e, d);
    return e;
}

// one complex md number -> S digits per part on ONE grid, the exponent of
// the larger part (the product pool's format): every term of
// a truncated product then has one alignment shift for both of its real
// products, and a digit row of y is one 16-byte (re, im) pair.  The smaller
// part keeps its digits down to R^(e-S) — the precision of the complex number
// normwise (R20).  NaN parts propagate as NaN digits.
template <int L, int S>
__device__ __forceinline__ int cplx_to_digits(const double (&re)[L], const double (&im)[L], double (&dr)[S],
                                              double (&di)[S]) {
    const int e = max(limbs_exponent<L>(re), limbs_exponent<L>(im));
    if (e == ZERO_E) {
#pragma unroll
        for (int j = 0; j < S; j++) dr[j] = di[j] = 0.0;
        return ZERO_E;
    }
    limbs_to_digits_at<L, S>(re, e, dr);
    limbs_to_digits_at<L, S>(im, e, di);
    return e;
}

// S digits (exponent e, digit j weight R^(e-1-j), any balance with
// |digit| < 2^52 / R; NORMALIZED = the caller already balanced digits 1..S-1)
// -> L limbs, rounded (md_renorm of exact pairs)
template <int L, int S, bool NORMALIZED = false>
__device__ __forceinline__ void digits_to_limbs(double (&A)[S], int e, double (&out)[L]) {
    constexpr int NV = 1 + S / 2;
    double vals[NV];
    if (!NORMALIZED) carry_normalize(A);
    if (e <= ZERO_E / 2) {
#pragma unroll
        for (int p = 0; p < L; p++) out[p] = 0.0;
        return;
    }
    vals[0] = __dmul_rn(A[0], radix_pow(e - 1));
#pragma unroll
    for (int m = 0; m < NV - 1; m++) {
        const int t = 1 + 2 * m;
        const double hi = A[t];
        const double lo = (t + 1 < S) ? A[t + 1] : 0.0;
        vals[m + 1] = __dmul_rn(__fma_rn(hi, RADIX, lo), radix_pow(e - 2 - t));
    }
    md_renorm(vals, out);
}

// ---------------------------------------------------------------------------
// to_digits: limb series [2][L][D] (src) -> digit pool slots slot0.. in the
// pool format: digits [S][D][2] (digit, coefficient, part), one exponent per
// complex coefficient [D].  One thread per (series, coefficient); `count`
// series, src contiguous.
template <int L>
__global__ void __launch_bounds__(128) to_digits_kernel(const double *__restrict__ src, int count, int D,
                                                       double *__restrict__ dpool,
                                                       int *__restrict__ epool, int slot0) {
    constexpr int S = digits_for(L);
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (long long)count * D) return;
    const int s = (int)(g / D), k = (int)(g - (long long)s * D);
    const double *x = src + (size_t)s * 2 * L * D;
    double *dd = dpool + (size_t)(slot0 + s) * dig_slot_stride(S, D);
    double re[L], im[L], dr[S], di[S];
#pragma unroll
    for (int p = 0; p < L; p++) {
        re[p] = x[p * D + k];
        im[p] = x[(L + p) * D + k];
    }
    const int e = cplx_to_digits<L, S>(re, im, dr, di);
#pragma unroll
    for (int j = 0; j < S; j++) *reinterpret_cast<double2 *>(dd + ((size_t)j * D + k) * 2) = make_double2(dr[j], di[j]);
    epool[(size_t)(slot0 + s) * dig_exp_stride(D) + k] = e;
}

// limbs -> digits (the pool format, cplx_to_digits) -> limbs round trip
// (unit test of the staging format); one thread per (series, coefficient)
template <int L>
__global__ void digits_roundtrip_kernel(const double *__restrict__ x, double *__restrict__ y, int count,
                                        int D) {
    constexpr int S = digits_for(L);
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (long long)count * D) return;
    const int s = (int)(g / D), k = (int)(g - (long long)s * D);
    double re[L], im[L], dr[S], di[S], out[L];
#pragma unroll
    for (int p = 0; p < L; p++) {
        re[p] = x[((size_t)s * 2 * L + p) * D + k];
        im[p] = x[((size_t)s * 2 * L + L + p) * D + k];
    }
    const int e = cplx_to_digits<L, S>(re, im, dr, di);
    digits_to_limbs<L, S>(dr, e, out);
#pragma unroll
    for (int p = 0; p < L; p++) y[((size_t)s * 2 * L + p) * D + k] = out[p];
    digits_to_limbs<L, S>(di, e, out);
#pragma unroll
    for (int p = 0; p < L; p++) y[((size_t)s * 2 * L + L + p) * D + k] = out[p];
}

}  // namespace mdps
