// kernels_dig.cuh — the B200-first product path (MDPS_ALGO_DIGITS).
//
// Why.  On sm_100a every FP64 instruction (DADD, DMUL, DFMA) costs one slot
// of the same 64-lane/SM pipe, so the cost of a complex md multiply-add is
// its FP64 instruction count.  The paper's md arithmetic (PAPER.md:76-80,
// Table 1) spends most of it on TwoSum cascades that keep every rounding
// error.  Here each real md coefficient is split ONCE into S signed digits of
// BETA = 22 bits on a radix-2^22 grid anchored at the coefficient's own
// exponent (an error-free split in the sense of Dekker/Veltkamp: every digit
// is an exact double).  A digit product is then exact (<= 44 bits), and the
// sum of up to ~2^8 of them is exact too, so one DFMA per digit pair does
// the work of a TwoProd plus its TwoSum cascade.  The truncated convolution
// z_k = sum_{i<=k} x_i y_{k-i} is accumulated EXACTLY
// into S integer-valued digit accumulators per output coefficient; the only
// rounding is the truncation below digit S-1, which S is chosen to put more
// than 8 bits below the md precision 2^(-53 L).
//
// Representation (pool slot s): digits [2][S][D] doubles (part, digit,
// coefficient) and radix exponents [2][D] int32.  Part value
//     v = sum_j  digit_j * R^(e - 1 - j),   R = 2^BETA,  |v| < R^e,
// digits balanced (|digit_j| <= R/2 for j >= 1, |digit_0| <= R); a zero part
// has e = ZERO_E.  Limb planes (the ABI layout) are converted to digits on
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

constexpr int BETA = 22;
constexpr double RADIX = 4194304.0;          // 2^22
constexpr double INV_RADIX = 1.0 / 4194304.0;
constexpr double MAGIC = 6755399441055744.0;  // 1.5 * 2^52: rounds |x| < 2^51 to an integer
constexpr int ZERO_E = -(1 << 24);

// digits per part for L limbs: (S-2)*BETA >= 53 L + 8 covers the worst case
// of both operands having a 1-bit top digit with 8 bits to spare.
__host__ __device__ constexpr int digits_for(int L) {
    int S = 2;
    while ((S - 2) * BETA < 53 * L + 8) S++;
    return S;
}
// terms between carry normalisations: 2 S (2^BETA)^2 per term per digit,
// accumulators balanced to R/2 after normalisation, exact below 2^53.
__host__ __device__ constexpr int norm_every(int S) { return 256 / S - 1; }

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

// balance digits 1..N-1 into [-R/2, R/2], carrying into digit 0 (exact)
template <int N>
__device__ __forceinline__ void carry_normalize(double (&A)[N]) {
#pragma unroll
    for (int t = N - 1; t >= 1; t--) {
        const double q = rint_magic(__dmul_rn(A[t], INV_RADIX));
        A[t] = __fma_rn(-q, RADIX, A[t]);
        A[t - 1] = __dadd_rn(A[t - 1], q);
    }
}

__device__ __forceinline__ int ceil_div(int a, int b) { return a >= 0 ? (a + b - 1) / b : -((-a) / b); }

// one real md number (L limbs, any overlap) -> S balanced digits + exponent
template <int L, int S>
__device__ __forceinline__ int limbs_to_digits(const double (&v0)[L], double (&d)[S]) {
    double v[L];
    double m = 0.0;
#pragma unroll
    for (int p = 0; p < L; p++) {
        v[p] = v0[p];
        m = __dadd_ru(m, fabs(v0[p]));
    }
    if (!(m > 0.0)) {  // zero (or NaN: also mapped to the zero encoding's exponent)
#pragma unroll
        for (int j = 0; j < S; j++) d[j] = (m == 0.0) ? 0.0 : m;
        return m == 0.0 ? ZERO_E : 0;
    }
    const int emin = ilogb(m) + 1;  // |v| <= m < 2^emin
    const int e = ceil_div(emin, BETA);
#pragma unroll
    for (int j = 0; j < S; j++) {
        const double G = radix_pow(e - 1 - j);
        const double C = __dmul_rn(MAGIC, G);
        double acc = 0.0;
#pragma unroll
        for (int p = 0; p < L; p++) {
            const double q = __dsub_rn(__dadd_rn(v[p], C), C);
            v[p] = __dsub_rn(v[p], q);
            acc = __dadd_rn(acc, q);
        }
        d[j] = __dmul_rn(acc, radix_pow(1 + j - e));
    }
    carry_normalize(d);
    return e;
}

// S digits (exponent e, digit j weight R^(e-1-j), any balance with
// |digit| < 2^52 / R) -> L limbs, rounded (md_renorm of exact pairs)
template <int L, int S>
__device__ __forceinline__ void digits_to_limbs(double (&A)[S], int e, double (&out)[L]) {
    constexpr int NV = 1 + S / 2;
    double vals[NV];
    carry_normalize(A);
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
// to_digits: limb series [2][L][D] (src[slot_src]) -> digit pool slot.
// one thread per (series, coefficient); `count` series, src contiguous.
template <int L>
__global__ void __launch_bounds__(128) to_digits_kernel(const double *__restrict__ src, int count, int D,
                                                       double *__restrict__ dpool,
                                                       int *__restrict__ epool, int slot0) {
    constexpr int S = digits_for(L);
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (long long)count * D) return;
    const int s = (int)(g / D), k = (int)(g - (long long)s * D);
    const double *x = src + (size_t)s * 2 * L * D;
    double *dd = dpool + (size_t)(slot0 + s) * 2 * S * D;
    int *ee = epool + (size_t)(slot0 + s) * 2 * D;
#pragma unroll
    for (int part = 0; part < 2; part++) {
        double v[L], d[S];
#pragma unroll
        for (int p = 0; p < L; p++) v[p] = x[(part * L + p) * D + k];
        const int e = limbs_to_digits<L, S>(v, d);
#pragma unroll
        for (int j = 0; j < S; j++) dd[(part * S + j) * D + k] = d[j];
        ee[part * D + k] = e;
    }
}

// ---------------------------------------------------------------------------
// conv_dig: product jobs z = x * y mod t^D on digit planes.
// Threads: P jobs per block; per job T = ceil(D/2) output pairs x F splits.
// Thread (t, f) owns outputs k1 = t and k2 = D-1-t (the folded triangle has
// D+1 terms for every t) and the fold iterations j = f, f+F, ...; the F
// partial accumulators of an output are added exactly at the end.
// Shared memory per job: x and y digit planes [2][S][D+1] (+1 skews banks),
// exponents [2][2][D]; then per thread parking (k1) and final (k2) partials.
struct ConvDigGeom {
    int T, F, P, threads;
};

__host__ __device__ inline size_t conv_dig_smem(int S, int D, int P, int threads) {
    const size_t ser = (size_t)2 * S * (D + 1);
    return (size_t)P * (2 * ser) * sizeof(double) + (size_t)threads * 2 * S * sizeof(double) +
           (size_t)P * 4 * D * sizeof(int) + 16;
}

template <int L, int PART>
__device__ __forceinline__ void conv_dig_pass(const double *__restrict__ sx, const double *__restrict__ sy,
                                              const int *__restrict__ ex, const int *__restrict__ ey,
                                              const double *zero, int D, int t, int f, int F, int eacc1,
                                              int eacc2, double *park, double *fin) {
    constexpr int S = digits_for(L);
    constexpr int NORM = norm_every(S);
    const int PD = D + 1;
    double A[S];
    md_zero(A);
    int cnt = 0;
    bool switched = false;
    for (int j = f; j <= D; j += F) {
        const bool first = j <= t;
        if (!first && !switched) {  // k1 partial complete: park it, start k2
            switched = true;
            carry_normalize(A);
#pragma unroll
            for (int s = 0; s < S; s++) {
                park[s] = A[s];
                A[s] = 0.0;
            }
            cnt = 0;
        }
        const int i = first ? j : j - t - 1;
        const int k = first ? t : D - 1 - t;
        const int kk = k - i;
        const int eacc = first ? eacc1 : eacc2;
        // operand U = x_i (registers), W = y_{k-i} (shifted through addresses)
        double Ur[S], Ui[S];
#pragma unroll
        for (int s = 0; s < S; s++) {
            Ur[s] = sx[s * PD + i];
            Ui[s] = sx[(S + s) * PD + i];
        }
        // PART 0 (re): Ur*Wr - Ui*Wi ;  PART 1 (im): Ur*Wi + Ui*Wr
        const int w1part = PART == 0 ? 0 : 1, w2part = PART == 0 ? 1 : 0;
        const int d1 = eacc - ex[i] - ey[w1part * D + kk];
        const int d2 = eacc - ex[D + i] - ey[w2part * D + kk];
        const double *W1 = sy + w1part * S * PD + kk;
        const double *W2 = sy + w2part * S * PD + kk;
#pragma unroll
        for (int l = 0; l < S; l++) {
            const double w1 = *((l >= d1) ? W1 + (l - d1) * PD : zero);
            const double w2 = *((l >= d2) ? W2 + (l - d2) * PD : zero);
#pragma unroll
            for (int u = 0; u < S - l; u++) {
                A[u + l] = __fma_rn(Ur[u], w1, A[u + l]);
                A[u + l] = __fma_rn(PART == 0 ? -Ui[u] : Ui[u], w2, A[u + l]);
            }
        }
        if (++cnt == NORM) {
            carry_normalize(A);
            cnt = 0;
        }
    }
    carry_normalize(A);
    if (!switched) {  // no k2 iterations: everything belongs to k1
#pragma unroll
        for (int s = 0; s < S; s++) {
            park[s] = A[s];
            fin[s] = 0.0;
        }
    } else {
#pragma unroll
        for (int s = 0; s < S; s++) fin[s] = A[s];
    }
}

// sum the F partials (stride 2S*? handled by caller), normalise, write the
// output digits (leading-zero shift) and exponent of one (k, part)
template <int L>
__device__ __forceinline__ void conv_dig_emit(const double *parts, int pstride, int F, int eacc,
                                              double *zd, int *ze, int D, int k, int part) {
    constexpr int S = digits_for(L);
    double A[S];
#pragma unroll
    for (int s = 0; s < S; s++) A[s] = parts[s];
    for (int g = 1; g < F; g++) {
#pragma unroll
        for (int s = 0; s < S; s++) A[s] = __dadd_rn(A[s], parts[g * pstride + s]);
    }
    carry_normalize(A);
    // Z = [c2, c1, c0, A_1 .. A_{S-1}], Z_u has weight R^(eacc - u)
    double Z[S + 2];
    {
        double a0 = A[0];
        const double c2 = rint_magic(__dmul_rn(a0, INV_RADIX * INV_RADIX));
        a0 = __fma_rn(-c2, RADIX * RADIX, a0);
        const double c1 = rint_magic(__dmul_rn(a0, INV_RADIX));
        const double c0 = __fma_rn(-c1, RADIX, a0);
        Z[0] = c2;
        Z[1] = c1;
        Z[2] = c0;
#pragma unroll
        for (int s = 1; s < S; s++) Z[s + 2] = A[s];
    }
    int z0 = S + 2;
#pragma unroll
    for (int u = S + 1; u >= 0; u--)
        if (Z[u] != 0.0) z0 = u;
    // shift left by z0 (barrel: z0 < 64)
#pragma unroll
    for (int b = 0; b < 6; b++) {
        const int sh = 1 << b;
        if (z0 & sh) {
#pragma unroll
            for (int u = 0; u < S + 2; u++) Z[u] = (u + sh < S + 2) ? Z[u + sh] : 0.0;
        }
    }
    const int e = (z0 >= S + 2 || eacc <= ZERO_E / 2) ? ZERO_E : eacc + 1 - z0;
#pragma unroll
    for (int s = 0; s < S; s++) zd[(part * S + s) * D + k] = (e == ZERO_E) ? 0.0 : Z[s];
    ze[part * D + k] = e;
}

template <int L>
__global__ void __launch_bounds__(128) conv_dig_kernel(double *__restrict__ dpool, int *__restrict__ epool,
                                                      const int *__restrict__ jobs, int njobs, int D,
                                                      int T, int F, int P) {
    constexpr int S = digits_for(L);
    const int PD = D + 1;
    const int SER = 2 * S * PD;  // doubles per staged series
    const int threads_per_job = T * F;
    extern __shared__ double sm[];
    double *sdig = sm;                                              // [P][2][SER]
    double *spart = sm + (size_t)P * 2 * SER;                       // [threads][2][S]
    int *sexp = (int *)(spart + (size_t)blockDim.x * 2 * S);        // [P][2 series][2][D]
    double *zero = (double *)(sexp + (size_t)P * 4 * D);            // one zero (aligned: D ints * 4P)

    const int job0 = blockIdx.x * P;
    // stage digit planes and exponents of both inputs of every job
    for (int idx = threadIdx.x; idx < P * 2 * 2 * S * D; idx += blockDim.x) {
        const int per_job = 2 * 2 * S * D;
        const int jl = idx / per_job, r = idx - jl * per_job;
        const int which = r / (2 * S * D), r2 = r - which * 2 * S * D;  // r2 = plane * D + k
        const int plane = r2 / D, k = r2 - plane * D;
        const int job = min(job0 + jl, njobs - 1);
        const int src = jobs[3 * job + which];
        sdig[(size_t)jl * 2 * SER + which * SER + plane * PD + k] = dpool[(size_t)src * 2 * S * D + r2];
    }
    for (int idx = threadIdx.x; idx < P * 2 * 2 * D; idx += blockDim.x) {
        const int jl = idx / (4 * D), r = idx - jl * 4 * D;
        const int which = r / (2 * D), r2 = r - which * 2 * D;
        const int job = min(job0 + jl, njobs - 1);
        const int src = jobs[3 * job + which];
        sexp[idx] = epool[(size_t)src * 2 * D + r2];
    }
    if (threadIdx.x == 0) *zero = 0.0;
    __syncthreads();

    const int jl = threadIdx.x / threads_per_job;
    const int r = threadIdx.x - jl * threads_per_job;
    const int t = r / F, f = r - t * F;
    const bool valid = jl < P && t < T;
    const int jlc = valid ? jl : 0;
    const double *sx = sdig + (size_t)jlc * 2 * SER, *sy = sx + SER;
    const int *ex = sexp + jlc * 4 * D, *ey = ex + 2 * D;
    const int tt = valid ? t : 0;

    // exponent pre-pass: e_acc of (k1, k2) x (re, im) over ALL terms
    int ea1r = ZERO_E, ea1i = ZERO_E, ea2r = ZERO_E, ea2i = ZERO_E;
    for (int j = 0; j <= D; j++) {
        const bool first = j <= tt;
        const int i = first ? j : j - tt - 1;
        const int k = first ? tt : D - 1 - tt;
        const int kk = k - i;
        const int xr = ex[i], xi = ex[D + i], yr = ey[kk], yi = ey[D + kk];
        const int er = max(xr + yr, xi + yi), ei = max(xr + yi, xi + yr);
        if (first) {
            ea1r = max(ea1r, er);
            ea1i = max(ea1i, ei);
        } else {
            ea2r = max(ea2r, er);
            ea2i = max(ea2i, ei);
        }
    }

    double *park = spart + (size_t)threadIdx.x * 2 * S;
    double *fin = park + S;
    const int job = job0 + jl;
    double *zd = nullptr;
    int *ze = nullptr;
    if (valid && job < njobs) {
        const int out = jobs[3 * job + 2];
        zd = dpool + (size_t)out * 2 * S * D;
        ze = epool + (size_t)out * 2 * D;
    }
#pragma unroll 1
    for (int part = 0; part < 2; part++) {
        if (valid) {
            if (part == 0)
                conv_dig_pass<L, 0>(sx, sy, ex, ey, zero, D, tt, f, F, ea1r, ea2r, park, fin);
            else
                conv_dig_pass<L, 1>(sx, sy, ex, ey, zero, D, tt, f, F, ea1i, ea2i, park, fin);
        }
        __syncthreads();
        if (valid && job < njobs) {
            // thread f == 0 emits k1, f == F-1 (or the same thread) emits k2
            const double *base = spart + (size_t)(threadIdx.x - f) * 2 * S;
            if (f == 0) conv_dig_emit<L>(base, 2 * S, F, part ? ea1i : ea1r, zd, ze, D, tt, part);
            if (f == F - 1 && D - 1 - tt != tt)
                conv_dig_emit<L>(base + S, 2 * S, F, part ? ea2i : ea2r, zd, ze, D, D - 1 - tt, part);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// accum_dig: addition jobs on digit planes -> limb outputs.
// one thread per (task, k); two parts.
template <int L>
__global__ void __launch_bounds__(128) accum_dig_kernel(const double *__restrict__ dpool,
                                                       const int *__restrict__ epool,
                                                       const int *__restrict__ task_ptr,
                                                       const int *__restrict__ ent_slot,
                                                       const int *__restrict__ ent_w, int ntasks, int n,
                                                       int D, double *__restrict__ values,
                                                       double *__restrict__ jac) {
    constexpr int S = digits_for(L);
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (long long)ntasks * D) return;
    const int task = (int)(g / D), k = (int)(g - (long long)task * D);
    const int e0 = task_ptr[task], e1 = task_ptr[task + 1];
    double *o = task < n ? values + (size_t)task * 2 * L * D : jac + (size_t)(task - n) * 2 * L * D;
#pragma unroll 1
    for (int part = 0; part < 2; part++) {
        int eacc = ZERO_E;
        for (int e = e0; e < e1; e++) eacc = max(eacc, epool[(size_t)ent_slot[e] * 2 * D + part * D + k]);
        // weights up to 2^20: the sum of up to 2^11 entries stays exact; one
        // headroom digit keeps the top accumulator digit small
        double A[S + 1];
        md_zero(A);
        int cnt = 0;
        for (int e = e0; e < e1; e++) {
            const int slot = ent_slot[e];
            const double w = (double)ent_w[e];
            const int delta = eacc - epool[(size_t)slot * 2 * D + part * D + k] + 1;
            const double *d = dpool + (size_t)slot * 2 * S * D + (size_t)part * S * D + k;
#pragma unroll
            for (int s = 0; s <= S; s++) {
                const int src = s - delta;
                const double v = (src >= 0 && src < S) ? d[(size_t)src * D] : 0.0;
                A[s] = __fma_rn(w, v, A[s]);
            }
            if (++cnt == 1024) {
                carry_normalize(A);
                cnt = 0;
            }
        }
        double out[L];
        digits_to_limbs<L, S + 1>(A, eacc + 1, out);
#pragma unroll
        for (int p = 0; p < L; p++) o[(part * L + p) * D + k] = out[p];
    }
}

// limbs -> digits -> limbs round trip (unit test of the staging format)
template <int L>
__global__ void digits_roundtrip_kernel(const double *__restrict__ x, double *__restrict__ y, int count,
                                        int D) {
    constexpr int S = digits_for(L);
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (long long)count * 2 * D) return;
    const int s = (int)(g / (2 * D)), r = (int)(g - (long long)s * 2 * D);
    const int part = r / D, k = r - part * D;
    double v[L], d[S], out[L];
#pragma unroll
    for (int p = 0; p < L; p++) v[p] = x[((size_t)s * 2 * L + part * L + p) * D + k];
    const int e = limbs_to_digits<L, S>(v, d);
    digits_to_limbs<L, S>(d, e, out);
#pragma unroll
    for (int p = 0; p < L; p++) y[((size_t)s * 2 * L + part * L + p) * D + k] = out[p];
}

}  // namespace mdps
