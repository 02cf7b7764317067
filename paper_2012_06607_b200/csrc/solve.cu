// solve.cu — block lower-triangular Toeplitz forward substitution on the GPU
// (include/libmdps.h "Block lower-triangular Toeplitz solver"; PAPER.md:266-333,
// §4).
//
//   (A_0 + A_1 t + ... + A_d t^d)(dx_0 + dx_1 t + ...) = b_0 + b_1 t + ...
//   A_0 dx_j = b_j - sum_{i=1..j} A_i dx_{j-i}
//
// Three launches per solve:
//  1. ts_pack_kernel: the Jacobian coefficients A_1..A_d -> digit elements
//     Ad[k-1][p][q] (kernels_dig.cuh representation: [2][S] digits + two
//     radix exponents; a group of lanes reading row p reads consecutive q),
//     the right-hand side -> the digit series R (r_k starts as b_k).
//  2. ts_gj_kernel (persistent, cooperative): W = A_0^-1 by Gauss-Jordan with
//     partial pivoting on [A_0 | I] in EFT md arithmetic (md.cuh): the pivots
//     are those of the paper's LU, A_0 is factored once,
//     and the d+1 solves become matrix-vector products; W -> digit elements.
//  3. ts_loop_kernel (persistent, cooperative): for j = 0..d
//       dx_j = W r_j                              (G lanes per row p)
//       r_k -= A_{k-j} dx_j  for all k > j        (G lanes per (k, p))
//     — the right-looking form of the paper's update ("one job is the update
//     of one right hand side vector after the computation of one update
//     vector"), so that every phase exposes (d-j) n
//     independent dot products.  Each dot product (and the subtraction from
//     r_k) is accumulated EXACTLY on digit planes as in the product kernel —
//     one DFMA per digit pair — and rounded once (to S digits for r_k and
//     dx_j, to L limbs for the output).
// Reductions across lanes are fixed trees (bitwise deterministic).  Grid-wide
// phases are separated by a software grid barrier (cooperative launch keeps
// all blocks co-resident).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <string>

#include "../../include/libmdps.h"
#include "conv_dig.cuh"
#include "md.cuh"

void mdps_internal_set_error(const std::string &s);  // libmdps.cu

namespace mdps {
namespace ts {

constexpr int THREADS = 256;

struct Barrier {
    unsigned int count;
    unsigned int gen;
};

// sense-free generation barrier over all blocks of a co-resident grid
__device__ __forceinline__ void grid_sync(Barrier *b) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int *vgen = &b->gen;
        const unsigned int g = *vgen;
        __threadfence();
        if (atomicAdd(&b->count, 1u) == gridDim.x - 1) {
            atomicExch(&b->count, 0u);
            __threadfence();
            atomicAdd(&b->gen, 1u);
        } else {
            while (*vgen == g) __nanosleep(40);
        }
        __threadfence();
    }
    __syncthreads();
}

// ---- complex md helpers (element = re limbs then im limbs, 2L doubles) --------
template <int L>
__device__ __forceinline__ void ld(const double *p, double (&re)[L], double (&im)[L]) {
#pragma unroll
    for (int l = 0; l < L; l++) {
        re[l] = p[l];
        im[l] = p[L + l];
    }
}

template <int L>
__device__ __forceinline__ void st(double *p, const double (&re)[L], const double (&im)[L]) {
#pragma unroll
    for (int l = 0; l < L; l++) {
        p[l] = re[l];
        p[L + l] = im[l];
    }
}

// (Br, Bi) += (NEG ? -1 : 1) * a * x   (re = ar xr - ai xi, im = ar xi + ai xr)
template <int L, bool NEG>
__device__ __forceinline__ void cfma(double (&Br)[L + 1], double (&Bi)[L + 1], const double (&ar)[L],
                                     const double (&ai)[L], const double (&xr)[L], const double (&xi)[L]) {
    double pr[L], pi[L], ni[L];
#pragma unroll
    for (int l = 0; l < L; l++) {
        pr[l] = NEG ? -ar[l] : ar[l];
        pi[l] = NEG ? -ai[l] : ai[l];
        ni[l] = -pi[l];
    }
    bins_fma<L>(Br, pr, xr);
    bins_fma<L>(Br, ni, xi);
    bins_fma<L>(Bi, pr, xi);
    bins_fma<L>(Bi, pi, xr);
}

template <int L>
__device__ __forceinline__ void cbins_add(double (&Br)[L + 1], double (&Bi)[L + 1], const double (&ar)[L],
                                          const double (&ai)[L]) {
    bins_add<L>(Br, ar);
    bins_add<L>(Bi, ai);
}

// B += C (bins of another accumulator: level o deposited at level o)
template <int L>
__device__ __forceinline__ void bins_merge(double (&B)[L + 1], const double (&C)[L + 1]) {
#pragma unroll
    for (int o = 0; o < L; o++) {
        double v = C[o];
#pragma unroll
        for (int t = o; t < L; t++) two_sum(B[t], v, B[t], v);
        B[L] = __dadd_rn(B[L], v);
    }
    B[L] = __dadd_rn(B[L], C[L]);
}

// tree reduction over aligned groups of G lanes (G a power of two <= 32);
// lane 0 of each group ends with the group's sum
template <int L>
__device__ __forceinline__ void group_reduce(double (&Br)[L + 1], double (&Bi)[L + 1], int G) {
    for (int off = G >> 1; off > 0; off >>= 1) {
        double Cr[L + 1], Ci[L + 1];
#pragma unroll
        for (int t = 0; t <= L; t++) {
            Cr[t] = __shfl_down_sync(0xffffffffu, Br[t], off, G);
            Ci[t] = __shfl_down_sync(0xffffffffu, Bi[t], off, G);
        }
        bins_merge<L>(Br, Cr);
        bins_merge<L>(Bi, Ci);
    }
}

template <int L>
__device__ __forceinline__ void cmul(const double (&ar)[L], const double (&ai)[L], const double (&xr)[L],
                                     const double (&xi)[L], double (&zr)[L], double (&zi)[L]) {
    double Br[L + 1], Bi[L + 1];
    md_zero(Br);
    md_zero(Bi);
    cfma<L, false>(Br, Bi, ar, ai, xr, xi);
    md_renorm(Br, zr);
    md_renorm(Bi, zi);
}

// z = y - a * x, rounded once
template <int L>
__device__ __forceinline__ void cfms(const double (&yr)[L], const double (&yi)[L], const double (&ar)[L],
                                     const double (&ai)[L], const double (&xr)[L], const double (&xi)[L],
                                     double (&zr)[L], double (&zi)[L]) {
    double Br[L + 1], Bi[L + 1];
    md_zero(Br);
    md_zero(Bi);
    cbins_add<L>(Br, Bi, yr, yi);
    cfma<L, true>(Br, Bi, ar, ai, xr, xi);
    md_renorm(Br, zr);
    md_renorm(Bi, zi);
}

// 1/a for a real md number a != 0 by Newton steps y <- y + y (1 - a y) at a
// growing precision: the step on the leading P limbs doubles the correct bits
// up to 53 P (P = 2, 4, 8, ..., L, then once more at L).
template <int L, int P>
__device__ __forceinline__ void recip_step(const double (&a)[L], double (&y)[L]) {
    double ap[P], yp[P], nap[P];
#pragma unroll
    for (int l = 0; l < P; l++) {
        ap[l] = a[l];
        nap[l] = -a[l];
        yp[l] = y[l];
    }
    double B[P + 1], e[P];
    md_zero(B);
    B[0] = 1.0;
    bins_fma<P>(B, nap, yp);
    md_renorm(B, e);
    double B2[P + 1];
    md_zero(B2);
    bins_add<P>(B2, yp);
    bins_fma<P>(B2, yp, e);
    md_renorm(B2, yp);
#pragma unroll
    for (int l = 0; l < L; l++) y[l] = l < P ? yp[l] : 0.0;
    (void)ap;
}

template <int L>
__device__ __forceinline__ void md_recip_fast(const double (&a)[L], double (&y)[L]) {
    md_zero(y);
    y[0] = __ddiv_rn(1.0, a[0]);
    recip_step<L, (L < 2 ? L : 2)>(a, y);
    if (L > 2) recip_step<L, (L < 4 ? L : 4)>(a, y);
    if (L > 4) recip_step<L, (L < 8 ? L : 8)>(a, y);
    if (L > 8) recip_step<L, L>(a, y);
    recip_step<L, L>(a, y);
}

template <int L>
__device__ __forceinline__ void c_recip_fast(const double (&ar)[L], const double (&ai)[L], double (&rr)[L],
                                             double (&ri)[L]) {
    double B[L + 1], den[L], y[L], t[L];
    md_zero(B);
    bins_fma<L>(B, ar, ar);
    bins_fma<L>(B, ai, ai);
    md_renorm(B, den);
    md_recip_fast<L>(den, y);
    md_mul<L>(ar, y, rr);
    md_mul<L>(ai, y, t);
#pragma unroll
    for (int l = 0; l < L; l++) ri[l] = -t[l];
}

// ---- 1. pack: Jacobian coefficients 1..d -> digit elements, rhs -> digit series ----
// Ad[k-1][p][q] = [2][S] digits (part, digit) + exponents Ae[..][2]; Rd / Re in
// the pool's series layout [n][2][S][D] / [n][2][D] (the
// right-hand sides r_k start as b_k, negated for a Newton step).
template <int L>
__global__ void __launch_bounds__(128) ts_pack_kernel(const double *__restrict__ J, const double *__restrict__ b,
                                                      double *__restrict__ Ad, int *__restrict__ Ae,
                                                      double *__restrict__ Rd, int *__restrict__ Re, int n, int D,
                                                      int negate) {
    constexpr int S = digits_for(L);
    const size_t nj = (size_t)n * n * (D - 1), total = nj + (size_t)n * D;
    for (size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (size_t)gridDim.x * blockDim.x) {
        if (g < nj) {  // (k >= 1, p, q): k fastest for coalesced limb reads
            const int k = 1 + (int)(g % (D - 1));
            const size_t pq = g / (D - 1);
            const double *src = J + pq * 2 * L * D + k;
            double *dst = Ad + (((size_t)(k - 1) * n * n) + pq) * 2 * S;
            int *de = Ae + (((size_t)(k - 1) * n * n) + pq) * 2;
#pragma unroll 1
            for (int part = 0; part < 2; part++) {
                double v[L], d[S];
#pragma unroll
                for (int l = 0; l < L; l++) v[l] = src[(size_t)(part * L + l) * D];
                de[part] = limbs_to_digits<L, S>(v, d);
#pragma unroll
                for (int t = 0; t < S; t++) dst[part * S + t] = d[t];
            }
        } else {
            const size_t g2 = g - nj;
            const int k = (int)(g2 % D);
            const size_t p = g2 / D;
#pragma unroll 1
            for (int part = 0; part < 2; part++) {
                double v[L], d[S];
#pragma unroll
                for (int l = 0; l < L; l++) {
                    const double x = b[(p * 2 * L + part * L + l) * D + k];
                    v[l] = negate ? -x : x;
                }
                Re[(p * 2 + part) * D + k] = limbs_to_digits<L, S>(v, d);
#pragma unroll
                for (int t = 0; t < S; t++) Rd[((p * 2 + part) * S + t) * D + k] = d[t];
            }
        }
    }
}

// ---- 2. W = A_0^-1 by Gauss-Jordan elimination with partial pivoting ------------------
// [A_0 | I] -> [I | A_0^-1] (GV83 §3.4): the pivots are those of the LU with
// partial pivoting of A_0 (rows below the pivot see the same Schur
// complement), so A_0 is still factored once; Gauss-Jordan needs n instead of
// 3n dependent steps.  Per step k one block picks the pivot (max |re_0| +
// |im_0|, lowest row on ties), swaps, inverts it (one warp) and scales row k;
// then the grid eliminates column k from every other row.  Complex md in EFT
// level bins; W is converted to digit elements at the end.
template <int L>
__global__ void __launch_bounds__(THREADS) ts_gj_kernel(const double *__restrict__ J, double *__restrict__ Ma,
                                                        double *__restrict__ Mi, int *__restrict__ piv,
                                                        int *__restrict__ status, double *__restrict__ Wd,
                                                        int *__restrict__ We, int n, int D, Barrier *bar) {
    constexpr int E = 2 * L;
    constexpr int S = digits_for(L);
    const int nth = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int tx = threadIdx.x;
    __shared__ double s_m[THREADS];
    __shared__ int s_i[THREADS];
    __shared__ double s_inv[E];

    for (size_t t = tid; t < (size_t)n * n; t += nth) {  // Ma = A_0 (coefficient 0 of J), Mi = I
#pragma unroll
        for (int u = 0; u < E; u++) {
            Ma[t * E + u] = J[(t * E + u) * D];
            Mi[t * E + u] = (u == 0 && t / n == t % n) ? 1.0 : 0.0;
        }
    }
    if (tid == 0) *status = 0;
    grid_sync(bar);

    for (int k = 0; k < n; k++) {
        if (blockIdx.x == 0) {
            double bm = -1.0;
            int bi = n;
            for (int i = k + tx; i < n; i += blockDim.x) {
                const double *a = Ma + ((size_t)i * n + k) * E;
                const double m = __dadd_rn(fabs(a[0]), fabs(a[L]));
                if (m > bm) {
                    bm = m;
                    bi = i;
                }
            }
            s_m[tx] = bm;
            s_i[tx] = bi;
            __syncthreads();
            for (int off = blockDim.x >> 1; off > 0; off >>= 1) {
                if (tx < off) {
                    const double m2 = s_m[tx + off];
                    const int i2 = s_i[tx + off];
                    if (m2 > s_m[tx] || (m2 == s_m[tx] && i2 < s_i[tx])) {
                        s_m[tx] = m2;
                        s_i[tx] = i2;
                    }
                }
                __syncthreads();
            }
            const bool sing = !(s_m[0] > 0.0) || s_i[0] >= n;
            const int p = sing ? k : s_i[0];
            if (p != k)
                for (int t = tx; t < 2 * n * E; t += blockDim.x) {
                    double *M = t < n * E ? Ma : Mi;
                    const int u = t < n * E ? t : t - n * E;
                    double *rk = M + (size_t)k * n * E + u, *rp = M + (size_t)p * n * E + u;
                    const double v = *rk;
                    *rk = *rp;
                    *rp = v;
                }
            __syncthreads();
            if (tx < 32) {  // one warp inverts the pivot
                double ir[L], ii[L];
                if (sing) {
                    md_zero(ir);
                    md_zero(ii);
                } else {
                    double ar[L], ai[L];
                    ld<L>(Ma + ((size_t)k * n + k) * E, ar, ai);
                    c_recip_fast<L>(ar, ai, ir, ii);
                }
                if (tx == 0) {
                    st<L>(s_inv, ir, ii);
                    piv[k] = p;
                    if (sing) atomicOr(status, 1);
                }
            }
            __syncthreads();
            double ir[L], ii[L];
            ld<L>(s_inv, ir, ii);
            // scale row k: Ma[k][c] (c > k) and Mi[k][c] (all c)
            for (int t = tx; t < 2 * n - k - 1; t += blockDim.x) {
                double *a = t < n - k - 1 ? Ma + ((size_t)k * n + k + 1 + t) * E : Mi + ((size_t)k * n + t - (n - k - 1)) * E;
                double ar[L], ai[L], zr[L], zi[L];
                ld<L>(a, ar, ai);
                cmul<L>(ir, ii, ar, ai, zr, zi);
                st<L>(a, zr, zi);
            }
        }
        grid_sync(bar);
        // eliminate column k from rows i != k
        const int cols = 2 * n - k - 1;
        for (int t = tid; t < (n - 1) * cols; t += nth) {
            int i = t / cols;
            const int c = t - i * cols;
            if (i >= k) i++;
            double *a = c < n - k - 1 ? Ma + ((size_t)i * n + k + 1 + c) * E : Mi + ((size_t)i * n + c - (n - k - 1)) * E;
            const double *u = c < n - k - 1 ? Ma + ((size_t)k * n + k + 1 + c) * E : Mi + ((size_t)k * n + c - (n - k - 1)) * E;
            double yr[L], yi[L], lr[L], li[L], ur[L], ui[L], zr[L], zi[L];
            ld<L>(a, yr, yi);
            ld<L>(Ma + ((size_t)i * n + k) * E, lr, li);
            ld<L>(u, ur, ui);
            cfms<L>(yr, yi, lr, li, ur, ui, zr, zi);
            st<L>(a, zr, zi);
        }
        grid_sync(bar);
    }

    // W = Mi -> digit elements [p][q][2][S] + exponents [p][q][2]
    for (size_t t = tid; t < (size_t)n * n; t += nth) {
#pragma unroll 1
        for (int part = 0; part < 2; part++) {
            double v[L], d[S];
#pragma unroll
            for (int l = 0; l < L; l++) v[l] = Mi[t * E + part * L + l];
            We[t * 2 + part] = limbs_to_digits<L, S>(v, d);
#pragma unroll
            for (int u = 0; u < S; u++) Wd[(t * 2 + part) * S + u] = d[u];
        }
    }
}

// ---- 3. the substitution loop on digits ---------------------------------------------
// Dot products sum_q a_q x_q of complex md numbers accumulated EXACTLY as in the
// product kernel (kernels_dig.cuh): a_q are digit elements read from global
// memory (row p of W or of A_{k-j}), x_q a digit vector staged in shared
// memory as planes [part][PADZ + S][n] (PADZ zero planes for the alignment
// shift); one real part per pass, one DFMA per digit pair.
template <int L>
__device__ __forceinline__ void ts_dot_pass(const double *__restrict__ arow, const int *__restrict__ aexp,
                                            const double *__restrict__ xs, const int *__restrict__ xe, int n,
                                            int q0, int G, int part, int eacc, double (&A)[digits_for(L)]) {
    constexpr int S = digits_for(L);
    constexpr int NORM = norm_every(S);
    constexpr int P2 = PADZ + S;
    // part 0 (re): ar xr - ai xi ; part 1 (im): ar xi + ai xr
    const int w1part = part, w2part = 1 - part;
    const long long sgn = part == 0 ? (long long)0x8000000000000000ULL : 0LL;
    md_zero(A);
    int cnt = 0;
    for (int q = q0; q < n; q += G) {
        const double *a = arow + (size_t)q * 2 * S;
        double Ur[S], Ui[S];
#pragma unroll
        for (int s = 0; s < S; s++) {
            Ur[s] = a[s];
            Ui[s] = __longlong_as_double(__double_as_longlong(a[S + s]) ^ sgn);
        }
        const int er = aexp[2 * q], ei = aexp[2 * q + 1];
        const int x1 = xe[w1part * n + q], x2 = xe[w2part * n + q];
        int d1 = eacc - er - x1, d2 = eacc - ei - x2;
        if (er + x1 <= ZERO_E / 2) d1 = 0;  // zero product: any plane will do
        if (ei + x2 <= ZERO_E / 2) d2 = 0;
        const double *W1 = xs + (size_t)w1part * P2 * n + q;
        const double *W2 = xs + (size_t)w2part * P2 * n + q;
        if (__all_sync(__activemask(), d1 <= PADZ && d2 <= PADZ)) {
            const double *V1 = W1 + (size_t)(PADZ - d1) * n, *V2 = W2 + (size_t)(PADZ - d2) * n;
            double w1 = V1[0], w2 = V2[0];
#pragma unroll
            for (int l = 0; l < S; l++) {
                double w1n = 0.0, w2n = 0.0;
                if (l + 1 < S) {
                    w1n = V1[(size_t)(l + 1) * n];
                    w2n = V2[(size_t)(l + 1) * n];
                }
#pragma unroll
                for (int u = 0; u < S - l; u++) {
                    A[u + l] = __fma_rn(Ur[u], w1, A[u + l]);
                    A[u + l] = __fma_rn(Ui[u], w2, A[u + l]);
                }
                w1 = w1n;
                w2 = w2n;
            }
        } else {
#pragma unroll
            for (int l = 0; l < S; l++) {
                const double w1 = (l >= d1) ? W1[(size_t)(PADZ + l - d1) * n] : 0.0;
                const double w2 = (l >= d2) ? W2[(size_t)(PADZ + l - d2) * n] : 0.0;
#pragma unroll
                for (int u = 0; u < S - l; u++) {
                    A[u + l] = __fma_rn(Ur[u], w1, A[u + l]);
                    A[u + l] = __fma_rn(Ui[u], w2, A[u + l]);
                }
            }
        }
        if (++cnt == NORM) {
            carry_pass(A);
            cnt = 0;
        }
    }
    carry_pass(A);
}

// stage coefficient k of the digit series vector (Xd, Xe) [n][2][S][D] as
// planes [part][PADZ + S][n] (+ exponents [part][n]), optionally negated
template <int L>
__device__ __forceinline__ void ts_stage(const double *__restrict__ Xd, const int *__restrict__ Xe, int n, int D,
                                         int k, bool negate, double *xs, int *xe) {
    constexpr int S = digits_for(L);
    constexpr int P2 = PADZ + S;
    for (int t = threadIdx.x; t < 2 * P2 * n; t += blockDim.x) {
        const int part = t / (P2 * n), r = t - part * P2 * n;
        const int pl = r / n, q = r - pl * n;
        double v = 0.0;
        if (pl >= PADZ) {
            v = Xd[(((size_t)q * 2 + part) * S + (pl - PADZ)) * D + k];
            if (negate) v = -v;
        }
        xs[t] = v;
    }
    for (int t = threadIdx.x; t < 2 * n; t += blockDim.x) {
        const int part = t / n, q = t - part * n;
        xe[t] = Xe[((size_t)q * 2 + part) * D + k];
    }
}

// One task: out = (init) + sum_q arow[q] x_q over the G lanes of a group,
// written as digits (zd/ze, coefficient k of a digit series) and optionally
// limbs (zl).  init: an element of a digit series (Id/Ie at coefficient k) or
// none.  All lanes of the warp call this (shuffles); `valid` masks the output.
template <int L>
__device__ __forceinline__ void ts_task(const double *__restrict__ arow, const int *__restrict__ aexp,
                                        const double *xs, const int *xe, int n, int lg, int G, bool valid,
                                        const double *Id, const int *Ie, double *zd, int *ze, double *zl, int D,
                                        int k, double *scratch) {
    constexpr int S = digits_for(L);
    // anchors per part: max exponent over the terms (and the init value + 1)
    int ear = ZERO_E, eai = ZERO_E;
    if (valid) {
        for (int q = lg; q < n; q += G) {
            const int er = aexp[2 * q], ei = aexp[2 * q + 1], xr = xe[q], xi = xe[n + q];
            ear = max(ear, max(er + xr, ei + xi));
            eai = max(eai, max(er + xi, ei + xr));
        }
        if (Id && lg == 0) {
            ear = max(ear, Ie[k] + 1);
            eai = max(eai, Ie[D + k] + 1);
        }
    }
    for (int off = G >> 1; off > 0; off >>= 1) {
        ear = max(ear, __shfl_xor_sync(0xffffffffu, ear, off, G));
        eai = max(eai, __shfl_xor_sync(0xffffffffu, eai, off, G));
    }
    ear = max(ear, ZERO_E);
    eai = max(eai, ZERO_E);
#pragma unroll 1
    for (int part = 0; part < 2; part++) {
        const int eacc = part ? eai : ear;
        double A[S];
        ts_dot_pass<L>(arow, aexp, xs, xe, valid ? n : 0, lg, G, part, eacc, A);
        if (valid && Id && lg == 0) {  // the init value: digit s has weight R^(eI-1-s) = slot s + eacc-1-eI
            const int eI = Ie[part * D + k];
            if (eI > ZERO_E / 2) {
                const int dI = eacc - 1 - eI;
                const double *src = Id + (size_t)part * S * D + k;
#pragma unroll
                for (int t = 0; t < S; t++) {
                    const int s = t - dI;
                    if (s >= 0 && s < S) A[t] = __dadd_rn(A[t], src[(size_t)s * D]);
                }
            }
        }
        for (int off = G >> 1; off > 0; off >>= 1) {
#pragma unroll
            for (int s = 0; s < S; s++) A[s] = __dadd_rn(A[s], __shfl_xor_sync(0xffffffffu, A[s], off, G));
        }
        if (valid && lg == 0) conv_dig_emit<L>(A, eacc, zd, ze, zl, D, k, part, scratch);
    }
}

template <int L>
__global__ void __launch_bounds__(128, L <= 8 ? 3 : 2) ts_loop_kernel(
    const double *__restrict__ Ad, const int *__restrict__ Ae, const double *__restrict__ Wd,
    const int *__restrict__ We, double *__restrict__ Rd, int *__restrict__ Re, double *__restrict__ Xd,
    int *__restrict__ Xe, double *__restrict__ dx, int n, int D, Barrier *bar) {
    constexpr int S = digits_for(L);
    constexpr int P2 = PADZ + S;
    extern __shared__ __align__(16) double sm[];
    double *xs = sm;                                  // [2][P2][n]
    int *xe = (int *)(xs + (size_t)2 * P2 * n);       // [2][n]
    double *scr = (double *)(xe + 2 * n + 2);         // [blockDim/4][S+2] emit scratch (one per group leader)
    const int nth = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const size_t SER = (size_t)2 * S * D;             // doubles per digit series

    for (int j = 0; j < D; j++) {
        // dx_j = W r_j: G lanes per row p
        ts_stage<L>(Rd, Re, n, D, j, false, xs, xe);
        __syncthreads();
        {
            int G = 4;
            while (G < 32 && (long long)n * G * 2 < nth) G <<= 1;
            const int ng = nth / G, g = tid / G, lg = tid % G;
            double *scratch = scr + (size_t)(threadIdx.x / 4) * (S + 2);
            for (int base = 0; base < n; base += ng) {
                const int p = base + g;
                const bool valid = p < n;
                const int pp = valid ? p : 0;
                ts_task<L>(Wd + (size_t)pp * n * 2 * S, We + (size_t)pp * n * 2, xs, xe, n, lg, G, valid, nullptr,
                           nullptr, Xd + pp * SER, Xe + (size_t)pp * 2 * D, dx + (size_t)pp * 2 * L * D, D, j,
                           scratch);
            }
        }
        grid_sync(bar);
        if (j + 1 == D) break;

        // r_k -= A_{k-j} dx_j for k = j+1..d: G lanes per (k, p)
        ts_stage<L>(Xd, Xe, n, D, j, true, xs, xe);
        __syncthreads();
        {
            const int T = (D - 1 - j) * n;
            int G = 4;
            while (G < 32 && (long long)T * G < nth) G <<= 1;
            const int ng = nth / G, g = tid / G, lg = tid % G;
            double *scratch = scr + (size_t)(threadIdx.x / 4) * (S + 2);
            for (int base = 0; base < T; base += ng) {
                const int task = base + g;
                const bool valid = task < T;
                const int k = j + 1 + (valid ? task / n : 0), p = valid ? task % n : 0;
                const size_t row = ((size_t)(k - j - 1) * n + p) * n;
                ts_task<L>(Ad + row * 2 * S, Ae + row * 2, xs, xe, n, lg, G, valid, Rd + p * SER,
                           Re + (size_t)p * 2 * D, Rd + p * SER, Re + (size_t)p * 2 * D, nullptr, D, k, scratch);
            }
        }
        grid_sync(bar);
    }
}

__host__ __device__ inline size_t ts_loop_smem(int S, int n, int threads) {
    return (size_t)2 * (PADZ + S) * n * sizeof(double) + (size_t)(2 * n + 2) * sizeof(int) +
           (size_t)(threads / 4) * (S + 2) * sizeof(double);
}

}  // namespace ts
}  // namespace mdps

using namespace mdps;

struct mdps_solver {
    int n = 0, D = 0, L = 0, S = 0;
    int device = 0;
    double *Ad = nullptr, *Ma = nullptr, *Mi = nullptr, *Wd = nullptr, *Rd = nullptr, *Xd = nullptr;
    int *Ae = nullptr, *We = nullptr, *Re = nullptr, *Xe = nullptr;
    int *piv = nullptr, *status = nullptr;
    ts::Barrier *bar = nullptr;
    int grid_gj = 0, grid_loop = 0;
    size_t smem_loop = 0;
    size_t bytes = 0;
    cudaStream_t last = nullptr;
};

#define TS_TRY(call, code)                                                              \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            mdps_internal_set_error(std::string(#call) + ": " + cudaGetErrorString(e_)); \
            return code;                                                                \
        }                                                                               \
    } while (0)

template <int L>
struct TsGeom {
    static int run(mdps_solver *s) {
        int dev = 0, sms = 0, per_gj = 0, per_loop = 0;
        TS_TRY(cudaGetDevice(&dev), MDPS_ECUDA);
        TS_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), MDPS_ECUDA);
        s->smem_loop = ts::ts_loop_smem(digits_for(L), s->n, 128);
        TS_TRY(cudaFuncSetAttribute(ts::ts_loop_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)s->smem_loop),
               MDPS_ECUDA);
        TS_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_gj, ts::ts_gj_kernel<L>, ts::THREADS, 0),
               MDPS_ECUDA);
        TS_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_loop, ts::ts_loop_kernel<L>, 128, s->smem_loop),
               MDPS_ECUDA);
        if (per_gj < 1 || per_loop < 1) {
            mdps_internal_set_error("solver kernels do not fit on an SM");
            return MDPS_ECUDA;
        }
        s->grid_gj = sms * per_gj;
        s->grid_loop = sms * per_loop;
        return MDPS_OK;
    }
};

template <int L>
struct TsRun {
    static int run(mdps_solver *s, const double *J, const double *b, double *dx, int negate, cudaStream_t st) {
        const int n = s->n, D = s->D;
        const size_t total = (size_t)n * n * (D - 1) + (size_t)n * D;
        const int pb = (int)std::min<size_t>((total + 127) / 128, 148 * 32);
        ts::ts_pack_kernel<L><<<pb, 128, 0, st>>>(J, b, s->Ad, s->Ae, s->Rd, s->Re, n, D, negate);
        TS_TRY(cudaGetLastError(), MDPS_ECUDA);
        TS_TRY(cudaMemsetAsync(s->bar, 0, sizeof(ts::Barrier), st), MDPS_ECUDA);
        {
            void *args[] = {(void *)&J, (void *)&s->Ma, (void *)&s->Mi, (void *)&s->piv, (void *)&s->status,
                            (void *)&s->Wd, (void *)&s->We, (void *)&s->n, (void *)&s->D, (void *)&s->bar};
            TS_TRY(cudaLaunchCooperativeKernel((const void *)ts::ts_gj_kernel<L>, dim3(s->grid_gj), dim3(ts::THREADS),
                                               args, 0, st),
                   MDPS_ECUDA);
        }
        {
            const double *Ad = s->Ad, *Wd = s->Wd;
            const int *Ae = s->Ae, *We = s->We;
            void *args[] = {(void *)&Ad, (void *)&Ae, (void *)&Wd, (void *)&We, (void *)&s->Rd, (void *)&s->Re,
                            (void *)&s->Xd, (void *)&s->Xe, (void *)&dx, (void *)&s->n, (void *)&s->D,
                            (void *)&s->bar};
            TS_TRY(cudaLaunchCooperativeKernel((const void *)ts::ts_loop_kernel<L>, dim3(s->grid_loop), dim3(128),
                                               args, s->smem_loop, st),
                   MDPS_ECUDA);
        }
        return MDPS_OK;
    }
};

template <template <int> class Fn, typename... Args>
static int ts_dispatch(int L, Args &&...args) {
    switch (L) {
        case 2: return Fn<2>::run(args...);
        case 3: return Fn<3>::run(args...);
        case 4: return Fn<4>::run(args...);
        case 5: return Fn<5>::run(args...);
        case 8: return Fn<8>::run(args...);
        case 10: return Fn<10>::run(args...);
    }
    mdps_internal_set_error("unsupported limb count");
    return MDPS_EINVAL;
}

static void solver_free(mdps_solver *s) {
    cudaFree(s->Ad);
    cudaFree(s->Ae);
    cudaFree(s->Ma);
    cudaFree(s->Mi);
    cudaFree(s->Wd);
    cudaFree(s->We);
    cudaFree(s->Rd);
    cudaFree(s->Re);
    cudaFree(s->Xd);
    cudaFree(s->Xe);
    cudaFree(s->piv);
    cudaFree(s->status);
    cudaFree(s->bar);
}

extern "C" mdps_solver *mdps_solver_create(int32_t n, int32_t degree, int32_t limbs) {
    if (n < 1 || n > 256 || degree < 0 || degree > 255 ||
        !(limbs == 2 || limbs == 3 || limbs == 4 || limbs == 5 || limbs == 8 || limbs == 10)) {
        mdps_internal_set_error("mdps_solver_create: need 1 <= n <= 256, 0 <= degree <= 255, limbs in {2,3,4,5,8,10}");
        return nullptr;
    }
    mdps_solver *s = new (std::nothrow) mdps_solver();
    if (!s) {
        mdps_internal_set_error("out of host memory");
        return nullptr;
    }
    s->n = n;
    s->D = degree + 1;
    s->L = limbs;
    s->S = digits_for(limbs);
    cudaGetDevice(&s->device);
    const size_t nn = (size_t)n * n, D = s->D, S = s->S;
    const size_t sz[] = {std::max<size_t>(1, nn * (D - 1) * 2 * S) * 8, std::max<size_t>(1, nn * (D - 1) * 2) * 4,
                         nn * 2 * limbs * 8, nn * 2 * limbs * 8, nn * 2 * S * 8, nn * 2 * 4,
                         n * 2 * S * D * 8, n * 2 * D * 4, n * 2 * S * D * 8, n * 2 * D * 4,
                         n * sizeof(int), sizeof(int), sizeof(ts::Barrier)};
    void **ptrs[] = {(void **)&s->Ad, (void **)&s->Ae, (void **)&s->Ma, (void **)&s->Mi, (void **)&s->Wd,
                     (void **)&s->We, (void **)&s->Rd, (void **)&s->Re, (void **)&s->Xd, (void **)&s->Xe,
                     (void **)&s->piv, (void **)&s->status, (void **)&s->bar};
    bool ok = true;
    for (size_t i = 0; i < sizeof(sz) / sizeof(sz[0]) && ok; i++) {
        ok = cudaMalloc(ptrs[i], sz[i]) == cudaSuccess;
        s->bytes += sz[i];
    }
    if (!ok) {
        cudaGetLastError();
        solver_free(s);
        delete s;
        mdps_internal_set_error("mdps_solver_create: device allocation failed");
        return nullptr;
    }
    cudaMemset(s->piv, 0, n * sizeof(int));
    cudaMemset(s->status, 0, sizeof(int));
    if (ts_dispatch<TsGeom>(limbs, s) != MDPS_OK) {
        solver_free(s);
        delete s;
        return nullptr;
    }
    return s;
}

int mdps_solve_internal(mdps_solver *s, const double *J, const double *b, double *dx, int negate,
                        cudaStream_t st) {
    if (!s || !J || !b || !dx) {
        mdps_internal_set_error("mdps_solve: NULL argument");
        return MDPS_EINVAL;
    }
    const size_t ser = (size_t)2 * s->L * s->D;
    const char *x0 = (const char *)dx, *x1 = x0 + (size_t)s->n * ser * sizeof(double);
    auto overlaps = [&](const void *p, size_t bytes) {
        const char *a = (const char *)p;
        return a < x1 && x0 < a + bytes;
    };
    if (overlaps(J, (size_t)s->n * s->n * ser * sizeof(double)) || overlaps(b, (size_t)s->n * ser * sizeof(double))) {
        mdps_internal_set_error("mdps_solve: dx_out aliases an input");
        return MDPS_EINVAL;
    }
    s->last = st;
    return ts_dispatch<TsRun>(s->L, s, J, b, dx, negate, st);
}

extern "C" int mdps_solve(mdps_solver *s, const double *J, const double *b, double *dx, mdps_stream_t stream) {
    return mdps_solve_internal(s, J, b, dx, 0, (cudaStream_t)stream);
}

extern "C" int mdps_solver_status(mdps_solver *s, int32_t *pivots, int32_t *singular) {
    if (!s) {
        mdps_internal_set_error("mdps_solver_status: NULL solver");
        return MDPS_EINVAL;
    }
    TS_TRY(cudaStreamSynchronize(s->last), MDPS_ECUDA);
    if (pivots) TS_TRY(cudaMemcpy(pivots, s->piv, s->n * sizeof(int), cudaMemcpyDeviceToHost), MDPS_ECUDA);
    if (singular) {
        int v = 0;
        TS_TRY(cudaMemcpy(&v, s->status, sizeof(int), cudaMemcpyDeviceToHost), MDPS_ECUDA);
        *singular = v & 1;
    }
    return MDPS_OK;
}

// complex md multiply-adds of one solve: Gauss-Jordan (row scaling + the
// elimination of [A_0 | I]) and the substitution loop (d+1 products W r_j and
// the n^2 d(d+1)/2 right-hand-side updates)
static int64_t solver_cfma_gj(int64_t n) {
    int64_t gj = 0;
    for (int64_t k = 0; k < n; k++) gj += (2 * n - k - 1) * n;
    return gj;
}
static int64_t solver_cfma_loop(int64_t n, int64_t D) { return D * n * n + n * n * D * (D - 1) / 2; }

extern "C" int mdps_solver_stats(const mdps_solver *s, mdps_solver_info *out) {
    if (!s || !out) {
        mdps_internal_set_error("mdps_solver_stats: NULL argument");
        return MDPS_EINVAL;
    }
    std::memset(out, 0, sizeof *out);
    const int64_t gj = solver_cfma_gj(s->n), loop = solver_cfma_loop(s->n, s->D);
    out->complex_fma = gj + loop;
    // EFT bins for Gauss-Jordan, digit DFMAs (4 truncated S x S triangles per
    // complex term) for the loop
    out->fp64_ops = gj * 4 * ops_bins_fma(s->L) + loop * 4 * (int64_t)(s->S * (s->S + 1) / 2);
    out->launches = 3;
    out->grid_blocks = s->grid_loop;
    out->workspace_bytes = s->bytes;
    return MDPS_OK;
}

extern "C" void mdps_solver_destroy(mdps_solver *s) {
    if (!s) return;
    cudaDeviceSynchronize();
    solver_free(s);
    delete s;
}
