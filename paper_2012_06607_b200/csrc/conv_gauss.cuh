// conv_gauss.cuh — product jobs on digit planes with three real products per
// complex term (MDPS_ALGO_DIGITS, the default product kernel).
//
// For x_i = a + ib and y_j = c + id the complex product needs
//     P1 = c (a + b),   P2 = a (d - c),   P3 = b (c + d),
//     re = P1 - P3 = ac - bd,   im = P1 + P2 = ad + bc
// (Gauss).  In floating point the trick loses accuracy to cancellation, which
// is why the md path (conv_eft) uses four products (reading R5); on
// digit planes every product and every sum is EXACT (integer digits below
// 2^53), so re and im come out exact and the trick costs nothing in accuracy:
// 3 instead of 4 digit convolutions per term (-25% DFMAs, +3S DADDs for the
// operand sums).  The sums a+b, d-c, c+d need a and b (c and d) on one
// digit grid: after staging, every coefficient's two parts are aligned to
// the larger part exponent (the smaller part shifted down, its lowest digits
// truncated: precision stays 2^-((S-1)*BETA) relative to |x_i|, normwise).
//
// Mapping: as conv_dig (one job per block for D >= 32, T = ceil(D/2) output
// pairs x F lanes, folded triangle), but each lane takes a CONTIGUOUS range
// of the D+1 fold iterations, so at most one lane per pair crosses from
// output k1 = t to k2 = D-1-t and parks its k1 partial in a per-pair slot;
// the other partials are combined by warp shuffles.  Three passes (P1, P2,
// P3) over the lane's terms; P1 of both outputs waits in shared memory until
// P2 gives im and P3 gives re, each emitted with its own exponent.
#pragma once
#include "conv_dig.cuh"

namespace mdps {

// shared memory: per job x planes [S][2][D], y planes [PADZ+S][2][D], part
// exponents [2 series][2][D], aligned exponents [2 series][D]; per output pair
// 4 slots of S+2 doubles (P1 of k1, P1 of k2, park, emit scratch); mbarrier
__host__ __device__ inline size_t conv_g_smem(int S, int D, int P, int T) {
    const size_t per_job = (size_t)2 * S * D + (size_t)2 * (PADZ + S) * D;
    return (size_t)P * per_job * sizeof(double) + ((size_t)P * T + 1) * 4 * (S + 2) * sizeof(double) +
           (size_t)P * 6 * D * sizeof(int) + 16;
}

// Z = [c2, c1, c0, A_1 .. A_{S-1}] of a carry-passed accumulator (weights
// R^(eacc-u)); all entries small, so Z vectors add and subtract exactly
template <int S>
__device__ __forceinline__ void acc_to_z(const double (&A)[S], double (&Z)[S + 2]) {
    double a0 = A[0];
    const double c2 = rint_magic(__dmul_rn(a0, INV_RADIX * INV_RADIX));
    a0 = __fma_rn(-c2, RADIX * RADIX, a0);
    const double c1 = rint_magic(__dmul_rn(a0, INV_RADIX));
    Z[0] = c2;
    Z[1] = c1;
    Z[2] = __fma_rn(-c1, RADIX, a0);
#pragma unroll
    for (int s = 1; s < S; s++) Z[s + 2] = A[s];
}

// normalise Z and write one output (k, part): digits + exponent (zd) and/or
// limbs (zl).  scratch: S+2 doubles of shared memory.
template <int L>
__device__ __forceinline__ void emit_z(double (&Z)[digits_for(L) + 2], int eacc, double *zd, int *ze, double *zl,
                                       int D, int k, int part, double *scratch) {
    constexpr int S = digits_for(L);
    carry_normalize(Z);
    if (zd) {
        int z0 = S + 2;
#pragma unroll
        for (int u = S + 1; u >= 0; u--) {
            scratch[u] = Z[u];
            if (Z[u] != 0.0) z0 = u;
        }
        const int e = (z0 >= S + 2 || eacc <= ZERO_E / 2) ? ZERO_E : eacc + 1 - z0;
        const double *src = scratch + z0;
        const int avail = S + 2 - z0;
#pragma unroll
        for (int s = 0; s < S; s++) zd[(part * S + s) * D + k] = (s < avail && e != ZERO_E) ? src[s] : 0.0;
        ze[part * D + k] = e;
    }
    if (zl) {
        double out[L];
        digits_to_limbs<L, S + 2, true>(Z, eacc + 1, out);  // Z_u has weight R^(eacc - u)
#pragma unroll
        for (int p = 0; p < L; p++) zl[(part * L + p) * D + k] = out[p];
    }
}

// one pass (0: P1 = c(a+b), 1: P2 = a(d-c), 2: P3 = b(c+d)) over the lane's
// contiguous fold iterations [j0, j1).  One code copy serves the three passes
// (instruction-cache footprint: the FMA block is ~5 KB of SASS per copy): the
// pass selects the x operand (a+b, a or b) in a small uniform branch and the
// y operand w = (d masked) + (c sign-flipped) with integer masks.
template <int L, int DT>
__device__ __forceinline__ void conv_g_pass(const double *__restrict__ sx, const double *__restrict__ sy,
                                            const int *__restrict__ ex, const int *__restrict__ ey, int Drt,
                                            int pass, int t, int j0, int j1, int eacc1, int eacc2,
                                            double (&A)[digits_for(L)], double *park) {
    constexpr int S = digits_for(L);
    constexpr int NORM = norm_every(S);
    const int D = DT > 0 ? DT : Drt;
    const int D2 = 2 * D;
    const long long dmask = pass == 0 ? 0LL : -1LL;                                 // w = c | d - c | c + d
    const long long csign = pass == 1 ? (long long)0x8000000000000000ULL : 0LL;
    const int uoff = pass == 2 ? 1 : 0;
    md_zero(A);
    int cnt = 0;
    for (int j = j0; j < j1; j++) {
        const bool first = j <= t;
        if (!first && j > j0 && j - 1 <= t) {  // this lane crosses the fold: park k1
            carry_pass(A);
#pragma unroll
            for (int s = 0; s < S; s++) {
                park[s] = A[s];
                A[s] = 0.0;
            }
            cnt = 0;
        }
        const int i = first ? j : j - t - 1;
        const int kk = (first ? t : D - 1 - t) - i;
        const int eacc = first ? eacc1 : eacc2;
        double U[S];
        const double *ux = sx + i;
        if (pass == 0) {
#pragma unroll
            for (int s = 0; s < S; s++) U[s] = __dadd_rn(ux[(2 * s) * D], ux[(2 * s + 1) * D]);
        } else {
#pragma unroll
            for (int s = 0; s < S; s++) U[s] = ux[(2 * s + uoff) * D];
        }
        const int exy = ex[i] + ey[kk];
        const int d = exy <= ZERO_E / 2 ? 0 : eacc - exy;  // zero product: any plane will do
        if (__all_sync(__activemask(), d <= PADZ)) {
            const double *Wc = sy + (PADZ - d) * D2 + kk;  // c planes; d planes at +D
            double wc = Wc[0], wd = Wc[D];
#pragma unroll
            for (int l = 0; l < S; l++) {
                double wcn = 0.0, wdn = 0.0;
                if (l + 1 < S) {
                    wcn = Wc[(l + 1) * D2];
                    wdn = Wc[(l + 1) * D2 + D];
                }
                const double w = __dadd_rn(__longlong_as_double(__double_as_longlong(wd) & dmask),
                                           __longlong_as_double(__double_as_longlong(wc) ^ csign));
#pragma unroll
                for (int u = 0; u < S - l; u++) A[u + l] = __fma_rn(U[u], w, A[u + l]);
                wc = wcn;
                wd = wdn;
            }
        } else {
            const double *Wc = sy + kk;
#pragma unroll
            for (int l = 0; l < S; l++) {
                double wc = 0.0, wd = 0.0;
                if (l >= d) {
                    wc = Wc[(PADZ + l - d) * D2];
                    wd = Wc[(PADZ + l - d) * D2 + D];
                }
                const double w = __dadd_rn(__longlong_as_double(__double_as_longlong(wd) & dmask),
                                           __longlong_as_double(__double_as_longlong(wc) ^ csign));
#pragma unroll
                for (int u = 0; u < S - l; u++) A[u + l] = __fma_rn(U[u], w, A[u + l]);
            }
        }
        if (++cnt == NORM) {
            carry_pass(A);
            cnt = 0;
        }
    }
    carry_pass(A);
}

// sums of the group's partials: X = k1 (without the park), Y = k2; F lanes
// of a pair are adjacent lanes
template <int S>
__device__ __forceinline__ void pair_reduce(const double (&A)[S], bool fin_k2, int F, double (&X)[S],
                                            double (&Y)[S]) {
#pragma unroll
    for (int s = 0; s < S; s++) {
        X[s] = fin_k2 ? 0.0 : A[s];
        Y[s] = fin_k2 ? A[s] : 0.0;
    }
    for (int off = F >> 1; off > 0; off >>= 1) {
#pragma unroll
        for (int s = 0; s < S; s++) {
            X[s] = __dadd_rn(X[s], __shfl_xor_sync(0xffffffffu, X[s], off));
            Y[s] = __dadd_rn(Y[s], __shfl_xor_sync(0xffffffffu, Y[s], off));
        }
    }
}

// Cold path, kept out of line so the hot loop's register budget is not
// sized by the epilogue: turn one reduced partial into its Z vector; pass 0
// stores P1, pass 1 emits im = P1 + P2, pass 2 emits re = P1 - P3.
template <int L>
__device__ __noinline__ void conv_g_output(const double *acc, const double *park, double *p1, int pass, int eacc,
                                           bool emit, double *zd, int *ze, double *zl, int D, int k,
                                           double *scratch) {
    constexpr int S = digits_for(L);
    double A[S], Z[S + 2];
#pragma unroll
    for (int s = 0; s < S; s++) A[s] = park ? __dadd_rn(acc[s], park[s]) : acc[s];
    acc_to_z(A, Z);
    if (pass == 0) {
#pragma unroll
        for (int u = 0; u < S + 2; u++) p1[u] = Z[u];
        return;
    }
#pragma unroll
    for (int u = 0; u < S + 2; u++) Z[u] = pass == 1 ? __dadd_rn(p1[u], Z[u]) : __dsub_rn(p1[u], Z[u]);
    if (emit) emit_z<L>(Z, eacc, zd, ze, zl, D, k, pass == 1 ? 1 : 0, scratch);
}

// Stage the digit planes of both inputs of every job of the block (TMA bulk
// copies for even D, plain loads otherwise), the PADZ zero planes and the
// part exponents, then align each coefficient's two parts to the larger part
// exponent (shx: aligned exponents [P][2 series][D]).  Ends with a block sync.
template <int L>
__device__ __forceinline__ void stage_aligned(const double *__restrict__ dpool, const int *__restrict__ epool,
                                              const int *__restrict__ jobs, int njobs, int D, int P, int job0,
                                              double *sdig, int *sexp, int *shx, uint64_t *bar) {
    constexpr int S = digits_for(L);
    const int SX = 2 * S * D, SY = 2 * (PADZ + S) * D;
    const bool use_tma = (D & 1) == 0;
    if (use_tma) {
        if (threadIdx.x == 0) mbar_init(bar, 1);
        __syncthreads();
        if (threadIdx.x < 32) {
            const int nrows = P * 4 * S;
            if (threadIdx.x == 0) mbar_expect_tx(bar, (unsigned)(nrows * D * 8));
            __syncwarp();
            for (int row = threadIdx.x; row < nrows; row += 32) {
                const int jl = row / (4 * S), rem = row - jl * 4 * S;
                const int which = rem / (2 * S), ps = rem - which * 2 * S;
                const int part = ps / S, s = ps - part * S;
                const int job = min(job0 + jl, njobs - 1);
                const double *g = dpool + (size_t)jobs[4 * job + which] * dig_slot_stride(S, D) + (size_t)ps * D;
                double *dst = sdig + (size_t)jl * (SX + SY) + (which ? SX + ((PADZ + s) * 2 + part) * D
                                                                       : (s * 2 + part) * D);
                bulk_g2s(dst, g, (unsigned)(D * 8), bar);
            }
        }
    } else {
        for (int idx = threadIdx.x; idx < P * 4 * S * D; idx += blockDim.x) {
            const int row = idx / D, k = idx - row * D;
            const int jl = row / (4 * S), rem = row - jl * 4 * S;
            const int which = rem / (2 * S), ps = rem - which * 2 * S;
            const int part = ps / S, s = ps - part * S;
            const int job = min(job0 + jl, njobs - 1);
            const double *g = dpool + (size_t)jobs[4 * job + which] * dig_slot_stride(S, D) + (size_t)ps * D;
            double *dst = sdig + (size_t)jl * (SX + SY) + (which ? SX + ((PADZ + s) * 2 + part) * D
                                                                   : (s * 2 + part) * D);
            dst[k] = __ldg(g + k);
        }
    }
    for (int idx = threadIdx.x; idx < P * 2 * PADZ * D; idx += blockDim.x) {
        const int jl = idx / (2 * PADZ * D), r = idx - jl * 2 * PADZ * D;
        sdig[(size_t)jl * (SX + SY) + SX + r] = 0.0;
    }
    for (int idx = threadIdx.x; idx < P * 4 * D; idx += blockDim.x) {
        const int jl = idx / (4 * D), r = idx - jl * 4 * D;
        const int which = r / (2 * D), r2 = r - which * 2 * D;
        const int job = min(job0 + jl, njobs - 1);
        sexp[idx] = epool[(size_t)jobs[4 * job + which] * 2 * D + r2];
    }
    if (use_tma) mbar_wait(bar, 0);
    __syncthreads();

    // ---- align each coefficient's parts to the larger exponent
    for (int idx = threadIdx.x; idx < P * 2 * D; idx += blockDim.x) {
        const int jl = idx / (2 * D), r = idx - jl * 2 * D;
        const int which = r / D, col = r - which * D;
        const int er = sexp[(jl * 2 + which) * 2 * D + col], ei = sexp[(jl * 2 + which) * 2 * D + D + col];
        const int e = max(er, ei);
        shx[idx] = e;
        const int small = er < ei ? 0 : 1;  // the part to shift down
        const int sh = er < ei ? ei - er : er - ei;
        if (sh > 0 && e > ZERO_E / 2 && min(er, ei) > ZERO_E / 2) {
            double *base = sdig + (size_t)jl * (SX + SY) + (which ? SX + (PADZ * 2 + small) * D : small * D) + col;
            for (int s = S - 1; s >= 0; s--)
                base[(size_t)s * 2 * D] = s >= sh ? base[(size_t)(s - sh) * 2 * D] : 0.0;
        }
    }
    __syncthreads();

}

template <int L, int DT>
__global__ void __launch_bounds__(DT == 128 || DT == 0 ? 256 : 128,
                                  DT == 128 || DT == 0 ? 1 : (L <= 8 ? 3 : 2))
    conv_g_kernel(double *__restrict__ dpool, int *__restrict__ epool, double *__restrict__ lpool,
                  const int *__restrict__ jobs, int njobs, int Drt, int T, int F, int P) {
    constexpr int S = digits_for(L);
    constexpr int ZS = S + 2;
    const int D = DT > 0 ? DT : Drt;
    const int SX = 2 * S * D, SY = 2 * (PADZ + S) * D;
    const int threads_per_job = T * F;
    extern __shared__ __align__(16) double sm[];
    double *sdig = sm;                                   // [P][SX + SY]
    double *sgrp = sm + (size_t)P * (SX + SY);           // [P*T][4][ZS]
    int *sexp = (int *)(sgrp + ((size_t)P * T + 1) * 4 * ZS);  // [P][2 series][2 parts][D]
    int *shx = sexp + (size_t)P * 4 * D;                 // [P][2 series][D] aligned exponents
    uint64_t *bar = reinterpret_cast<uint64_t *>(shx + (size_t)P * 2 * D);
    const int job0 = blockIdx.x * P;

    stage_aligned<L>(dpool, epool, jobs, njobs, D, P, job0, sdig, sexp, shx, bar);

    const int jl0 = threadIdx.x / threads_per_job;
    const int jl = min(jl0, P - 1);  // padding lanes shadow the last job
    const int r = threadIdx.x - jl0 * threads_per_job;
    const int t = min(r / F, T - 1), f = r - (r / F) * F;
    const double *sx = sdig + (size_t)jl * (SX + SY), *sy = sx + SX;
    const int *ex = shx + jl * 2 * D, *ey = ex + D;
    const int Q = (D + 1 + F - 1) / F;
    const int j0 = min(f * Q, D + 1), j1 = min(j0 + Q, D + 1);

    // ---- anchors: e_acc of k1 and k2 (one per output: all three products of a term share it)
    int ea1 = ZERO_E, ea2 = ZERO_E;
    for (int j = j0; j < j1; j++) {
        const bool first = j <= t;
        const int i = first ? j : j - t - 1;
        const int kk = (first ? t : D - 1 - t) - i;
        const int e = ex[i] + ey[kk];
        if (first) ea1 = max(ea1, e);
        else ea2 = max(ea2, e);
    }
    for (int off = F >> 1; off > 0; off >>= 1) {
        ea1 = max(ea1, __shfl_xor_sync(0xffffffffu, ea1, off));
        ea2 = max(ea2, __shfl_xor_sync(0xffffffffu, ea2, off));
    }
    ea1 = max(ea1, ZERO_E);
    ea2 = max(ea2, ZERO_E);

    const int job = job0 + jl0;
    const bool writer = jl0 < P && job < njobs && r / F < T;
    double *zd = dpool, *zl = nullptr;
    int *ze = epool;
    int wdig = 0;
    if (writer) {
        const int out = jobs[4 * job + 2], code = jobs[4 * job + 3];
        zd = dpool + (size_t)out * dig_slot_stride(S, D);
        ze = epool + (size_t)out * 2 * D;
        wdig = code & 1;
        if (code & 2) zl = lpool + (size_t)(code >> 2) * 2 * L * D;
    }
    // per output pair: [P1 k1][P1 k2][park][scratch]; padding lanes get a dummy group
    const bool real_lane = jl0 < P && r / F < T;
    double *grp = sgrp + (real_lane ? ((size_t)jl * T + t) : (size_t)P * T) * 4 * ZS;
    double *park = grp + 2 * ZS, *scratch = grp + 3 * ZS;
    const int k1 = t, k2 = D - 1 - t;
    const bool fin_k2 = j1 > j0 && j1 - 1 > t;  // the lane's last term belongs to k2
    const bool emit1 = writer && f == 0, emit2 = writer && f == (F > 1 ? 1 : 0) && k2 != k1;

#pragma unroll 1
    for (int pass = 0; pass < 3; pass++) {
        if (f == 0) {
#pragma unroll
            for (int s = 0; s < S; s++) park[s] = 0.0;
        }
        __syncwarp();
        double A[S];
        conv_g_pass<L, DT>(sx, sy, ex, ey, D, pass, t, j0, j1, ea1, ea2, A, park);
        double X[S], Y[S];
        pair_reduce(A, fin_k2, F, X, Y);
        __syncwarp();
        // lane 0 owns k1 (X + park), lane 1 owns k2 (Y); F == 1: one lane owns both
        if (F == 1) {
            conv_g_output<L>(X, park, grp, pass, ea1, emit1, wdig ? zd : nullptr, ze, zl, D, k1, park);
            if (k2 != k1)
                conv_g_output<L>(Y, nullptr, grp + ZS, pass, ea2, emit2, wdig ? zd : nullptr, ze, zl, D, k2, scratch);
        } else if (f < 2) {  // one call site: lanes 0 and 1 run the epilogue together
            if (f == 1) {
#pragma unroll
                for (int s = 0; s < S; s++) X[s] = Y[s];
            }
            if (f == 0 || k2 != k1)
                conv_g_output<L>(X, f == 0 ? park : nullptr, grp + f * ZS, pass, f == 0 ? ea1 : ea2,
                                 f == 0 ? emit1 : emit2, wdig ? zd : nullptr, ze, zl, D, f == 0 ? k1 : k2,
                                 f == 0 ? park : scratch);
        }
        __syncwarp();
    }
}

}  // namespace mdps
