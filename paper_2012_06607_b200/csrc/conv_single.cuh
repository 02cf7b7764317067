// conv_single.cuh — product jobs on digit planes, real and imaginary parts
// in ONE pass (MDPS_ALGO_DIGITS default for L >= 8).
//
// After staging, each coefficient's two parts are aligned to the larger part
// exponent (conv_gauss.cuh), so every term x_i y_{k-i} has a single alignment
// shift: per term the 2S digits of x_i are loaded once into registers and
// per digit row two digits of y (c_l, d_l) are streamed from shared memory,
// feeding 4 DFMAs per digit pair into the real and imaginary accumulators
//     re += a c - b d,   im += a d + b c.
// Against the two-pass kernel (conv_dig.cuh) this halves the x loads and the
// per-term overhead and gives every warp two independent accumulator sets
// (ILP), at the price of 4S live doubles (two blocks per SM at L >= 8).
// Lanes take contiguous ranges of the folded triangle (conv_gauss.cuh): at
// most one lane per output pair parks its k1 partials.
#pragma once
#include "conv_gauss.cuh"

namespace mdps {

// per job: x planes [S][2][D], y planes [PADZ+S][2][D], part exponents
// [2 series][2][D], aligned exponents [2 series][D]; per output pair (+1
// dummy for padding lanes) 3 slots of S+2 doubles: park re, park im,
// scratch; mbarrier
__host__ __device__ inline size_t conv_s_smem(int S, int D, int P, int T) {
    const size_t per_job = (size_t)2 * S * D + (size_t)2 * (PADZ + S) * D;
    return (size_t)P * per_job * sizeof(double) + ((size_t)P * T + 1) * 3 * (S + 2) * sizeof(double) +
           (size_t)P * 6 * D * sizeof(int) + 16;
}

template <int L, int DT>
__device__ __forceinline__ void conv_s_pass(const double *__restrict__ sx, const double *__restrict__ sy,
                                            const int *__restrict__ ex, const int *__restrict__ ey, int Drt, int t,
                                            int j0, int j1, int eacc1, int eacc2, double (&Ar)[digits_for(L)],
                                            double (&Ai)[digits_for(L)], double *park_r, double *park_i) {
    constexpr int S = digits_for(L);
    constexpr int NORM = norm_every(S);
    const int D = DT > 0 ? DT : Drt;
    const int D2 = 2 * D;
    md_zero(Ar);
    md_zero(Ai);
    int cnt = 0;
    for (int j = j0; j < j1; j++) {
        const bool first = j <= t;
        if (!first && j > j0 && j - 1 <= t) {  // this lane crosses the fold: park k1
            carry_pass(Ar);
            carry_pass(Ai);
#pragma unroll
            for (int s = 0; s < S; s++) {
                park_r[s] = Ar[s];
                park_i[s] = Ai[s];
                Ar[s] = 0.0;
                Ai[s] = 0.0;
            }
            cnt = 0;
        }
        const int i = first ? j : j - t - 1;
        const int kk = (first ? t : D - 1 - t) - i;
        const int eacc = first ? eacc1 : eacc2;
        double Ur[S], Ui[S];
        const double *ux = sx + i;
#pragma unroll
        for (int s = 0; s < S; s++) {
            Ur[s] = ux[(2 * s) * D];
            Ui[s] = ux[(2 * s + 1) * D];
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
#pragma unroll
                for (int u = 0; u < S - l; u++) {
                    Ar[u + l] = __fma_rn(Ur[u], wc, Ar[u + l]);
                    Ai[u + l] = __fma_rn(Ur[u], wd, Ai[u + l]);
                }
#pragma unroll
                for (int u = 0; u < S - l; u++) {
                    Ar[u + l] = __fma_rn(-Ui[u], wd, Ar[u + l]);
                    Ai[u + l] = __fma_rn(Ui[u], wc, Ai[u + l]);
                }
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
#pragma unroll
                for (int u = 0; u < S - l; u++) {
                    Ar[u + l] = __fma_rn(Ur[u], wc, Ar[u + l]);
                    Ai[u + l] = __fma_rn(Ur[u], wd, Ai[u + l]);
                }
#pragma unroll
                for (int u = 0; u < S - l; u++) {
                    Ar[u + l] = __fma_rn(-Ui[u], wd, Ar[u + l]);
                    Ai[u + l] = __fma_rn(Ui[u], wc, Ai[u + l]);
                }
            }
        }
        if (++cnt == NORM) {
            carry_pass(Ar);
            carry_pass(Ai);
            cnt = 0;
        }
    }
    carry_pass(Ar);
    carry_pass(Ai);
}

// cold epilogue (out of line): one output coefficient, both parts
template <int L>
__device__ __noinline__ void conv_s_output(const double *re, const double *im, const double *park_r,
                                           const double *park_i, int eacc, double *zd, int *ze, double *zl, int D,
                                           int k, double *scratch) {
    constexpr int S = digits_for(L);
#pragma unroll 1
    for (int part = 0; part < 2; part++) {
        const double *acc = part ? im : re;
        const double *pk = part ? park_i : park_r;
        double A[S], Z[S + 2];
#pragma unroll
        for (int s = 0; s < S; s++) A[s] = pk ? __dadd_rn(acc[s], pk[s]) : acc[s];
        acc_to_z(A, Z);
        emit_z<L>(Z, eacc, zd, ze, zl, D, k, part, scratch);
    }
}

template <int L, int DT>
__global__ void __launch_bounds__(DT == 128 || DT == 0 ? 256 : 128, DT == 128 || DT == 0 ? 1 : 2)
    conv_s_kernel(double *__restrict__ dpool, int *__restrict__ epool, double *__restrict__ lpool,
                  const int *__restrict__ jobs, int njobs, int Drt, int T, int F, int P) {
    constexpr int S = digits_for(L);
    constexpr int ZS = S + 2;
    const int D = DT > 0 ? DT : Drt;
    const int SX = 2 * S * D, SY = 2 * (PADZ + S) * D;
    const int threads_per_job = T * F;
    extern __shared__ __align__(16) double sm[];
    double *sdig = sm;                                   // [P][SX + SY]
    double *sgrp = sm + (size_t)P * (SX + SY);           // [P*T + 1][3][ZS]
    int *sexp = (int *)(sgrp + ((size_t)P * T + 1) * 3 * ZS);
    int *shx = sexp + (size_t)P * 4 * D;
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
    const bool real_lane = jl0 < P && r / F < T;
    const bool writer = real_lane && job < njobs;
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
    double *grp = sgrp + (real_lane ? ((size_t)jl * T + t) : (size_t)P * T) * 3 * ZS;
    double *park_r = grp, *park_i = grp + ZS, *scratch2 = grp + 2 * ZS;
    const int k1 = t, k2 = D - 1 - t;
    const bool fin_k2 = j1 > j0 && j1 - 1 > t;

    if (f == 0) {
#pragma unroll
        for (int s = 0; s < S; s++) {
            park_r[s] = 0.0;
            park_i[s] = 0.0;
        }
    }
    __syncwarp();
    double Ar[S], Ai[S];
    conv_s_pass<L, DT>(sx, sy, ex, ey, D, t, j0, j1, ea1, ea2, Ar, Ai, park_r, park_i);
    double Xr[S], Yr[S];
    pair_reduce(Ar, fin_k2, F, Xr, Yr);
    double Xi[S], Yi[S];
    pair_reduce(Ai, fin_k2, F, Xi, Yi);
    __syncwarp();
    if (F == 1) {
        if (writer) {
            // k1 (park added) first: its emit scratch reuses park_r after the sum
            conv_s_output<L>(Xr, Xi, park_r, park_i, ea1, wdig ? zd : nullptr, ze, zl, D, k1, scratch2);
            if (k2 != k1) conv_s_output<L>(Yr, Yi, nullptr, nullptr, ea2, wdig ? zd : nullptr, ze, zl, D, k2, scratch2);
        }
    } else if (f < 2 && writer && (f == 0 || k2 != k1)) {  // one call site: lanes 0 (k1) and 1 (k2)
        if (f == 1) {
#pragma unroll
            for (int s = 0; s < S; s++) {
                Xr[s] = Yr[s];
                Xi[s] = Yi[s];
            }
        }
        conv_s_output<L>(Xr, Xi, f == 0 ? park_r : nullptr, f == 0 ? park_i : nullptr, f == 0 ? ea1 : ea2,
                         wdig ? zd : nullptr, ze, zl, D, f == 0 ? k1 : k2, f == 0 ? park_r + 0 : scratch2);
    }
}

}  // namespace mdps
