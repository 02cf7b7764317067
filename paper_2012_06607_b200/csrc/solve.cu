// solve.cu — block lower-triangular Toeplitz forward substitution on the GPU
// (include/libmdps.h "Block lower-triangular Toeplitz solver"; PAPER.md:266-333,
// §4).
//
//   (A_0 + A_1 t + ... + A_d t^d)(dx_0 + dx_1 t + ...) = b_0 + b_1 t + ...
//   A_0 dx_j = b_j - sum_{i=1..j} A_i dx_{j-i}
//
// Three launches per solve:
//  1. ts_pack_kernel: the Jacobian series [p][q][2][L][D] -> coefficient-major
//     complex md elements Aw[k][p][q][2L] (a group of lanes reading one row p
//     reads consecutive q: coalesced), the right-hand side -> R[k][p][2L].
//  2. ts_lu_kernel (persistent, cooperative): LU with partial pivoting of A_0
//      — per pivot step one block picks the pivot, swaps,
//     inverts it and scales the column, then the whole grid applies the Schur
//     update — followed by W = A_0^-1 from the factors (one block per column:
//     unit-lower forward substitution, diagonal scaling, unit-upper back
//     substitution).
//  3. ts_loop_kernel (persistent, cooperative): for j = 0..d
//       dx_j = W r_j                              (one block per row p)
//       r_k -= A_{k-j} dx_j  for all k > j        (groups of G lanes per (k, p))
//     — the right-looking form of the paper's update ("one job is the update of
//     one right hand side vector after the computation of one update vector",
//     PAPER.md:410-413), so that every launch-free phase exposes (d-j) n
//     independent dot products.
// Arithmetic: complex md numbers with the level-bin accumulators of md.cuh
// (TwoProd/TwoSum EFTs); every dot product is accumulated in
// bins and renormalised once; reductions across lanes are fixed trees, so the
// result is bitwise deterministic.  Grid-wide phases are separated by a
// software grid barrier (all blocks co-resident: cooperative launch).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <string>

#include "../../include/libmdps.h"
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

// 1/a for a real md number a != 0: Newton y <- y + y (1 - a y), each step
// doubling the correct bits from 53 (ceil(log2 L) + 1 steps)
template <int L>
__device__ __forceinline__ void md_recip(const double (&a)[L], double (&y)[L]) {
    constexpr int IT = (L <= 2 ? 2 : (L <= 4 ? 3 : (L <= 8 ? 4 : 5)));
    md_zero(y);
    y[0] = __ddiv_rn(1.0, a[0]);
    double na[L];
#pragma unroll
    for (int l = 0; l < L; l++) na[l] = -a[l];
#pragma unroll 1
    for (int it = 0; it < IT; it++) {
        double B[L + 1], e[L];
        md_zero(B);
        B[0] = 1.0;
        bins_fma<L>(B, na, y);
        md_renorm(B, e);
        double B2[L + 1];
        md_zero(B2);
        bins_add<L>(B2, y);
        bins_fma<L>(B2, y, e);
        md_renorm(B2, y);
    }
}

// 1/(ar + i ai) = (ar - i ai) / (ar^2 + ai^2)
template <int L>
__device__ __forceinline__ void c_recip(const double (&ar)[L], const double (&ai)[L], double (&rr)[L],
                                        double (&ri)[L]) {
    double B[L + 1], den[L], y[L], t[L];
    md_zero(B);
    bins_fma<L>(B, ar, ar);
    bins_fma<L>(B, ai, ai);
    md_renorm(B, den);
    md_recip<L>(den, y);
    md_mul<L>(ar, y, rr);
    md_mul<L>(ai, y, t);
#pragma unroll
    for (int l = 0; l < L; l++) ri[l] = -t[l];
}

// ---- 1. pack --------------------------------------------------------------------
template <int L>
__global__ void __launch_bounds__(THREADS) ts_pack_kernel(const double *__restrict__ J, const double *__restrict__ b,
                                                          double *__restrict__ Aw, double *__restrict__ R, int n,
                                                          int D, int negate) {
    constexpr int E = 2 * L;
    const size_t nj = (size_t)n * n * D, total = nj + (size_t)n * D;
    for (size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (size_t)gridDim.x * blockDim.x) {
        if (g < nj) {
            const int k = (int)(g % D);
            const size_t pq = g / D;
            const size_t p = pq / n, q = pq % n;
            double *dst = Aw + (((size_t)k * n + p) * n + q) * E;
#pragma unroll
            for (int t = 0; t < E; t++) dst[t] = J[(pq * E + t) * D + k];
        } else {
            const size_t g2 = g - nj;
            const int k = (int)(g2 % D);
            const size_t p = g2 / D;
            double *dst = R + ((size_t)k * n + p) * E;
#pragma unroll
            for (int t = 0; t < E; t++) {
                const double v = b[(p * E + t) * D + k];
                dst[t] = negate ? -v : v;
            }
        }
    }
}

// ---- 2. LU of A_0 with partial pivoting, then W = A_0^-1 ----------------------------
template <int L>
__global__ void __launch_bounds__(THREADS) ts_lu_kernel(const double *__restrict__ A0, double *__restrict__ LU,
                                                        double *__restrict__ dinv, int *__restrict__ piv,
                                                        int *__restrict__ status, double *__restrict__ W, int n,
                                                        Barrier *bar) {
    constexpr int E = 2 * L;
    const int nth = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int tx = threadIdx.x;
    __shared__ double s_m[THREADS];
    __shared__ int s_i[THREADS];
    __shared__ int s_pos;
    extern __shared__ double sy[];  // [n][E] one column of W in the making

    for (size_t t = tid; t < (size_t)n * n * E; t += nth) LU[t] = A0[t];
    if (tid == 0) *status = 0;
    grid_sync(bar);

    for (int k = 0; k < n; k++) {
        if (blockIdx.x == 0) {
            // pivot: max |re_0| + |im_0| over rows i >= k, lowest index on ties
            double bm = -1.0;
            int bi = n;
            for (int i = k + tx; i < n; i += blockDim.x) {
                const double *a = LU + ((size_t)i * n + k) * E;
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
                for (int t = tx; t < n * E; t += blockDim.x) {
                    double *rk = LU + (size_t)k * n * E + t, *rp = LU + (size_t)p * n * E + t;
                    const double v = *rk;
                    *rk = *rp;
                    *rp = v;
                }
            __syncthreads();
            double ir[L], ii[L];
            if (sing) {
                md_zero(ir);
                md_zero(ii);
            } else {
                double ar[L], ai[L];
                ld<L>(LU + ((size_t)k * n + k) * E, ar, ai);
                c_recip<L>(ar, ai, ir, ii);
            }
            if (tx == 0) {
                piv[k] = p;
                if (sing) atomicOr(status, 1);
                st<L>(dinv + (size_t)k * E, ir, ii);
            }
            for (int i = k + 1 + tx; i < n; i += blockDim.x) {
                double ar[L], ai[L], lr[L], li[L];
                double *a = LU + ((size_t)i * n + k) * E;
                ld<L>(a, ar, ai);
                cmul<L>(ar, ai, ir, ii, lr, li);
                st<L>(a, lr, li);
            }
        }
        grid_sync(bar);
        const int m = n - k - 1;
        for (int t = tid; t < m * m; t += nth) {
            const int i = k + 1 + t / m, q = k + 1 + t % m;
            double yr[L], yi[L], lr[L], li[L], ur[L], ui[L], zr[L], zi[L];
            double *a = LU + ((size_t)i * n + q) * E;
            ld<L>(a, yr, yi);
            ld<L>(LU + ((size_t)i * n + k) * E, lr, li);
            ld<L>(LU + ((size_t)k * n + q) * E, ur, ui);
            cfms<L>(yr, yi, lr, li, ur, ui, zr, zi);
            st<L>(a, zr, zi);
        }
        grid_sync(bar);
    }

    // unit upper factor: U_iq <- U_ii^-1 U_iq (q > i), so U w = y <=> Uhat w = D^-1 y
    for (int t = tid; t < n * n; t += nth) {
        const int i = t / n, q = t % n;
        if (q > i) {
            double ar[L], ai[L], dr[L], di[L], zr[L], zi[L];
            double *a = LU + (size_t)t * E;
            ld<L>(a, ar, ai);
            ld<L>(dinv + (size_t)i * E, dr, di);
            cmul<L>(dr, di, ar, ai, zr, zi);
            st<L>(a, zr, zi);
        }
    }
    grid_sync(bar);

    // column c of W = A_0^-1 = U^-1 L^-1 P: solve for P e_c
    for (int c = blockIdx.x; c < n; c += gridDim.x) {
        if (tx == 0) {  // where row c of the identity lands after the swaps
            int pos = c;
            for (int k = 0; k < n; k++) {
                const int p = piv[k];
                if (pos == k) pos = p;
                else if (pos == p) pos = k;
            }
            s_pos = pos;
        }
        for (int t = tx; t < n * E; t += blockDim.x) sy[t] = 0.0;
        __syncthreads();
        const int s0 = s_pos;
        if (tx == 0) sy[(size_t)s0 * E] = 1.0;
        __syncthreads();
        for (int q = s0; q < n - 1; q++) {  // unit lower: y_i -= l_iq y_q, i > q
            double xr[L], xi[L];
            ld<L>(sy + (size_t)q * E, xr, xi);
            for (int i = q + 1 + tx; i < n; i += blockDim.x) {
                double yr[L], yi[L], lr[L], li[L], zr[L], zi[L];
                ld<L>(sy + (size_t)i * E, yr, yi);
                ld<L>(LU + ((size_t)i * n + q) * E, lr, li);
                cfms<L>(yr, yi, lr, li, xr, xi, zr, zi);
                st<L>(sy + (size_t)i * E, zr, zi);
            }
            __syncthreads();
        }
        for (int i = tx; i < n; i += blockDim.x) {  // y <- D^-1 y
            double yr[L], yi[L], dr[L], di[L], zr[L], zi[L];
            ld<L>(sy + (size_t)i * E, yr, yi);
            ld<L>(dinv + (size_t)i * E, dr, di);
            cmul<L>(dr, di, yr, yi, zr, zi);
            st<L>(sy + (size_t)i * E, zr, zi);
        }
        __syncthreads();
        for (int q = n - 1; q > 0; q--) {  // unit upper: y_i -= uhat_iq y_q, i < q
            double xr[L], xi[L];
            ld<L>(sy + (size_t)q * E, xr, xi);
            for (int i = tx; i < q; i += blockDim.x) {
                double yr[L], yi[L], ur[L], ui[L], zr[L], zi[L];
                ld<L>(sy + (size_t)i * E, yr, yi);
                ld<L>(LU + ((size_t)i * n + q) * E, ur, ui);
                cfms<L>(yr, yi, ur, ui, xr, xi, zr, zi);
                st<L>(sy + (size_t)i * E, zr, zi);
            }
            __syncthreads();
        }
        for (int t = tx; t < n * E; t += blockDim.x) {
            const int i = t / E, u = t % E;
            W[((size_t)i * n + c) * E + u] = sy[t];
        }
        __syncthreads();
    }
}

// ---- 3. the substitution loop ----------------------------------------------------------
template <int L>
__global__ void __launch_bounds__(THREADS) ts_loop_kernel(const double *__restrict__ Aw, const double *__restrict__ W,
                                                          double *__restrict__ R, double *__restrict__ X,
                                                          double *__restrict__ dx, int n, int D, Barrier *bar) {
    constexpr int E = 2 * L;
    const int nth = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int tx = threadIdx.x, lane = tx & 31, warp = tx >> 5;
    __shared__ double s_red[THREADS / 32][2 * (L + 1)];

    for (int j = 0; j < D; j++) {
        // dx_j = W r_j: one block per row p
        for (int p = blockIdx.x; p < n; p += gridDim.x) {
            double Br[L + 1], Bi[L + 1];
            md_zero(Br);
            md_zero(Bi);
            for (int q = tx; q < n; q += blockDim.x) {
                double ar[L], ai[L], xr[L], xi[L];
                ld<L>(W + ((size_t)p * n + q) * E, ar, ai);
                ld<L>(R + ((size_t)j * n + q) * E, xr, xi);
                cfma<L, false>(Br, Bi, ar, ai, xr, xi);
            }
            group_reduce<L>(Br, Bi, 32);
            if (lane == 0)
#pragma unroll
                for (int t = 0; t <= L; t++) {
                    s_red[warp][t] = Br[t];
                    s_red[warp][L + 1 + t] = Bi[t];
                }
            __syncthreads();
            if (tx == 0) {
                for (int w = 1; w < (int)(blockDim.x >> 5); w++) {
                    double Cr[L + 1], Ci[L + 1];
#pragma unroll
                    for (int t = 0; t <= L; t++) {
                        Cr[t] = s_red[w][t];
                        Ci[t] = s_red[w][L + 1 + t];
                    }
                    bins_merge<L>(Br, Cr);
                    bins_merge<L>(Bi, Ci);
                }
                double zr[L], zi[L];
                md_renorm(Br, zr);
                md_renorm(Bi, zi);
                st<L>(X + ((size_t)j * n + p) * E, zr, zi);
#pragma unroll
                for (int l = 0; l < L; l++) {
                    dx[(((size_t)p * 2 + 0) * L + l) * D + j] = zr[l];
                    dx[(((size_t)p * 2 + 1) * L + l) * D + j] = zi[l];
                }
            }
            __syncthreads();
        }
        grid_sync(bar);
        if (j + 1 == D) break;

        // r_k -= A_{k-j} dx_j for k = j+1..d: groups of G lanes per (k, p)
        const int T = (D - 1 - j) * n;
        int G = 4;
        while (G < 32 && (long long)T * G < nth) G <<= 1;
        const int ng = nth / G, g = tid / G, lg = tid % G;
        for (int base = 0; base < T; base += ng) {
            const int task = base + g;
            const bool valid = task < T;
            const int k = j + 1 + (valid ? task / n : 0), p = valid ? task % n : 0;
            double Br[L + 1], Bi[L + 1];
            md_zero(Br);
            md_zero(Bi);
            if (valid) {
                if (lg == 0) {
                    double yr[L], yi[L];
                    ld<L>(R + ((size_t)k * n + p) * E, yr, yi);
                    cbins_add<L>(Br, Bi, yr, yi);
                }
                const double *Arow = Aw + (((size_t)(k - j) * n + p) * n) * E;
                for (int q = lg; q < n; q += G) {
                    double ar[L], ai[L], xr[L], xi[L];
                    ld<L>(Arow + (size_t)q * E, ar, ai);
                    ld<L>(X + ((size_t)j * n + q) * E, xr, xi);
                    cfma<L, true>(Br, Bi, ar, ai, xr, xi);
                }
            }
            group_reduce<L>(Br, Bi, G);
            if (valid && lg == 0) {
                double zr[L], zi[L];
                md_renorm(Br, zr);
                md_renorm(Bi, zi);
                st<L>(R + ((size_t)k * n + p) * E, zr, zi);
            }
        }
        grid_sync(bar);
    }
}

}  // namespace ts
}  // namespace mdps

using namespace mdps;

struct mdps_solver {
    int n = 0, D = 0, L = 0;
    int device = 0;
    double *Aw = nullptr, *LU = nullptr, *W = nullptr, *R = nullptr, *X = nullptr, *dinv = nullptr;
    int *piv = nullptr, *status = nullptr;
    ts::Barrier *bar = nullptr;
    int grid_lu = 0, grid_loop = 0;
    size_t smem_lu = 0;
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
        int dev = 0, sms = 0, per_lu = 0, per_loop = 0;
        TS_TRY(cudaGetDevice(&dev), MDPS_ECUDA);
        TS_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), MDPS_ECUDA);
        s->smem_lu = (size_t)s->n * 2 * L * sizeof(double);
        if (s->smem_lu > 48 * 1024)
            TS_TRY(cudaFuncSetAttribute(ts::ts_lu_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)s->smem_lu),
                   MDPS_ECUDA);
        TS_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_lu, ts::ts_lu_kernel<L>, ts::THREADS, s->smem_lu),
               MDPS_ECUDA);
        TS_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_loop, ts::ts_loop_kernel<L>, ts::THREADS, 0),
               MDPS_ECUDA);
        if (per_lu < 1 || per_loop < 1) {
            mdps_internal_set_error("solver kernels do not fit on an SM");
            return MDPS_ECUDA;
        }
        s->grid_lu = sms * per_lu;
        s->grid_loop = sms * per_loop;
        return MDPS_OK;
    }
};

template <int L>
struct TsRun {
    static int run(mdps_solver *s, const double *J, const double *b, double *dx, int negate, cudaStream_t st) {
        const int n = s->n, D = s->D;
        const size_t total = (size_t)n * n * D + (size_t)n * D;
        const int pb = (int)std::min<size_t>((total + ts::THREADS - 1) / ts::THREADS, 148 * 16);
        ts::ts_pack_kernel<L><<<pb, ts::THREADS, 0, st>>>(J, b, s->Aw, s->R, n, D, negate);
        TS_TRY(cudaGetLastError(), MDPS_ECUDA);
        TS_TRY(cudaMemsetAsync(s->bar, 0, sizeof(ts::Barrier), st), MDPS_ECUDA);
        {
            const double *A0 = s->Aw;
            void *args[] = {(void *)&A0, (void *)&s->LU, (void *)&s->dinv, (void *)&s->piv, (void *)&s->status,
                            (void *)&s->W, (void *)&s->n, (void *)&s->bar};
            TS_TRY(cudaLaunchCooperativeKernel((const void *)ts::ts_lu_kernel<L>, dim3(s->grid_lu), dim3(ts::THREADS),
                                               args, s->smem_lu, st),
                   MDPS_ECUDA);
        }
        {
            const double *Aw = s->Aw, *W = s->W;
            void *args[] = {(void *)&Aw, (void *)&W, (void *)&s->R, (void *)&s->X, (void *)&dx,
                            (void *)&s->n, (void *)&s->D, (void *)&s->bar};
            TS_TRY(cudaLaunchCooperativeKernel((const void *)ts::ts_loop_kernel<L>, dim3(s->grid_loop),
                                               dim3(ts::THREADS), args, 0, st),
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
    cudaFree(s->Aw);
    cudaFree(s->LU);
    cudaFree(s->W);
    cudaFree(s->R);
    cudaFree(s->X);
    cudaFree(s->dinv);
    cudaFree(s->piv);
    cudaFree(s->status);
    cudaFree(s->bar);
}

extern "C" mdps_solver *mdps_solver_create(int32_t n, int32_t degree, int32_t limbs) {
    if (n < 1 || n > 512 || degree < 0 || degree > 255 ||
        !(limbs == 2 || limbs == 3 || limbs == 4 || limbs == 5 || limbs == 8 || limbs == 10)) {
        mdps_internal_set_error("mdps_solver_create: need 1 <= n <= 512, 0 <= degree <= 255, limbs in {2,3,4,5,8,10}");
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
    cudaGetDevice(&s->device);
    const size_t E = (size_t)2 * limbs * sizeof(double);
    const size_t nn = (size_t)n * n;
    bool ok = cudaMalloc(&s->Aw, nn * s->D * E) == cudaSuccess && cudaMalloc(&s->LU, nn * E) == cudaSuccess &&
              cudaMalloc(&s->W, nn * E) == cudaSuccess && cudaMalloc(&s->R, (size_t)n * s->D * E) == cudaSuccess &&
              cudaMalloc(&s->X, (size_t)n * s->D * E) == cudaSuccess &&
              cudaMalloc(&s->dinv, (size_t)n * E) == cudaSuccess && cudaMalloc(&s->piv, n * sizeof(int)) == cudaSuccess &&
              cudaMalloc(&s->status, sizeof(int)) == cudaSuccess &&
              cudaMalloc(&s->bar, sizeof(ts::Barrier)) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        solver_free(s);
        delete s;
        mdps_internal_set_error("mdps_solver_create: device allocation failed");
        return nullptr;
    }
    s->bytes = nn * s->D * E + 2 * nn * E + 2 * (size_t)n * s->D * E + (size_t)n * E + n * sizeof(int) + 64;
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

// complex md multiply-adds of one solve: LU (column scaling + Schur updates),
// the inverse (unit-upper scaling, forward and back substitution with the
// worst-case start, diagonal scaling) and the substitution loop
static int64_t solver_cfma(int64_t n, int64_t D) {
    int64_t lu = 0;
    for (int64_t k = 0; k < n; k++) lu += (n - k - 1) * (n - k - 1) + (n - k - 1);
    const int64_t inv = n * (n - 1) / 2 + n * (n * (n - 1) / 2) * 2 + n * n;
    const int64_t loop = D * n * n + n * n * D * (D - 1) / 2;
    return lu + inv + loop;
}

extern "C" int mdps_solver_stats(const mdps_solver *s, mdps_solver_info *out) {
    if (!s || !out) {
        mdps_internal_set_error("mdps_solver_stats: NULL argument");
        return MDPS_EINVAL;
    }
    std::memset(out, 0, sizeof *out);
    out->complex_fma = solver_cfma(s->n, s->D);
    out->fp64_ops = out->complex_fma * 4 * ops_bins_fma(s->L);
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
