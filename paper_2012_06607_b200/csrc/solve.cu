// solve.cu — block lower-triangular Toeplitz forward substitution on the GPU
// (include/libmdps.h "Block lower-triangular Toeplitz solver"; PAPER.md:266-333,
// §4).
//
//   (A_0 + A_1 t + ... + A_d t^d)(dx_0 + dx_1 t + ...) = b_0 + b_1 t + ...
//   A_0 dx_j = b_j - sum_{i=1..j} A_i dx_{j-i}
//
// Three launches per solve:
//  1. ts_pack_kernel: the Jacobian coefficients A_0..A_d -> digit elements
//     Ad[k][p][q] (kernels_dig.cuh representation: [2][S] digits + two radix
//     exponents; a group of lanes reading row p reads consecutive q), the
//     right-hand side -> digit planes R[k][2][S][n] (r_k starts as b_k).
//  2. ts_gj_kernel (one block): A_0 is factored once — Gauss-Jordan with
//     partial pivoting on [A_0 | I] in complex double on the leading limbs
//     (the pivots of the paper's LU with partial pivoting, PAPER.md:260-262,
//     GV83 §3.4) — giving W_0 ~ A_0^-1 to double precision.
//  3. ts_main_kernel (persistent, cooperative):
//     a. Newton-Schulz refinement W <- W + W (I - A_0 W) until
//        ||I - A_0 W||^2 is below the md precision (each step squares it):
//        two n-by-n matrix products per step, every entry an exact digit dot
//        product — throughput work instead of 3n latency-bound md steps;
//     b. for j = 0..d
//          dx_j = W r_j                              (G lanes per row p)
//          r_k -= A_{k-j} dx_j  for all k > j        (G lanes per (k, p))
//        — the right-looking form of the paper's update ("one job is the
//        update of one right hand side vector after the computation of one
//        update vector"), so that every phase exposes
//        (d-j) n independent dot products.
// Every dot product (with its initial value: r_k, W_pc or the identity) is
// accumulated EXACTLY on digit planes as in the product kernel — one DFMA per
// digit pair — and rounded once (to S digits for r_k, W, dx_j in digits, to L
// limbs for dx_out).  Reductions across lanes are fixed trees (bitwise
// deterministic).  Grid-wide phases are separated by a software grid barrier
// (the cooperative launch keeps all blocks co-resident).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <new>
#include <string>

#include <cooperative_groups.h>

#include "../../include/libmdps.h"
#include "conv_dig.cuh"

void mdps_internal_set_error(const std::string &s);  // libmdps.cu
int mdps_internal_system_shape(const mdps_system *s, int *N, int *n, int *D, int *L);

namespace mdps {

// normalise one digit vector entry of the solver (planes [part][S][stride],
// exponents [part][stride], its own grid per part) and store it: two carry
// passes balance the partial sums, then the leading-zero shift
template <int L>
__device__ __forceinline__ void ts_emit(double (&A)[digits_for(L)], int eacc, double *zd, int *ze, int stride,
                                        int part, double *scratch) {
    constexpr int S = digits_for(L);
    carry_pass(A);
    carry_pass(A);
    const int z0 = conv_dig_z<S>(A, scratch);
    const int e = (z0 >= S + 2 || eacc <= ZERO_E / 2) ? ZERO_E : eacc + 1 - z0;
    const double *src = scratch + z0;
    const int avail = S + 2 - z0;
#pragma unroll
    for (int s = 0; s < S; s++) zd[(size_t)(part * S + s) * stride] = (s < avail && e != ZERO_E) ? src[s] : 0.0;
    ze[(size_t)part * stride] = e;
}
namespace ts {

constexpr int GJ_THREADS = 1024;
// persistent solver kernel: 128-thread blocks, 3 per SM (L <= 8); 256-thread
// blocks, 1 per SM at L = 10 (255 registers, two staged vectors of 61 KB)
__host__ __device__ constexpr int main_threads(int L) { return L == 10 ? 256 : 128; }
constexpr int MAX_REFINE = 8;

struct Ctl {              // device control block (memset to 0 before every solve)
    unsigned int count;   // grid barrier
    unsigned int gen;
    int emax;             // max radix exponent of the entries of E = I - A_0 W (+ bias), 0 = none
    int status;           // bit 0: singular A_0; bit 1: the refinement missed its bound (MDPS_SOLVE_NOT_CONVERGED)
    int refine_steps;     // Newton-Schulz steps run
    int ntrace;           // entries of the phase trace written
    unsigned int rdy;     // substitution loop: right-hand-side entries final (cumulative)
    int pad[1];
};
constexpr int TRACE_MAX = 1024;

__device__ __forceinline__ long long global_ns() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
constexpr int EMAX_BIAS = 1 << 20;

__device__ __forceinline__ bool tid0() { return blockIdx.x == 0 && threadIdx.x == 0; }

// generation barrier over all blocks of a co-resident grid; block 0 stamps
// the completion time of every barrier into trace (diagnostics)
__device__ __forceinline__ void grid_sync(Ctl *c, long long *trace) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int *vgen = &c->gen;
        const unsigned int g = *vgen;
        __threadfence();
        if (atomicAdd(&c->count, 1u) == gridDim.x - 1) {
            atomicExch(&c->count, 0u);
            __threadfence();
            atomicAdd(&c->gen, 1u);
        } else {
            while (*vgen == g) __nanosleep(100);
        }
        __threadfence();
        if (blockIdx.x == 0 && c->ntrace < TRACE_MAX) trace[c->ntrace++] = global_ns();
    }
    __syncthreads();
}

// ---- 1. pack ---------------------------------------------------------------------
// A(t) has N rows (equations) and n columns (unknowns), N >= n.  Row p of A_k
// as a digit vector in planes: Ad[k][p][2][S][n] + exponents Ae[k][p][2][n]
// (q fastest, so that the lanes of a group reading consecutive q load
// consecutive addresses); A_0's columns as planes Ac[c][2][S][N] (for the
// refinement); R planes [k][2][S][N] + exponents [k][2][N] (r_k starts as b_k,
// negated for a Newton step).
template <int L>
__global__ void __launch_bounds__(128) ts_pack_kernel(const double *__restrict__ J, const double *__restrict__ b,
                                                      double *__restrict__ Ad, int *__restrict__ Ae,
                                                      double *__restrict__ Ac, int *__restrict__ Ace,
                                                      double *__restrict__ Rp, int *__restrict__ Re, int N, int n,
                                                      int D, int negate) {
    constexpr int S = digits_for(L);
    const size_t nj = (size_t)N * n * D, total = nj + (size_t)N * D;
    for (size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (size_t)gridDim.x * blockDim.x) {
        if (g < nj) {  // (k, p, q): q fastest for coalesced digit-plane writes
            const int q = (int)(g % n);
            const size_t kp = g / n;
            const int p = (int)(kp % N), k = (int)(kp / N);
            const double *src = J + ((size_t)p * n + q) * 2 * L * D + k;
            double *dst = Ad + kp * 2 * S * n + q;
            int *de = Ae + kp * 2 * n + q;
#pragma unroll 1
            for (int part = 0; part < 2; part++) {
                double v[L], d[S];
#pragma unroll
                for (int l = 0; l < L; l++) v[l] = src[(size_t)(part * L + l) * D];
                const int e = limbs_to_digits<L, S>(v, d);
                de[(size_t)part * n] = e;
                if (k == 0) Ace[((size_t)q * 2 + part) * N + p] = e;
#pragma unroll
                for (int t = 0; t < S; t++) {
                    dst[(size_t)(part * S + t) * n] = d[t];
                    if (k == 0) Ac[(((size_t)q * 2 + part) * S + t) * N + p] = d[t];
                }
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
                Re[((size_t)k * 2 + part) * N + p] = limbs_to_digits<L, S>(v, d);
#pragma unroll
                for (int t = 0; t < S; t++) Rp[(((size_t)k * 2 + part) * S + t) * N + p] = d[t];
            }
        }
    }
}

// ---- 2. factor A_0 once: Gauss-Jordan, partial pivoting, complex double -------------
// Square (N = n): [A_0 | I] -> [I | W_0], W_0 ~ A_0^-1.  Least squares (N > n,
// PAPER.md:258-262): [G | I] -> [I | V_0], V_0 ~ G^-1, G = A_0^H A_0 (the
// refinement then makes V = G^-1 exact to md precision and forms A_0^+ =
// V A_0^H).  Leading limbs, one block, M in global memory (L2-resident).
// Pivot k = the row i >= k maximising |re| + |im| (lowest row on ties).  The
// n x n result -> digit planes of its rows [p][2][S][n] and columns [c][2][S][n].
template <int L>
__global__ void __launch_bounds__(GJ_THREADS) ts_gj_kernel(const double *__restrict__ J, double *__restrict__ M,
                                                           int *__restrict__ piv, Ctl *ctl, double *__restrict__ Wr,
                                                           int *__restrict__ Wre, double *__restrict__ Wc,
                                                           int *__restrict__ Wce, int N, int n, int D) {
    constexpr int S = digits_for(L);
    const int tx = threadIdx.x, nt = blockDim.x;
    const int W2 = 2 * n;  // row length of [left | I] in complex entries
    __shared__ double s_m[GJ_THREADS];
    __shared__ int s_i[GJ_THREADS];
    __shared__ double s_p[2];
    double2 *Mc = reinterpret_cast<double2 *>(M);
    auto a0 = [&](int r, int c) {  // leading limbs of A_0[r][c]
        const double *src = J + ((size_t)r * n + c) * 2 * L * D;
        return make_double2(src[0], src[(size_t)L * D]);
    };
    for (int t = tx; t < n * W2; t += nt) {
        const int i = t / W2, c = t - i * W2;
        double2 v;
        if (c >= n) {
            v = make_double2(c - n == i ? 1.0 : 0.0, 0.0);
        } else if (N == n) {
            v = a0(i, c);
        } else {  // G[i][c] = sum_r conj(A_0[r][i]) A_0[r][c]
            double re = 0.0, im = 0.0;
            for (int r = 0; r < N; r++) {
                const double2 x = a0(r, i), y = a0(r, c);
                re = __fma_rn(x.x, y.x, __fma_rn(x.y, y.y, re));
                im = __fma_rn(x.x, y.y, __fma_rn(-x.y, y.x, im));
            }
            v = make_double2(re, im);
        }
        Mc[t] = v;
    }
    __syncthreads();
    bool singular = false;
    for (int k = 0; k < n; k++) {
        double bm = -1.0;
        int bi = n;
        for (int i = k + tx; i < n; i += nt) {
            const double2 a = Mc[(size_t)i * W2 + k];
            const double m = __dadd_rn(fabs(a.x), fabs(a.y));
            if (m > bm) {
                bm = m;
                bi = i;
            }
        }
        s_m[tx] = bm;
        s_i[tx] = bi;
        __syncthreads();
        for (int off = nt >> 1; off > 0; off >>= 1) {
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
        singular |= sing;
        __syncthreads();
        if (p != k)
            for (int c = tx; c < W2; c += nt) {
                const double2 v = Mc[(size_t)k * W2 + c];
                Mc[(size_t)k * W2 + c] = Mc[(size_t)p * W2 + c];
                Mc[(size_t)p * W2 + c] = v;
            }
        if (tx == 0) piv[k] = p;
        __syncthreads();
        if (tx == 0) {  // 1 / pivot
            const double2 a = Mc[(size_t)k * W2 + k];
            const double den = __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y));
            s_p[0] = sing ? 0.0 : __ddiv_rn(a.x, den);
            s_p[1] = sing ? 0.0 : __ddiv_rn(-a.y, den);
        }
        __syncthreads();
        const double ir = s_p[0], ii = s_p[1];
        for (int c = k + tx; c < W2; c += nt) {  // scale row k
            const double2 v = Mc[(size_t)k * W2 + c];
            Mc[(size_t)k * W2 + c] = make_double2(__dsub_rn(__dmul_rn(v.x, ir), __dmul_rn(v.y, ii)),
                                                  __dadd_rn(__dmul_rn(v.x, ii), __dmul_rn(v.y, ir)));
        }
        __syncthreads();
        const int cols = W2 - k - 1;
        for (int t = tx; t < (n - 1) * cols; t += nt) {  // eliminate column k from rows i != k
            int i = t / cols;
            const int c = k + 1 + (t - i * cols);
            if (i >= k) i++;
            const double2 f = Mc[(size_t)i * W2 + k], u = Mc[(size_t)k * W2 + c], v = Mc[(size_t)i * W2 + c];
            Mc[(size_t)i * W2 + c] =
                make_double2(__dsub_rn(v.x, __dsub_rn(__dmul_rn(f.x, u.x), __dmul_rn(f.y, u.y))),
                             __dsub_rn(v.y, __dadd_rn(__dmul_rn(f.x, u.y), __dmul_rn(f.y, u.x))));
        }
        __syncthreads();
    }
    if (tx == 0 && singular) atomicOr(&ctl->status, 1);
    for (int t = tx; t < n * n; t += nt) {  // W_0 (or V_0) -> digits
        const int p = t / n, q = t - p * n;
        const double2 w = Mc[(size_t)p * W2 + n + q];
#pragma unroll 1
        for (int part = 0; part < 2; part++) {
            double v[L], d[S];
#pragma unroll
            for (int l = 0; l < L; l++) v[l] = l == 0 ? (part ? w.y : w.x) : 0.0;
            const int e = limbs_to_digits<L, S>(v, d);
            Wre[((size_t)p * 2 + part) * n + q] = e;
            Wce[((size_t)q * 2 + part) * n + p] = e;
#pragma unroll
            for (int s = 0; s < S; s++) {
                Wr[(((size_t)p * 2 + part) * S + s) * n + q] = d[s];
                Wc[(((size_t)q * 2 + part) * S + s) * n + p] = d[s];
            }
        }
    }
}

// The same Gauss-Jordan on a thread-block cluster: the rows of [left | I] are
// distributed over the C CTAs' shared memory; the pivot candidates, the row
// swap and the pivot row travel through distributed shared memory (DSMEM),
// phases are separated by cluster barriers (hardware, ~0.2 us) instead of
// L2 round trips — n dependent steps at DSMEM latency rather than one SM's
// L2 bandwidth.
constexpr int GJC_THREADS = 512;

__device__ __forceinline__ void gj_argmax_merge(double &bm, int &bi, double m2, int i2) {
    if (m2 > bm || (m2 == bm && i2 < bi)) {
        bm = m2;
        bi = i2;
    }
}

template <int L>
__global__ void __launch_bounds__(GJC_THREADS) ts_gj_cluster_kernel(const double *__restrict__ J,
                                                                    int *__restrict__ piv, Ctl *ctl,
                                                                    double *__restrict__ Wr, int *__restrict__ Wre,
                                                                    double *__restrict__ Wc, int *__restrict__ Wce,
                                                                    int N, int n, int D, int rows_per) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    constexpr int S = digits_for(L);
    const int rank = (int)cluster.block_rank();
    const int tx = threadIdx.x, nt = blockDim.x, lane = tx & 31, warp = tx >> 5;
    const int W2 = 2 * n;
    extern __shared__ __align__(16) double smraw[];
    double2 *Mloc = reinterpret_cast<double2 *>(smraw);    // [rows_per][W2]
    double2 *rowk = Mloc + (size_t)rows_per * W2;           // [W2] swap / pivot-row buffer
    double *slot_m = reinterpret_cast<double *>(rowk + W2);  // this CTA's pivot candidate
    int *slot_i = reinterpret_cast<int *>(slot_m + 1);
    __shared__ double s_m[32];
    __shared__ int s_i[32];
    __shared__ int s_p;
    __shared__ double s_inv[2];
    const int r0 = rank * rows_per, r1 = min(n, r0 + rows_per);
    auto a0 = [&](int r, int c) {
        const double *src = J + ((size_t)r * n + c) * 2 * L * D;
        return make_double2(src[0], src[(size_t)L * D]);
    };
    for (int t = tx; t < (r1 - r0) * W2; t += nt) {
        const int i = r0 + t / W2, c = t % W2;
        double2 v;
        if (c >= n) {
            v = make_double2(c - n == i ? 1.0 : 0.0, 0.0);
        } else if (N == n) {
            v = a0(i, c);
        } else {
            double re = 0.0, im = 0.0;
            for (int r = 0; r < N; r++) {
                const double2 x = a0(r, i), y = a0(r, c);
                re = __fma_rn(x.x, y.x, __fma_rn(x.y, y.y, re));
                im = __fma_rn(x.x, y.y, __fma_rn(-x.y, y.x, im));
            }
            v = make_double2(re, im);
        }
        Mloc[t] = v;
    }
    bool singular = false;
    cluster.sync();
    for (int k = 0; k < n; k++) {
        double bm = -1.0;
        int bi = n;
        for (int i = max(k, r0) + tx; i < r1; i += nt) {
            const double2 a = Mloc[(size_t)(i - r0) * W2 + k];
            gj_argmax_merge(bm, bi, __dadd_rn(fabs(a.x), fabs(a.y)), i);
        }
        for (int off = 16; off > 0; off >>= 1)
            gj_argmax_merge(bm, bi, __shfl_xor_sync(0xffffffffu, bm, off), __shfl_xor_sync(0xffffffffu, bi, off));
        if (lane == 0) {
            s_m[warp] = bm;
            s_i[warp] = bi;
        }
        __syncthreads();
        if (tx == 0) {
            for (int w = 1; w < nt / 32; w++) gj_argmax_merge(bm, bi, s_m[w], s_i[w]);
            *slot_m = bm;
            *slot_i = bi;
        }
        cluster.sync();
        if (tx == 0) {  // every CTA merges all candidates the same way
            double m = -1.0;
            int p = n;
            for (int r = 0; r < (int)cluster.num_blocks(); r++)
                gj_argmax_merge(m, p, *cluster.map_shared_rank(slot_m, r), *cluster.map_shared_rank(slot_i, r));
            const bool sing = !(m > 0.0) || p >= n;
            s_p = sing ? -1 - k : p;
        }
        __syncthreads();
        const bool sing = s_p < 0;
        const int p = sing ? k : s_p;
        singular |= sing;
        const int ok = k / rows_per, op = p / rows_per;
        if (p != k) {  // swap rows k and p (through the owners' shared memory)
            if (ok == op) {
                if (rank == ok)
                    for (int c = tx; c < W2; c += nt) {
                        const double2 v = Mloc[(size_t)(k - r0) * W2 + c];
                        Mloc[(size_t)(k - r0) * W2 + c] = Mloc[(size_t)(p - r0) * W2 + c];
                        Mloc[(size_t)(p - r0) * W2 + c] = v;
                    }
                cluster.sync();
            } else {
                if (rank == ok) {
                    const double2 *src = cluster.map_shared_rank(Mloc, op) + (size_t)(p - op * rows_per) * W2;
                    for (int c = tx; c < W2; c += nt) rowk[c] = src[c];
                } else if (rank == op) {
                    const double2 *src = cluster.map_shared_rank(Mloc, ok) + (size_t)(k - ok * rows_per) * W2;
                    for (int c = tx; c < W2; c += nt) rowk[c] = src[c];
                }
                cluster.sync();
                if (rank == ok)
                    for (int c = tx; c < W2; c += nt) Mloc[(size_t)(k - r0) * W2 + c] = rowk[c];
                else if (rank == op)
                    for (int c = tx; c < W2; c += nt) Mloc[(size_t)(p - r0) * W2 + c] = rowk[c];
                cluster.sync();
            }
        }
        if (rank == ok) {  // invert the pivot, scale row k
            if (tx == 0) {
                const double2 a = Mloc[(size_t)(k - r0) * W2 + k];
                const double den = __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y));
                s_inv[0] = sing ? 0.0 : __ddiv_rn(a.x, den);
                s_inv[1] = sing ? 0.0 : __ddiv_rn(-a.y, den);
                piv[k] = p;
            }
            __syncthreads();
            const double ir = s_inv[0], ii = s_inv[1];
            for (int c = k + tx; c < W2; c += nt) {
                const double2 v = Mloc[(size_t)(k - r0) * W2 + c];
                Mloc[(size_t)(k - r0) * W2 + c] = make_double2(__dsub_rn(__dmul_rn(v.x, ir), __dmul_rn(v.y, ii)),
                                                               __dadd_rn(__dmul_rn(v.x, ii), __dmul_rn(v.y, ir)));
            }
        }
        cluster.sync();
        {  // the scaled pivot row into every CTA
            const double2 *src = cluster.map_shared_rank(Mloc, ok) + (size_t)(k - ok * rows_per) * W2;
            for (int c = k + tx; c < W2; c += nt) rowk[c] = src[c];
        }
        __syncthreads();
        const int cols = W2 - k - 1;
        for (int t = tx; t < (r1 - r0) * cols; t += nt) {  // eliminate column k from the local rows i != k
            const int li = t / cols, i = r0 + li;
            if (i == k) continue;
            const int c = k + 1 + (t - li * cols);
            const double2 f = Mloc[(size_t)li * W2 + k], u = rowk[c], v = Mloc[(size_t)li * W2 + c];
            Mloc[(size_t)li * W2 + c] =
                make_double2(__dsub_rn(v.x, __dsub_rn(__dmul_rn(f.x, u.x), __dmul_rn(f.y, u.y))),
                             __dsub_rn(v.y, __dadd_rn(__dmul_rn(f.x, u.y), __dmul_rn(f.y, u.x))));
        }
        cluster.sync();  // row k read by everyone before its owner changes it again
    }
    if (tx == 0 && rank == 0 && singular) atomicOr(&ctl->status, 1);
    for (int t = tx; t < (r1 - r0) * n; t += nt) {  // the local rows of W_0 (or V_0) -> digits
        const int p = r0 + t / n, q = t % n;
        const double2 w = Mloc[(size_t)(p - r0) * W2 + n + q];
#pragma unroll 1
        for (int part = 0; part < 2; part++) {
            double v[L], d[S];
#pragma unroll
            for (int l = 0; l < L; l++) v[l] = l == 0 ? (part ? w.y : w.x) : 0.0;
            const int e = limbs_to_digits<L, S>(v, d);
            Wre[((size_t)p * 2 + part) * n + q] = e;
            Wce[((size_t)q * 2 + part) * n + p] = e;
#pragma unroll
            for (int sd = 0; sd < S; sd++) {
                Wr[(((size_t)p * 2 + part) * S + sd) * n + q] = d[sd];
                Wc[(((size_t)q * 2 + part) * S + sd) * n + p] = d[sd];
            }
        }
    }
}

// ---- 3. exact digit dot products -------------------------------------------------------
// sum_q a_q x_q of complex md numbers: a (row p of a matrix) a digit vector
// in planes [2][S][n] read from global memory, x a digit vector staged in shared
// memory as planes [part][PADZ + S][n] (PADZ zero planes for the alignment
// shift).  One real part per pass, one DFMA per digit pair.
template <int L, int SE = digits_for(L)>
__device__ __forceinline__ void ts_dot_pass(const double *__restrict__ arow, const int *__restrict__ aexp,
                                            const double *__restrict__ xs, const int *__restrict__ xe, int n,
                                            int q0, int G, int part, int eacc, double (&A)[digits_for(L)],
                                            bool zero = true) {
    // SE <= S: the digit triangle is truncated at SE (only digit pairs with
    // u + l < SE are formed) — products needed to fewer bits than the md
    // precision (the early Newton-Schulz steps); the accumulator stays S wide
    constexpr int S = digits_for(L);
    constexpr int NORM = norm_every(S);
    constexpr int P2 = PADZ + S;
    // part 0 (re): ar xr - ai xi ; part 1 (im): ar xi + ai xr
    const int w1part = part, w2part = 1 - part;
    const long long sgn = part == 0 ? (long long)0x8000000000000000ULL : 0LL;
    if (zero) md_zero(A);
    int cnt = 0;
    for (int q = q0; q < n; q += G) {
        const double *a = arow + q;
        double Ur[SE], Ui[SE];
#pragma unroll
        for (int s = 0; s < SE; s++) {
            Ur[s] = a[(size_t)s * n];
            Ui[s] = __longlong_as_double(__double_as_longlong(a[(size_t)(S + s) * n]) ^ sgn);
        }
        const int er = aexp[q], ei = aexp[n + q];
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
            for (int l = 0; l < SE; l++) {
                double w1n = 0.0, w2n = 0.0;
                if (l + 1 < SE) {
                    w1n = V1[(size_t)(l + 1) * n];
                    w2n = V2[(size_t)(l + 1) * n];
                }
#pragma unroll
                for (int u = 0; u < SE - l; u++) {
                    A[u + l] = __fma_rn(Ur[u], w1, A[u + l]);
                    A[u + l] = __fma_rn(Ui[u], w2, A[u + l]);
                }
                w1 = w1n;
                w2 = w2n;
            }
        } else {
#pragma unroll
            for (int l = 0; l < SE; l++) {
                const double w1 = (l >= d1) ? W1[(size_t)(PADZ + l - d1) * n] : 0.0;
                const double w2 = (l >= d2) ? W2[(size_t)(PADZ + l - d2) * n] : 0.0;
#pragma unroll
                for (int u = 0; u < SE - l; u++) {
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

// stage a digit vector given as planes [2][S][n] (+ exponents [2][n]) into
// shared planes [2][PADZ + S][n], optionally negated
template <int L>
// mode: 0 as is, 1 negated, 2 conjugated (imaginary part negated)
__device__ __forceinline__ void ts_stage(const double *__restrict__ src, const int *__restrict__ srce, int n,
                                         int mode, double *xs, int *xe) {
    constexpr int S = digits_for(L);
    constexpr int P2 = PADZ + S;
    const int SN = S * n;
#pragma unroll
    for (int part = 0; part < 2; part++) {
        double *dst = xs + ((size_t)part * P2 + PADZ) * n;
        const double *s0 = src + (size_t)part * SN;
        const bool neg = mode == 1 || (mode == 2 && part == 1);
#pragma unroll 4
        for (int t = threadIdx.x; t < SN; t += blockDim.x) {
            const double v = __ldcg(s0 + t);
            dst[t] = neg ? -v : v;
        }
        double *z = xs + (size_t)part * P2 * n;
        for (int t = threadIdx.x; t < PADZ * n; t += blockDim.x) z[t] = 0.0;
    }
    for (int t = threadIdx.x; t < 2 * n; t += blockDim.x) xe[t] = srce[t];
}

// A digit vector element in planes: digit s of part at d[(part*S + s)*stride],
// its exponent at e[part*stride].
struct DigRef {
    const double *d;
    const int *e;
    int stride;
};
struct DigOut {
    double *d;
    int *e;
    int stride;
};

// One task: out = init + sum_q arow[q] x_q over the G lanes of a group (G a
// power of two; groups aligned in the warp).  init: a digit value (init.d) or
// the identity (one: +1 to the real part) or nothing.  The result is written
// as digits (out) and optionally as L limbs at zl[(part*L + l)*lstride].
// Returns the larger output part exponent.  All lanes of the warp call it
// (shuffles); `valid` masks the work and the output.
// A dot-product segment: row `a` (digit planes [2][S][n], exponents [2][n])
// times the staged vector (xs, xe).
struct Seg {
    const double *a;
    const int *ae;
    const double *xs;
    const int *xe;
};

// pbeg, pend: the output parts this group computes — both (0, 2), or one
// when the task is split over two groups, one per part (the latency-bound
// substitution loop: the dependent task takes one pass instead of two).
template <int L, int SE = digits_for(L)>
__device__ __forceinline__ int ts_task(const double *__restrict__ arow, const int *__restrict__ aexp,
                                       const double *xs, const int *xe, int n, int lg, int G, bool valid,
                                       DigRef init, bool one, DigOut out, double *zl, int lstride,
                                       double *scratch, Seg seg2 = Seg{nullptr, nullptr, nullptr, nullptr},
                                       int pbeg = 0, int pend = 2) {
    constexpr int S = digits_for(L);
    int ea0 = ZERO_E, ea1 = ZERO_E;
    if (valid) {
        for (int q = lg; q < n; q += G) {
            const int er = aexp[q], ei = aexp[n + q], xr = xe[q], xi = xe[n + q];
            ea0 = max(ea0, max(er + xr, ei + xi));
            ea1 = max(ea1, max(er + xi, ei + xr));
        }
        if (seg2.a)
            for (int q = lg; q < n; q += G) {
                const int er = seg2.ae[q], ei = seg2.ae[n + q], xr = seg2.xe[q], xi = seg2.xe[n + q];
                ea0 = max(ea0, max(er + xr, ei + xi));
                ea1 = max(ea1, max(er + xi, ei + xr));
            }
        if (lg == 0) {
            if (init.d) {
                ea0 = max(ea0, init.e[0] + 1);
                ea1 = max(ea1, init.e[init.stride] + 1);
            }
            if (one) ea0 = max(ea0, 2);  // 1 = digit 0 of exponent 1
        }
    }
    for (int off = G >> 1; off > 0; off >>= 1) {  // xor partners stay inside the aligned group
        ea0 = max(ea0, __shfl_xor_sync(0xffffffffu, ea0, off));
        ea1 = max(ea1, __shfl_xor_sync(0xffffffffu, ea1, off));
    }
    int eout = ZERO_E;
#pragma unroll 1
    for (int part = pbeg; part < pend; part++) {
        const int eacc = max(part ? ea1 : ea0, ZERO_E);
        int eI = ZERO_E;
        if (valid && lg == 0 && init.d) {  // fetch the init digits early (they land during the pass)
            eI = init.e[part * init.stride];
            const double *src = init.d + (size_t)part * S * init.stride;
#pragma unroll
            for (int t = 0; t < S; t++) scratch[t] = __ldcg(src + (size_t)t * init.stride);
        }
        double A[S];
        ts_dot_pass<L, SE>(arow, aexp, xs, xe, valid ? n : 0, lg, G, part, eacc, A);
        if (seg2.a) ts_dot_pass<L, SE>(seg2.a, seg2.ae, seg2.xs, seg2.xe, valid ? n : 0, lg, G, part, eacc, A, false);
        if (valid && lg == 0) {
            if (init.d && eI > ZERO_E / 2) {  // digit s of the init value has weight R^(eI-1-s): slot s + eacc-1-eI
                const int dI = eacc - 1 - eI;
#pragma unroll
                for (int t = 0; t < S; t++) {
                    const int s = t - dI;
                    if (s >= 0 && s < S) A[t] = __dadd_rn(A[t], scratch[s]);
                }
            }
            if (one && part == 0) {  // weight R^0 = slot eacc - 2
                const int t0 = eacc - 2;
#pragma unroll
                for (int u = 0; u < S; u++)
                    if (u == t0) A[u] = __dadd_rn(A[u], 1.0);
            }
        }
        for (int off = G >> 1; off > 0; off >>= 1) {
#pragma unroll
            for (int s = 0; s < S; s++) A[s] = __dadd_rn(A[s], __shfl_xor_sync(0xffffffffu, A[s], off));
        }
        if (valid && lg == 0) {
            ts_emit<L>(A, eacc, out.d, out.e, out.stride, part, scratch);
            eout = max(eout, out.e[part * out.stride]);
            if (zl) {  // A is carry-normalised by the emit
                double o[L];
                digits_to_limbs<L, S, true>(A, eacc - 1, o);
#pragma unroll
                for (int l = 0; l < L; l++) zl[(size_t)(part * L + l) * lstride] = o[l];
            }
        }
    }
    return eout;
}

template <int V>
struct IC {
    static constexpr int value = V;
};
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }

// lanes per task: as many as keep >= 4 terms per lane (G <= 32): the lanes of
// a group read consecutive q of one row, so wide groups make every digit-plane
// load one contiguous run (the loads, not the DFMAs, bound narrow groups)
__device__ __forceinline__ int pick_group(long long tasks, int n, long long avail) {
    (void)tasks;
    (void)avail;
    int G = 4;
    while (G < 32 && n >= 8 * G) G <<= 1;
    return G;
}

// Matrix-product phases: task (column c, row p) with the column staged once
// per block; blocks are split into `bpc` blocks per column, each taking a
// chunk of the rows.
struct ColSplit {
    int c0, cstep, r0, r1;
};
__device__ __forceinline__ ColSplit col_split(int ncols, int nrows) {
    const int bpc = max(1, (int)gridDim.x / ncols), ncb = (int)gridDim.x / bpc;
    const int cslot = blockIdx.x / bpc, rchunk = blockIdx.x % bpc, rpb = (nrows + bpc - 1) / bpc;
    ColSplit cs;
    cs.c0 = cslot < ncb ? cslot : ncols;
    cs.cstep = ncb;
    cs.r0 = rchunk * rpb;
    cs.r1 = min(nrows, cs.r0 + rpb);
    return cs;
}

// Newton-Schulz refinement of W ~ A_0^+, the two-coefficient operator M, then
// the substitution loop.  A(t): N x n (N >= n); W, M: n x N.
template <int L>
__global__ void __launch_bounds__(main_threads(L), L == 10 ? 1 : 3) ts_main_kernel(
    const double *__restrict__ Ad, const int *__restrict__ Ae, const double *__restrict__ Ac,
    const int *__restrict__ Ace, double *__restrict__ Wr, int *__restrict__ Wre, double *Wc, int *Wce,
    double *Wc2, int *Wce2, double *__restrict__ Er, int *__restrict__ Ere, double *__restrict__ Pc,
    int *__restrict__ Pce, double *__restrict__ Mr, int *__restrict__ Mre, double *__restrict__ Rp,
    int *__restrict__ Re, double *__restrict__ Xp, int *__restrict__ Xe, double *__restrict__ dx,
    double *__restrict__ Gc, int *__restrict__ Gce, int N, int n, int D, Ctl *ctl, long long *trace) {
    constexpr int S = digits_for(L);
    constexpr int P2 = PADZ + S;
    if (tid0()) trace[ctl->ntrace++] = global_ns();
    extern __shared__ __align__(16) double sm[];
    double *xs = sm;                              // [2][P2][N]  staged vector 0
    double *xs1 = sm + (size_t)2 * P2 * N;        // [2][P2][N]  staged vector 1
    int *xe = (int *)(xs1 + (size_t)2 * P2 * N);  // [2][N]
    int *xe1 = xe + 2 * N;                        // [2][N]
    double *scr = (double *)(xe1 + 2 * N + 2);    // [blockDim/4][S+2] emit scratch (one per group leader)
    __shared__ int s_emax;
    const int nth = gridDim.x * blockDim.x;
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const size_t VN = (size_t)2 * S * n, VM = (size_t)2 * S * N;  // doubles per digit vector of length n / N
    double *scratch = scr + (size_t)(threadIdx.x / 4) * (S + 2);
    const DigRef none{nullptr, nullptr, 0};

    // a0. least squares (N > n): G = A_0^H A_0 (n x n, exact dot products): the
    //     task for staged conj(A_0[:, c]) and row p computes sum_r A_0[r][p]
    //     conj(A_0[r][c]) = G[c][p] (G is Hermitian), written to column p.
    const bool lsq = N > n;
    if (lsq) {
        const ColSplit cs = col_split(n, n);
        const int G = pick_group(cs.r1 - cs.r0, N, blockDim.x);
        const int gpb = blockDim.x / G, g = threadIdx.x / G, lg = threadIdx.x % G;
        for (int c = cs.c0; c < n; c += cs.cstep) {
            ts_stage<L>(Ac + (size_t)c * VM, Ace + (size_t)c * 2 * N, N, 2, xs, xe);
            __syncthreads();
            for (int base = cs.r0; base < cs.r1; base += gpb) {
                const int p = base + g;
                const bool valid = p < cs.r1;
                const int pp = valid ? p : 0;
                ts_task<L>(Ac + (size_t)pp * VM, Ace + (size_t)pp * 2 * N, xs, xe, N, lg, G, valid, none, false,
                           DigOut{Gc + (size_t)pp * VN + c, Gce + (size_t)pp * 2 * n + c, n}, nullptr, 0, scratch);
            }
            __syncthreads();
        }
        grid_sync(ctl, trace);
    }
    // a. W <- W + (I - W A) W, the left Newton-Schulz step: W -> A_0^-1 (N = n)
    //    or V -> G^-1 (N > n, A = G); E = I - W A (n x n, row planes), W' = W + E W.
    const int RL = lsq ? n : N;                    // length of W's rows / A's columns here
    const double *RA = lsq ? Gc : Ac;
    const int *RAe = lsq ? Gce : Ace;
    const size_t VR = (size_t)2 * S * RL;
    for (int it = 0; it < MAX_REFINE; it++) {
        // digits kept in this step's products: step it squares an error of
        // ~2^-(48 * 2^it) (double-precision start), so its products need about
        // 2 * 48 * 2^it + 40 bits below the largest term: 8, 13, 21 digits, then S
        const int se_level = it < 3 ? it : 3;
        if (threadIdx.x == 0) s_emax = ZERO_E;
        {
            const ColSplit cs = col_split(n, n);
            const int G = pick_group(cs.r1 - cs.r0, RL, blockDim.x);
            const int gpb = blockDim.x / G, g = threadIdx.x / G, lg = threadIdx.x % G;
            for (int c = cs.c0; c < n; c += cs.cstep) {  // E[:, c] = e_c - W A[:, c]
                ts_stage<L>(RA + (size_t)c * VR, RAe + (size_t)c * 2 * RL, RL, 1, xs, xe);
                __syncthreads();
                for (int base = cs.r0; base < cs.r1; base += gpb) {
                    const int p = base + g;
                    const bool valid = p < cs.r1;
                    const int pp = valid ? p : 0;
                    auto task = [&](auto se) {
                        return ts_task<L, decltype(se)::value>(
                            Wr + (size_t)pp * VR, Wre + (size_t)pp * 2 * RL, xs, xe, RL, lg, G, valid, none, pp == c,
                            DigOut{Er + (size_t)pp * VN + c, Ere + (size_t)pp * 2 * n + c, n}, nullptr, 0, scratch);
                    };
                    const int e = se_level == 0 ? task(IC<cmin(8, S)>{})
                                : se_level == 1 ? task(IC<cmin(13, S)>{})
                                : se_level == 2 ? task(IC<cmin(21, S)>{}) : task(IC<S>{});
                    if (valid && lg == 0) atomicMax(&s_emax, e);
                }
                __syncthreads();
            }
        }
        if (threadIdx.x == 0 && s_emax > ZERO_E / 2) atomicMax(&ctl->emax, s_emax + EMAX_BIAS);
        grid_sync(ctl, trace);
        // ||E|| < R^emax / 2; the step leaves an error ~||E||^2: stop once that
        // is below 2^-(53 L + 16)
        const int eraw = *(volatile int *)&ctl->emax;
        const bool conv = eraw == 0 || 2 * (BETA * (eraw - EMAX_BIAS) - 1) < -(53 * L + 16);
        const bool last = conv || it + 1 == MAX_REFINE;
        // MAX_REFINE steps without reaching the bound: ||I - W A_0|| was not
        // < 1 at the double-precision seed (A_0 too ill-conditioned for the
        // double Gauss-Jordan, kappa >~ 1e16): reported, dx unspecified
        if (!conv && last && blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&ctl->status, 2);
        {
            const ColSplit cs = col_split(RL, n);
            const int G = pick_group(cs.r1 - cs.r0, n, blockDim.x);
            const int gpb = blockDim.x / G, g = threadIdx.x / G, lg = threadIdx.x % G;
            for (int c = cs.c0; c < RL; c += cs.cstep) {  // W'[:, c] = W[:, c] + E W[:, c]
                ts_stage<L>(Wc + (size_t)c * VN, Wce + (size_t)c * 2 * n, n, 0, xs, xe);
                __syncthreads();
                for (int base = cs.r0; base < cs.r1; base += gpb) {
                    const int p = base + g;
                    const bool valid = p < cs.r1;
                    const int pp = valid ? p : 0;
                    auto task = [&](auto se) {
                        ts_task<L, decltype(se)::value>(
                            Er + (size_t)pp * VN, Ere + (size_t)pp * 2 * n, xs, xe, n, lg, G, valid,
                            DigRef{Wc + (size_t)c * VN + pp, Wce + (size_t)c * 2 * n + pp, n}, false,
                            DigOut{Wc2 + (size_t)c * VN + pp, Wce2 + (size_t)c * 2 * n + pp, n}, nullptr, 0, scratch);
                    };
                    if (se_level == 0) task(IC<cmin(8, S)>{});
                    else if (se_level == 1) task(IC<cmin(13, S)>{});
                    else if (se_level == 2) task(IC<cmin(21, S)>{});
                    else task(IC<S>{});
                }
                __syncthreads();
            }
        }
        grid_sync(ctl, trace);
        {  // W' becomes W (column planes); row planes from it
            double *t = Wc;
            Wc = Wc2;
            Wc2 = t;
            int *te = Wce;
            Wce = Wce2;
            Wce2 = te;
        }
        for (size_t t = tid; t < (size_t)n * RL; t += nth) {
            const int pr = (int)(t / RL), c = (int)(t % RL);
#pragma unroll
            for (int part = 0; part < 2; part++) {
                Wre[((size_t)pr * 2 + part) * RL + c] = Wce[((size_t)c * 2 + part) * n + pr];
#pragma unroll
                for (int sd = 0; sd < S; sd++)
                    Wr[(size_t)pr * VR + (size_t)(part * S + sd) * RL + c] =
                        Wc[(size_t)c * VN + (size_t)(part * S + sd) * n + pr];
            }
        }
        if (tid == 0) {
            ctl->emax = 0;
            ctl->refine_steps = it + 1;
        }
        grid_sync(ctl, trace);
        if (last) break;
    }
    // a2. least squares: W = V A_0^H (n x N): column c of W is V conj(A_0[c, :])^T
    if (lsq) {
        {
            const ColSplit cs = col_split(N, n);
            const int G = pick_group(cs.r1 - cs.r0, n, blockDim.x);
            const int gpb = blockDim.x / G, g = threadIdx.x / G, lg = threadIdx.x % G;
            for (int c = cs.c0; c < N; c += cs.cstep) {
                ts_stage<L>(Ad + (size_t)c * VN, Ae + (size_t)c * 2 * n, n, 2, xs, xe);  // row c of A_0
                __syncthreads();
                for (int base = cs.r0; base < cs.r1; base += gpb) {
                    const int p = base + g;
                    const bool valid = p < cs.r1;
                    const int pp = valid ? p : 0;
                    ts_task<L>(Wr + (size_t)pp * VN, Wre + (size_t)pp * 2 * n, xs, xe, n, lg, G, valid, none, false,
                               DigOut{Wc2 + (size_t)c * VN + pp, Wce2 + (size_t)c * 2 * n + pp, n}, nullptr, 0,
                               scratch);
                }
                __syncthreads();
            }
        }
        grid_sync(ctl, trace);
        {
            double *t = Wc;
            Wc = Wc2;
            Wc2 = t;
            int *te = Wce;
            Wce = Wce2;
            Wce2 = te;
        }
        for (size_t t = tid; t < (size_t)n * N; t += nth) {  // row planes (length N) <- columns
            const int pr = (int)(t / N), c = (int)(t % N);
#pragma unroll
            for (int part = 0; part < 2; part++) {
                Wre[((size_t)pr * 2 + part) * N + c] = Wce[((size_t)c * 2 + part) * n + pr];
#pragma unroll
                for (int sd = 0; sd < S; sd++)
                    Wr[(size_t)pr * VM + (size_t)(part * S + sd) * N + c] =
                        Wc[(size_t)c * VN + (size_t)(part * S + sd) * n + pr];
            }
        }
        grid_sync(ctl, trace);
    }

    // b. M = -W A_1 W (n x N, row planes in Mr): with it two coefficients per step,
    //      dx_j     = W r_j
    //      dx_{j+1} = W r'_{j+1} + M r_j,   r'_{j+1} = r_{j+1} before A_1 dx_j
    //    (r_{j+1} = r'_{j+1} - A_1 dx_j and dx_j = W r_j): half the dependent steps.
    if (D >= 2) {
        {
            const ColSplit cs = col_split(N, N);
            const int G = pick_group(cs.r1 - cs.r0, n, blockDim.x);
            const int gpb = blockDim.x / G, g = threadIdx.x / G, lg = threadIdx.x % G;
            for (int c = cs.c0; c < N; c += cs.cstep) {  // P[:, c] = A_1 W[:, c]  (N x N)
                ts_stage<L>(Wc + (size_t)c * VN, Wce + (size_t)c * 2 * n, n, 0, xs, xe);
                __syncthreads();
                for (int base = cs.r0; base < cs.r1; base += gpb) {
                    const int p = base + g;
                    const bool valid = p < cs.r1;
                    const int pp = valid ? p : 0;
                    const size_t row = (size_t)N + pp;  // row p of A_1
                    ts_task<L>(Ad + row * VN, Ae + row * 2 * n, xs, xe, n, lg, G, valid, none, false,
                               DigOut{Pc + (size_t)c * VM + pp, Pce + (size_t)c * 2 * N + pp, N}, nullptr, 0, scratch);
                }
                __syncthreads();
            }
        }
        grid_sync(ctl, trace);
        {
            const ColSplit cs = col_split(N, n);
            const int G = pick_group(cs.r1 - cs.r0, N, blockDim.x);
            const int gpb = blockDim.x / G, g = threadIdx.x / G, lg = threadIdx.x % G;
            for (int c = cs.c0; c < N; c += cs.cstep) {  // M[:, c] = -W P[:, c]  (columns into Wc2)
                ts_stage<L>(Pc + (size_t)c * VM, Pce + (size_t)c * 2 * N, N, 1, xs, xe);
                __syncthreads();
                for (int base = cs.r0; base < cs.r1; base += gpb) {
                    const int p = base + g;
                    const bool valid = p < cs.r1;
                    const int pp = valid ? p : 0;
                    ts_task<L>(Wr + (size_t)pp * VM, Wre + (size_t)pp * 2 * N, xs, xe, N, lg, G, valid, none, false,
                               DigOut{Wc2 + (size_t)c * VN + pp, Wce2 + (size_t)c * 2 * n + pp, n}, nullptr, 0,
                               scratch);
                }
                __syncthreads();
            }
        }
        grid_sync(ctl, trace);
        for (size_t t = tid; t < (size_t)n * N; t += nth) {  // Mr (row planes) <- columns
            const int pr = (int)(t / N), c = (int)(t % N);
#pragma unroll
            for (int part = 0; part < 2; part++) {
                Mre[((size_t)pr * 2 + part) * N + c] = Wce2[((size_t)c * 2 + part) * n + pr];
#pragma unroll
                for (int sd = 0; sd < S; sd++)
                    Mr[(size_t)pr * VM + (size_t)(part * S + sd) * N + c] =
                        Wc2[(size_t)c * VN + (size_t)(part * S + sd) * n + pr];
            }
        }
        grid_sync(ctl, trace);
    }

    // c. the substitution loop, two coefficients per step.  Dataflow overlap:
    //    the update phase for pair j computes r_{j+2}, r_{j+3} first (tasks
    //    0 .. 2N-1, all in the first sweep of its groups, on the first blocks),
    //    each task's writer signals ctl->rdy, and the LAST blocks of the grid,
    //    after their own share of the updates, wait for those 2N signals and
    //    compute dx_{j+2}, dx_{j+3} right there — so the dependent dx step of
    //    the next pair runs under the bulk of the updates and the loop takes one
    //    grid barrier per pair instead of two.  dx vectors are double-buffered
    //    (pair parity): blocks may still stage dx_j while dx_{j+2} is written.
    //    Falls back to a separate dx phase when the grid is too small for the
    //    first-sweep / disjoint-blocks guarantee (no spinning block ever waits
    //    on work assigned to itself or to a block behind it).
    auto xbuf = [&](int j, int which) { return Xp + (size_t)(((j >> 1) & 1) * 2 + which) * VN; };
    auto xebuf = [&](int j, int which) { return Xe + (size_t)(((j >> 1) & 1) * 2 + which) * 2 * n; };
    // dx_j = W r_j ; dx_{j+1} = W r'_{j+1} + M r_j on blocks [b0, gridDim)
    auto dx_phase = [&](int j, int b0) {
        const bool pair = j + 1 < D;
        ts_stage<L>(Rp + (size_t)j * VM, Re + (size_t)j * 2 * N, N, 0, xs, xe);
        if (pair) ts_stage<L>(Rp + (size_t)(j + 1) * VM, Re + (size_t)(j + 1) * 2 * N, N, 0, xs1, xe1);
        __syncthreads();
        const int nthd = ((int)gridDim.x - b0) * blockDim.x;
        const int tidd = ((int)blockIdx.x - b0) * blockDim.x + threadIdx.x;
        const int T = pair ? 2 * n : n;
        const int G = pick_group(T, pair ? 2 * N : N, nthd);
        // one group of G lanes per output part (2G lanes per task)
        const int G2 = 2 * G;
        const int ng = nthd / G2, g = tidd / G2, lg = tidd % G, pt = (tidd % G2) / G;
        double *X0 = xbuf(j, 0), *X1 = xbuf(j, 1);
        int *E0 = xebuf(j, 0), *E1 = xebuf(j, 1);
        for (int base = 0; base < T; base += ng) {
            const int task = base + g;
            const bool valid = task < T;
            const int second = valid && task >= n;
            const int pp = valid ? task - (second ? n : 0) : 0;
            const double *wr = Wr + (size_t)pp * VM;
            const int *wre = Wre + (size_t)pp * 2 * N;
            if (!second)
                ts_task<L>(wr, wre, xs, xe, N, lg, G, valid, none, false, DigOut{X0 + pp, E0 + pp, n},
                           dx + (size_t)pp * 2 * L * D + j, D, scratch, Seg{nullptr, nullptr, nullptr, nullptr},
                           pt, pt + 1);
            else
                ts_task<L>(wr, wre, xs1, xe1, N, lg, G, valid, none, false, DigOut{X1 + pp, E1 + pp, n},
                           dx + (size_t)pp * 2 * L * D + j + 1, D, scratch,
                           Seg{Mr + (size_t)pp * VM, Mre + (size_t)pp * 2 * N, xs, xe}, pt, pt + 1);
        }
    };
    dx_phase(0, 0);
    grid_sync(ctl, trace);
    unsigned int rdy_target = 0;
    for (int j = 0; j + 2 < D; j += 2) {
        // r_k -= A_{k-j} dx_j + A_{k-j-1} dx_{j+1}, k = j+2..d
        const int T = (D - 2 - j) * N;
        const int G = pick_group(T, 2 * n, nth);
        // one group of G lanes per output part once the tasks fit about three
        // sweeps that way (the latency-bound later pairs: the dependent task
        // takes one pass instead of two); both parts per group while the
        // updates are throughput-bound (measured, od: splitting every pair
        // slows the early ones 100 -> 120 us, speeds the late ones 80 -> 58)
        const bool split = (long long)T * 2 * G <= 3LL * nth;
        const int G2 = split ? 2 * G : G;
        const int ng = nth / G2, g = tid / G2, lg = tid % G, pt = split ? (tid % G2) / G : 0;
        const int nnext = j + 3 < D ? 2 * N : N;  // tasks of r_{j+2}, r_{j+3}
        // the dx blocks of the next pair: the last ones, disjoint from the
        // blocks holding the r_{j+2}, r_{j+3} tasks
        const bool pair2 = j + 3 < D;
        const int Tdx = pair2 ? 2 * n : n, lendx = pair2 ? 2 * N : N;
        int nbdx = 0;
        {
            const int Gd = 2 * pick_group(Tdx, lendx, nth);  // upper bound of the subset's group width (2 parts)
            nbdx = (int)(((long long)Tdx * Gd + blockDim.x - 1) / blockDim.x);
        }
        const int rblocks = (int)(((long long)nnext * G2 + blockDim.x - 1) / blockDim.x);
        const bool overlap = ng >= nnext && rblocks + nbdx <= (int)gridDim.x;
        const int b0 = (int)gridDim.x - nbdx;
        ts_stage<L>(xbuf(j, 0), xebuf(j, 0), n, 1, xs, xe);
        ts_stage<L>(xbuf(j, 1), xebuf(j, 1), n, 1, xs1, xe1);
        __syncthreads();
        for (int base = 0; base < T; base += ng) {
            const int task = base + g;
            const bool valid = task < T;
            const int k = j + 2 + (valid ? task / N : 0), p = valid ? task % N : 0;
            const size_t row0 = (size_t)(k - j) * N + p, row1 = (size_t)(k - j - 1) * N + p;
            double *rk = Rp + (size_t)k * VM + p;
            int *rke = Re + (size_t)k * 2 * N + p;
            ts_task<L>(Ad + row0 * VN, Ae + row0 * 2 * n, xs, xe, n, lg, G, valid, DigRef{rk, rke, N}, false,
                       DigOut{rk, rke, N}, nullptr, 0, scratch, Seg{Ad + row1 * VN, Ae + row1 * 2 * n, xs1, xe1},
                       split ? pt : 0, split ? pt + 1 : 2);
            if (overlap && valid && lg == 0 && task < nnext) {  // r_{j+2} / r_{j+3} entry part final
                __threadfence();
                atomicAdd(&ctl->rdy, 1u);
            }
        }
        rdy_target += overlap ? (split ? 2u : 1u) * (unsigned)nnext : 0u;  // one signal per group
        if (overlap && (int)blockIdx.x >= b0) {
            __syncthreads();  // this block's update tasks no longer read xs / xs1
            if (threadIdx.x == 0) {
                volatile unsigned int *vr = &ctl->rdy;
                while (*vr < rdy_target) __nanosleep(64);
                __threadfence();
            }
            __syncthreads();
            dx_phase(j + 2, b0);
        }
        grid_sync(ctl, trace);
        if (!overlap) {
            dx_phase(j + 2, 0);
            grid_sync(ctl, trace);
        }
    }
}

__host__ __device__ inline size_t ts_main_smem(int S, int n, int threads) {
    return (size_t)4 * (PADZ + S) * n * sizeof(double) + (size_t)(4 * n + 2) * sizeof(int) +
           (size_t)(threads / 4) * (S + 2) * sizeof(double);
}

// ---- Newton update: x <- x + dx and ||dx|| ------------------------------------------
// One thread per (component, coefficient); md addition in EFT level bins;
// the update norm max_{q,k} |dx_{q,k}| (complex modulus of the leading
// limbs) is reduced per block and combined with an atomic max on the bit
// pattern (non-negative doubles order like their 64-bit patterns).
template <int L>
__global__ void __launch_bounds__(128) ts_update_kernel(double *__restrict__ x, const double *__restrict__ dx, int n,
                                                        int D, unsigned long long *__restrict__ norm_bits) {
    __shared__ double s_max[4];
    double m = 0.0;
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n * D) {
        const int q = g / D, k = g - q * D;
        double v[2];
#pragma unroll
        for (int part = 0; part < 2; part++) {
            double a[L], b[L], c[L];
            double *xp = x + ((size_t)q * 2 + part) * L * D + k;
            const double *dp = dx + ((size_t)q * 2 + part) * L * D + k;
#pragma unroll
            for (int l = 0; l < L; l++) {
                a[l] = xp[(size_t)l * D];
                b[l] = dp[(size_t)l * D];
            }
            v[part] = b[0];
            md_add<L>(a, b, c);
#pragma unroll
            for (int l = 0; l < L; l++) xp[(size_t)l * D] = c[l];
        }
        m = hypot(v[0], v[1]);
    }
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); w++) m = fmax(m, s_max[w]);
        if (m > 0.0) atomicMax(norm_bits, (unsigned long long)__double_as_longlong(m));
    }
}

}  // namespace ts
}  // namespace mdps

using namespace mdps;

struct mdps_solver {
    int N = 0, n = 0, D = 0, L = 0, S = 0;  // N equations (rows) >= n unknowns
    int device = 0;
    double *Ad = nullptr, *Ac = nullptr, *M = nullptr, *Wr = nullptr, *Wc = nullptr, *Wc2 = nullptr, *Er = nullptr,
           *Pc = nullptr, *Mr = nullptr, *Rp = nullptr, *Xp = nullptr;
    int *Ae = nullptr, *Ace = nullptr, *Wre = nullptr, *Wce = nullptr, *Wce2 = nullptr, *Ere = nullptr,
        *Pce = nullptr, *Mre = nullptr, *Re = nullptr, *Xe = nullptr;
    double *Gc = nullptr;  // least squares: A_0^H A_0, column planes
    int *Gce = nullptr;
    int *piv = nullptr;
    ts::Ctl *ctl = nullptr;
    long long *trace = nullptr;
    double *nv = nullptr, *nj = nullptr, *ndx = nullptr;  // Newton workspace (lazy): f, J, dx
    unsigned long long *nnorm = nullptr;
    int grid_main = 0;
    size_t smem_main = 0;
    int gj_cluster = 0, gj_rows = 0;  // cluster Gauss-Jordan: CTAs, rows per CTA (0: single-block kernel)
    size_t gj_smem = 0;
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
        int dev = 0, sms = 0, per = 0;
        TS_TRY(cudaGetDevice(&dev), MDPS_ECUDA);
        TS_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), MDPS_ECUDA);
        s->smem_main = ts::ts_main_smem(digits_for(L), s->N, ts::main_threads(L));
        if (s->smem_main > 227 * 1024) {
            mdps_internal_set_error("mdps_solver_create: N too large for this limb count (two staged digit vectors "
                                    "exceed 227 KB of shared memory)");
            return MDPS_EINVAL;
        }
        TS_TRY(cudaFuncSetAttribute(ts::ts_main_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)s->smem_main),
               MDPS_ECUDA);
        TS_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ts::ts_main_kernel<L>, ts::main_threads(L),
                                                             s->smem_main),
               MDPS_ECUDA);
        if (per < 1) {
            mdps_internal_set_error("solver kernel does not fit on an SM");
            return MDPS_ECUDA;
        }
        s->grid_main = sms * per;
        // Gauss-Jordan on a cluster: C CTAs (8, or 16 non-portable) holding
        // ceil(n / C) rows of [left | I] each; else the single-block kernel
        const int C = std::min(8, s->n);
        const int rows = (s->n + C - 1) / C;
        const size_t gsm = ((size_t)rows * 2 * s->n + 2 * s->n) * 16 + 16;
        if (gsm <= 200 * 1024) {
            bool ok = cudaFuncSetAttribute(ts::ts_gj_cluster_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)gsm) == cudaSuccess;
            if (ok && C > 8)
                ok = cudaFuncSetAttribute(ts::ts_gj_cluster_kernel<L>,
                                          cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
            if (ok) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(C);
                cfg.blockDim = dim3(ts::GJC_THREADS);
                cfg.dynamicSmemBytes = gsm;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = C;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                int nclusters = 0;
                ok = cudaOccupancyMaxActiveClusters(&nclusters, ts::ts_gj_cluster_kernel<L>, &cfg) == cudaSuccess &&
                     nclusters >= 1;
            }
            cudaGetLastError();
            if (ok) {
                s->gj_cluster = C;
                s->gj_rows = rows;
                s->gj_smem = gsm;
            }
        }
        return MDPS_OK;
    }
};

template <int L>
struct TsRun {
    static int run(mdps_solver *s, const double *J, const double *b, double *dx, int negate, cudaStream_t st) {
        const int N = s->N, n = s->n, D = s->D;
        const size_t total = (size_t)N * n * D + (size_t)N * D;
        const int pb = (int)std::min<size_t>((total + 127) / 128, 148 * 32);
        TS_TRY(cudaMemsetAsync(s->ctl, 0, sizeof(ts::Ctl), st), MDPS_ECUDA);
        ts::ts_pack_kernel<L><<<pb, 128, 0, st>>>(J, b, s->Ad, s->Ae, s->Ac, s->Ace, s->Rp, s->Re, N, n, D, negate);
        TS_TRY(cudaGetLastError(), MDPS_ECUDA);
        if (s->gj_cluster > 0) {  // Gauss-Jordan on a thread-block cluster (DSMEM)
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(s->gj_cluster);
            cfg.blockDim = dim3(ts::GJC_THREADS);
            cfg.dynamicSmemBytes = s->gj_smem;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = s->gj_cluster;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            TS_TRY(cudaLaunchKernelEx(&cfg, ts::ts_gj_cluster_kernel<L>, J, s->piv, s->ctl, s->Wr, s->Wre, s->Wc,
                                      s->Wce, N, n, D, s->gj_rows),
                   MDPS_ECUDA);
        } else {
            ts::ts_gj_kernel<L><<<1, ts::GJ_THREADS, 0, st>>>(J, s->M, s->piv, s->ctl, s->Wr, s->Wre, s->Wc, s->Wce,
                                                              N, n, D);
            TS_TRY(cudaGetLastError(), MDPS_ECUDA);
        }
        const double *Ad = s->Ad, *Ac = s->Ac;
        const int *Ae = s->Ae, *Ace = s->Ace;
        void *args[] = {(void *)&Ad,     (void *)&Ae,    (void *)&Ac,    (void *)&Ace,    (void *)&s->Wr,
                        (void *)&s->Wre, (void *)&s->Wc, (void *)&s->Wce, (void *)&s->Wc2, (void *)&s->Wce2,
                        (void *)&s->Er,  (void *)&s->Ere, (void *)&s->Pc, (void *)&s->Pce, (void *)&s->Mr,
                        (void *)&s->Mre, (void *)&s->Rp, (void *)&s->Re, (void *)&s->Xp,  (void *)&s->Xe,
                        (void *)&dx,     (void *)&s->Gc, (void *)&s->Gce, (void *)&s->N,  (void *)&s->n,
                        (void *)&s->D,   (void *)&s->ctl, (void *)&s->trace};
        TS_TRY(cudaLaunchCooperativeKernel((const void *)ts::ts_main_kernel<L>, dim3(s->grid_main),
                                           dim3(ts::main_threads(L)), args, s->smem_main, st),
               MDPS_ECUDA);
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
    cudaFree(s->nv);
    cudaFree(s->nj);
    cudaFree(s->ndx);
    cudaFree(s->nnorm);
    void *ptrs[] = {s->Ad, s->Ae,  s->Ac,  s->Ace, s->M,  s->Wr, s->Wre, s->Wc,  s->Wce, s->Wc2, s->Wce2, s->Er,
                    s->Ere, s->Pc, s->Pce, s->Mr, s->Mre, s->Rp, s->Re, s->Xp, s->Xe, s->piv, s->ctl, s->trace,
                    s->Gc, s->Gce};
    for (void *p : ptrs) cudaFree(p);
}

extern "C" mdps_solver *mdps_solver_create_ls(int32_t N, int32_t n, int32_t degree, int32_t limbs) {
    // N <= 128 keeps every exact digit accumulator below 2^53: a dot product
    // has at most 2N terms (two segments), each < 2^44 units of the top digit
    if (n < 1 || N < n || N > 128 || degree < 0 || degree > 255 ||
        !(limbs == 2 || limbs == 3 || limbs == 4 || limbs == 5 || limbs == 8 || limbs == 10)) {
        mdps_internal_set_error(
            "mdps_solver_create: need 1 <= n <= N <= 128, 0 <= degree <= 255, limbs in {2,3,4,5,8,10}");
        return nullptr;
    }
    mdps_solver *s = new (std::nothrow) mdps_solver();
    if (!s) {
        mdps_internal_set_error("out of host memory");
        return nullptr;
    }
    s->N = N;
    s->n = n;
    s->D = degree + 1;
    s->L = limbs;
    s->S = digits_for(limbs);
    cudaGetDevice(&s->device);
    const size_t D = s->D, S = s->S, VN = 2 * S * n, VM = 2 * S * N, Nn = (size_t)N * n;
    const size_t sz[] = {
        D * Nn * 2 * S * 8, D * Nn * 2 * 4,          // Ad, Ae: rows of A_k
        Nn * 2 * S * 8,     Nn * 2 * 4,              // Ac, Ace: columns of A_0
        (size_t)n * 2 * n * 2 * 8,                  // M: Gauss-Jordan [n][2n] complex
        n * VM * 8,         (size_t)n * 2 * N * 4,   // Wr, Wre
        N * VN * 8,         (size_t)N * 2 * n * 4,   // Wc, Wce
        N * VN * 8,         (size_t)N * 2 * n * 4,   // Wc2, Wce2
        n * VN * 8,         (size_t)n * 2 * n * 4,   // Er, Ere
        N * VM * 8,         (size_t)N * 2 * N * 4,   // Pc, Pce
        n * VM * 8,         (size_t)n * 2 * N * 4,   // Mr, Mre
        D * VM * 8,         D * 2 * N * 4,           // Rp, Re
        4 * VN * 8,         8 * (size_t)n * 4,       // Xp, Xe (two vectors, double-buffered)
        n * sizeof(int),    sizeof(ts::Ctl),         // piv, ctl
        ts::TRACE_MAX * sizeof(long long),           // trace
        (size_t)n * VN * 8, (size_t)n * 2 * n * 4};  // Gc, Gce
    void **ptrs[] = {(void **)&s->Ad,  (void **)&s->Ae,   (void **)&s->Ac,  (void **)&s->Ace, (void **)&s->M,
                     (void **)&s->Wr,  (void **)&s->Wre,  (void **)&s->Wc,  (void **)&s->Wce, (void **)&s->Wc2,
                     (void **)&s->Wce2, (void **)&s->Er,  (void **)&s->Ere, (void **)&s->Pc,  (void **)&s->Pce,
                     (void **)&s->Mr,  (void **)&s->Mre,  (void **)&s->Rp,  (void **)&s->Re,  (void **)&s->Xp,
                     (void **)&s->Xe,  (void **)&s->piv,  (void **)&s->ctl, (void **)&s->trace, (void **)&s->Gc,
                     (void **)&s->Gce};
    static_assert(sizeof(sz) / sizeof(sz[0]) == sizeof(ptrs) / sizeof(ptrs[0]), "buffer table");
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
    cudaMemset(s->ctl, 0, sizeof(ts::Ctl));
    if (ts_dispatch<TsGeom>(limbs, s) != MDPS_OK) {
        solver_free(s);
        delete s;
        return nullptr;
    }
    return s;
}

extern "C" mdps_solver *mdps_solver_create(int32_t n, int32_t degree, int32_t limbs) {
    return mdps_solver_create_ls(n, n, degree, limbs);
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
    if (overlaps(J, (size_t)s->N * s->n * ser * sizeof(double)) || overlaps(b, (size_t)s->N * ser * sizeof(double))) {
        mdps_internal_set_error("mdps_solve: dx_out aliases an input");
        return MDPS_EINVAL;
    }
    s->last = st;
    return ts_dispatch<TsRun>(s->L, s, J, b, dx, negate, st);
}

extern "C" int mdps_solve(mdps_solver *s, const double *J, const double *b, double *dx, mdps_stream_t stream) {
    return mdps_solve_internal(s, J, b, dx, 0, (cudaStream_t)stream);
}

extern "C" int mdps_solver_flags(mdps_solver *s, int32_t *flags) {
    if (!s || !flags) {
        mdps_internal_set_error("mdps_solver_flags: NULL argument");
        return MDPS_EINVAL;
    }
    TS_TRY(cudaStreamSynchronize(s->last), MDPS_ECUDA);
    ts::Ctl c;
    TS_TRY(cudaMemcpy(&c, s->ctl, sizeof c, cudaMemcpyDeviceToHost), MDPS_ECUDA);
    *flags = c.status & (MDPS_SOLVE_SINGULAR | MDPS_SOLVE_NOT_CONVERGED);
    return MDPS_OK;
}

extern "C" int mdps_solver_status(mdps_solver *s, int32_t *pivots, int32_t *singular) {
    if (!s) {
        mdps_internal_set_error("mdps_solver_status: NULL solver");
        return MDPS_EINVAL;
    }
    TS_TRY(cudaStreamSynchronize(s->last), MDPS_ECUDA);
    if (pivots) TS_TRY(cudaMemcpy(pivots, s->piv, s->n * sizeof(int), cudaMemcpyDeviceToHost), MDPS_ECUDA);
    if (singular) {
        ts::Ctl c;
        TS_TRY(cudaMemcpy(&c, s->ctl, sizeof c, cudaMemcpyDeviceToHost), MDPS_ECUDA);
        *singular = c.status & 1;
    }
    return MDPS_OK;
}

// Algorithmic work of one solve in complex md multiply-adds: the substitution
// loop (d+1 products W r_j and N n d(d+1)/2 right-hand-side terms) plus one
// Newton-Schulz step (I - W A_0 and E W: 2 n^2 N).  FP64
// instructions: 4 truncated S x S digit triangles per complex term.
extern "C" int mdps_solver_stats(const mdps_solver *s, mdps_solver_info *out) {
    if (!s || !out) {
        mdps_internal_set_error("mdps_solver_stats: NULL argument");
        return MDPS_EINVAL;
    }
    std::memset(out, 0, sizeof *out);
    const int64_t N = s->N, n = s->n, D = s->D;
    const int64_t loop = D * n * N + N * n * D * (D - 1) / 2, refine = n * n * N + n * N * n;
    out->complex_fma = loop + refine;
    out->fp64_ops = out->complex_fma * 4 * (int64_t)(s->S * (s->S + 1) / 2);
    out->launches = 3;
    out->grid_blocks = s->grid_main;
    out->workspace_bytes = s->bytes;
    return MDPS_OK;
}

extern "C" void mdps_solver_destroy(mdps_solver *s) {
    if (!s) return;
    cudaDeviceSynchronize();
    solver_free(s);
    delete s;
}

extern "C" int mdps_solver_trace(mdps_solver *s, int64_t *ns, int32_t max, int32_t *refine_steps) {
    if (!s || !ns) {
        mdps_internal_set_error("mdps_solver_trace: NULL argument");
        return MDPS_EINVAL;
    }
    TS_TRY(cudaStreamSynchronize(s->last), MDPS_ECUDA);
    ts::Ctl c;
    TS_TRY(cudaMemcpy(&c, s->ctl, sizeof c, cudaMemcpyDeviceToHost), MDPS_ECUDA);
    const int cnt = std::min(c.ntrace, (int)max);
    if (cnt > 0) TS_TRY(cudaMemcpy(ns, s->trace, cnt * sizeof(long long), cudaMemcpyDeviceToHost), MDPS_ECUDA);
    if (refine_steps) *refine_steps = c.refine_steps;
    return cnt;
}

// ---- Newton's method on power series (§6 stopping rule) ----------
template <int L>
struct TsUpdate {
    static int run(double *x, const double *dx, int n, int D, unsigned long long *norm, cudaStream_t st) {
        const int blocks = (n * D + 127) / 128;
        ts::ts_update_kernel<L><<<blocks, 128, 0, st>>>(x, dx, n, D, norm);
        TS_TRY(cudaGetLastError(), MDPS_ECUDA);
        return MDPS_OK;
    }
};

extern "C" int mdps_newton_step(mdps_system *sys, mdps_solver *s, double *x, double *dx_out, double *update_norm,
                                mdps_stream_t stream) {
    if (!sys || !s || !x) {
        mdps_internal_set_error("mdps_newton_step: NULL argument");
        return MDPS_EINVAL;
    }
    int sN = 0, sn = 0, sD = 0, sL = 0;
    mdps_internal_system_shape(sys, &sN, &sn, &sD, &sL);
    if (sN != s->N || sn != s->n || sD != s->D || sL != s->L) {
        mdps_internal_set_error("mdps_newton_step: system and solver differ in N, n, degree or limbs");
        return MDPS_EINVAL;
    }
    const size_t ser = (size_t)2 * s->L * s->D;
    if (!s->nv) {
        if (cudaMalloc(&s->nv, (size_t)s->N * ser * 8) != cudaSuccess ||
            cudaMalloc(&s->nj, (size_t)s->N * s->n * ser * 8) != cudaSuccess ||
            cudaMalloc(&s->ndx, (size_t)s->n * ser * 8) != cudaSuccess ||
            cudaMalloc(&s->nnorm, sizeof(unsigned long long)) != cudaSuccess) {
            cudaGetLastError();
            mdps_internal_set_error("mdps_newton_step: device allocation failed");
            return MDPS_ENOMEM;
        }
        s->bytes += (size_t)(s->N + s->n + s->N * s->n) * ser * 8 + 8;
    }
    cudaStream_t cs = (cudaStream_t)stream;
    int rc = mdps_eval_diff(sys, x, s->nv, s->nj, stream);
    if (rc != MDPS_OK) return rc;
    double *dx = dx_out ? dx_out : s->ndx;
    rc = mdps_solve_internal(s, s->nj, s->nv, dx, /*negate=*/1, cs);  // J dx = -f
    if (rc != MDPS_OK) return rc;
    TS_TRY(cudaMemsetAsync(s->nnorm, 0, sizeof(unsigned long long), cs), MDPS_ECUDA);
    rc = ts_dispatch<TsUpdate>(s->L, x, (const double *)dx, s->n, s->D, s->nnorm, cs);
    if (rc != MDPS_OK) return rc;
    if (update_norm) TS_TRY(cudaMemcpyAsync(update_norm, s->nnorm, sizeof(double), cudaMemcpyDeviceToDevice, cs),
                            MDPS_ECUDA);
    return MDPS_OK;
}

extern "C" int mdps_newton(mdps_system *sys, mdps_solver *s, double *x, int32_t max_iters, double tol,
                           double *last_norm, mdps_stream_t stream) {
    if (max_iters < 1 || !(tol >= 0.0)) {
        mdps_internal_set_error("mdps_newton: need max_iters >= 1 and tol >= 0");
        return MDPS_EINVAL;
    }
    double norm = 0.0;
    int it = 0;
    while (it < max_iters) {
        const int rc = mdps_newton_step(sys, s, x, nullptr, nullptr, stream);
        if (rc != MDPS_OK) return rc;
        it++;
        unsigned long long bits = 0;
        TS_TRY(cudaMemcpyAsync(&bits, s->nnorm, sizeof bits, cudaMemcpyDeviceToHost, (cudaStream_t)stream),
               MDPS_ECUDA);
        TS_TRY(cudaStreamSynchronize((cudaStream_t)stream), MDPS_ECUDA);
        std::memcpy(&norm, &bits, sizeof norm);
        if (norm <= tol) break;
    }
    if (last_norm) *last_norm = norm;
    return it;
}
