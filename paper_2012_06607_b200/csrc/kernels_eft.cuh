// kernels_eft.cuh — product and accumulation kernels on limb planes
// (MDPS_ALGO_EFT): the paper's md arithmetic transcribed to sm_100a.
//
// conv_eft: one product job z = x * y mod t^D per group of
// T = ceil(D/2) threads; P jobs per block.  Both input series are staged in
// shared memory.  Thread t computes z_t and z_{D-1-t} ("folded" triangle:
// D+1 terms per thread, no idle lanes); each complex term adds
// re += ar*br - ai*bi, im += ar*bi + ai*br into (L+1) level bins
// (md.cuh), renormalised to L limbs at the end.
//
// accum_eft: one thread per (output series, coefficient k): the value and
// Jacobian addition jobs, summing a CSR list of pool
// series with integer weights (the exponents a_l) in fixed order.
#pragma once
#include "md.cuh"

namespace mdps {

// pool series layout: [slot][2][L][D] doubles
template <int L>
__global__ void __launch_bounds__(128) conv_eft_kernel(double *__restrict__ pool,
                                                      const int *__restrict__ jobs, int njobs, int D,
                                                      int T, int P) {
    extern __shared__ double sm[];
    const int LD2 = 2 * L * D;      // doubles per series
    const int JS = 2 * LD2 + 2;     // per-job stride (+2: skew banks across jobs)
    const int jl = threadIdx.x / T, t = threadIdx.x - jl * T;
    const int job0 = blockIdx.x * P;
    for (int idx = threadIdx.x; idx < P * 2 * LD2; idx += blockDim.x) {
        const int j2 = idx / (2 * LD2), r = idx - j2 * 2 * LD2;
        const int job = job0 + j2;
        if (job < njobs) {
            const int which = r >= LD2, off = r - which * LD2;
            const int src = jobs[4 * job + which];
            sm[j2 * JS + r] = pool[(size_t)src * LD2 + off];
        }
    }
    __syncthreads();
    const int job = job0 + jl;
    if (jl >= P || job >= njobs) return;
    const double *sx = sm + jl * JS, *sy = sx + LD2;
    double *save = sm + P * JS + (size_t)threadIdx.x * 2 * (L + 1);

    double Br[L + 1], Bi[L + 1];
    md_zero(Br);
    md_zero(Bi);
    const int k1 = t, k2 = D - 1 - t;
    for (int j = 0; j <= D; j++) {
        const bool first = j <= t;
        const int i = first ? j : j - t - 1;
        const int k = first ? k1 : k2;
        double ar[L], ai[L], nai[L], br[L], bi[L];
#pragma unroll
        for (int p = 0; p < L; p++) {
            ar[p] = sx[p * D + i];
            ai[p] = sx[(L + p) * D + i];
            nai[p] = -ai[p];
            br[p] = sy[p * D + (k - i)];
            bi[p] = sy[(L + p) * D + (k - i)];
        }
        bins_fma<L>(Br, ar, br);
        bins_fma<L>(Br, nai, bi);
        bins_fma<L>(Bi, ar, bi);
        bins_fma<L>(Bi, ai, br);
        if (j == t) {  // z_{k1} complete: park its bins, start z_{k2}
#pragma unroll
            for (int p = 0; p <= L; p++) {
                save[p] = Br[p];
                save[L + 1 + p] = Bi[p];
                Br[p] = 0.0;
                Bi[p] = 0.0;
            }
        }
    }
    double *z = pool + (size_t)jobs[4 * job + 2] * LD2;
    double zr[L], zi[L], Fr[L + 1], Fi[L + 1];
#pragma unroll
    for (int p = 0; p <= L; p++) {
        Fr[p] = save[p];
        Fi[p] = save[L + 1 + p];
    }
    md_renorm(Fr, zr);
    md_renorm(Fi, zi);
#pragma unroll
    for (int p = 0; p < L; p++) {
        z[p * D + k1] = zr[p];
        z[(L + p) * D + k1] = zi[p];
    }
    md_renorm(Br, zr);
    md_renorm(Bi, zi);
#pragma unroll
    for (int p = 0; p < L; p++) {
        z[p * D + k2] = zr[p];
        z[(L + p) * D + k2] = zi[p];
    }
}

// B += the bins of another partial sum (level o at level o; guard plainly)
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

// lanes per (addition job, coefficient): a value sums one series per monomial
// of its polynomial (64..128 entries in the configs), a Jacobian entry one per
// monomial that contains its variable (8..24) — one thread per output would
// run the value jobs' chains (entries x one dependent md addition) long after
// the Jacobian jobs are done.  Fixed per job type and (L, D), so the summation
// order of an output never depends on the system it is part of (shards and
// batches stay bitwise equal to the whole).  Jacobian jobs of long, wide
// series (L D >= 320) fill the GPU on one lane each and are throughput-bound:
// a second lane only adds its merge (measured: deca 0.88 -> 1.01 ms with two).
constexpr int ACCUM_LANES_VALUE = 8;
__host__ __device__ constexpr int accum_lanes_jac(int L, int D) { return L * D >= 320 ? 1 : 2; }

// one addition job's coefficient k on G adjacent lanes: lane g sums entries
// e0 + g, e0 + g + G, ... in order, then the lanes' bins are merged pairwise
// in a fixed tree (lane g takes lane g + off's bins, off = 1, 2, 4, ...), and
// lane 0 renormalises and stores.  Deterministic: no atomics, fixed order.
// Structural zeros (no entries) are written as exact zeros.
// `active` false: a padding thread (it still takes part in the shuffles).
template <int L, int G>
__device__ __forceinline__ void accum_lanes(const double *__restrict__ pool, const int *__restrict__ task_ptr,
                                            const int *__restrict__ ent_slot, const int *__restrict__ ent_w,
                                            int task, int k, int g, bool active, int n, int D,
                                            double *__restrict__ values, double *__restrict__ jac) {
    const int LD2 = 2 * L * D;
    double Br[L + 1], Bi[L + 1];
    md_zero(Br);
    md_zero(Bi);
    // software pipeline over the lane's entries: entry e+G's limbs (and
    // e+2G's slot index) are loaded while entry e is summed — the loop is
    // bound by the chained loads (slot index, then limbs), not by the bins
    const int e0 = active ? task_ptr[task] + g : 0, e1 = active ? task_ptr[task + 1] : 0;
    auto load = [&](double (&ar)[L], double (&ai)[L], int slot) {
        const double *s = pool + (size_t)slot * LD2;
#pragma unroll
        for (int p = 0; p < L; p++) {
            ar[p] = s[p * D + k];
            ai[p] = s[(L + p) * D + k];
        }
    };
    double ar[L], ai[L];
    int w = 0, slot_next = 0;
    if (e0 < e1) {
        load(ar, ai, ent_slot[e0]);
        w = ent_w[e0];
        if (e0 + G < e1) slot_next = ent_slot[e0 + G];
    }
    for (int e = e0; e < e1; e += G) {
        double nr[L], ni[L];
        int nw = 0, slot_nn = 0;
        if (e + G < e1) {
            load(nr, ni, slot_next);
            nw = ent_w[e + G];
            if (e + 2 * G < e1) slot_nn = ent_slot[e + 2 * G];
        }
        if (w == 1) {
            bins_add<L>(Br, ar);
            bins_add<L>(Bi, ai);
        } else {
            bins_add_scaled<L>(Br, ar, (double)w);
            bins_add_scaled<L>(Bi, ai, (double)w);
        }
#pragma unroll
        for (int p = 0; p < L; p++) {
            ar[p] = nr[p];
            ai[p] = ni[p];
        }
        w = nw;
        slot_next = slot_nn;
    }
#pragma unroll
    for (int off = 1; off < G; off <<= 1) {
        double Cr[L + 1], Ci[L + 1];
#pragma unroll
        for (int p = 0; p <= L; p++) {
            Cr[p] = __shfl_down_sync(0xffffffffu, Br[p], off);
            Ci[p] = __shfl_down_sync(0xffffffffu, Bi[p], off);
        }
        bins_merge<L>(Br, Cr);  // only lanes with g % (2 off) == 0 carry the result on
        bins_merge<L>(Bi, Ci);
    }
    if (!active || g != 0) return;
    double zr[L], zi[L];
    md_renorm(Br, zr);
    md_renorm(Bi, zi);
    double *o = task < n ? values + (size_t)task * LD2 : jac + (size_t)(task - n) * LD2;
#pragma unroll
    for (int p = 0; p < L; p++) {
        o[p * D + k] = zr[p];
        o[(L + p) * D + k] = zi[p];
    }
}

// Addition jobs of one chunk in one launch: the value jobs [v0, v0 + nv) on
// ACCUM_LANES_VALUE lanes per coefficient (blocks [0, vblocks)), the Jacobian
// jobs [j0, j0 + nj) on GJ = accum_lanes_jac(L, D) (the other blocks); tasks [0, n) are
// values_out, [n, n + n*nvars) jacobian_out (row-major).  Threads of a job
// type: [job][coefficient k][lane g].
template <int L, int GJ>
__global__ void __launch_bounds__(128) accum_eft_kernel(const double *__restrict__ pool,
                                                       const int *__restrict__ task_ptr,
                                                       const int *__restrict__ ent_slot,
                                                       const int *__restrict__ ent_w, int v0, int nv, int vblocks,
                                                       int j0, int nj, int n, int D, double *__restrict__ values,
                                                       double *__restrict__ jac) {
    if ((int)blockIdx.x < vblocks) {
        constexpr int G = ACCUM_LANES_VALUE;
        const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
        const long long job = t / ((long long)D * G);
        const int r = (int)(t - job * D * G);
        accum_lanes<L, G>(pool, task_ptr, ent_slot, ent_w, v0 + (int)job, r / G, r % G, job < nv, n, D, values, jac);
    } else {
        constexpr int G = GJ;
        const long long t = (long long)(blockIdx.x - vblocks) * blockDim.x + threadIdx.x;
        const long long job = t / ((long long)D * G);
        const int r = (int)(t - job * D * G);
        accum_lanes<L, G>(pool, task_ptr, ent_slot, ent_w, j0 + (int)job, r / G, r % G, job < nj, n, D, values, jac);
    }
}

}  // namespace mdps
