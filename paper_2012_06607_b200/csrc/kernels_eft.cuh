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

// tasks [task0, task0 + ntasks) of [0, n) values_out, [n, n + n*n) jacobian_out (row-major)
template <int L>
__global__ void __launch_bounds__(128) accum_eft_kernel(const double *__restrict__ pool,
                                                       const int *__restrict__ task_ptr,
                                                       const int *__restrict__ ent_slot,
                                                       const int *__restrict__ ent_w, int task0, int ntasks,
                                                       int n, int D, double *__restrict__ values,
                                                       double *__restrict__ jac) {
    const int LD2 = 2 * L * D;
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (long long)ntasks * D) return;
    const int task = task0 + (int)(g / D), k = (int)(g % D);
    double Br[L + 1], Bi[L + 1];
    md_zero(Br);
    md_zero(Bi);
    // software pipeline over the entries: entry e+1's limbs (and e+2's slot
    // index) are loaded while entry e is summed — the loop is bound by the
    // chained loads (slot index, then limbs), not by the bins arithmetic
    const int e0 = task_ptr[task], e1 = task_ptr[task + 1];
    auto load = [&](int e, double (&ar)[L], double (&ai)[L], int slot) {
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
        load(e0, ar, ai, ent_slot[e0]);
        w = ent_w[e0];
        if (e0 + 1 < e1) slot_next = ent_slot[e0 + 1];
    }
    for (int e = e0; e < e1; e++) {
        double nr[L], ni[L];
        int nw = 0, slot_nn = 0;
        if (e + 1 < e1) {
            load(e + 1, nr, ni, slot_next);
            nw = ent_w[e + 1];
            if (e + 2 < e1) slot_nn = ent_slot[e + 2];
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

}  // namespace mdps
