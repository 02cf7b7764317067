// md.cuh — header-only device multiple-double arithmetic for sm_100a.
//
// A multiple-double number is an unevaluated sum of L hardware doubles
// (§2), limb 0 most significant, L in {2,3,4,5,8,10}
// (Table 1).  Every operation here is built from the
// error-free transformations of PAPER.md:76-80: TwoSum, TwoProd via fused
// multiply-add, and renormalisation.  All arithmetic uses explicit
// round-to-nearest intrinsics (__dadd_rn, __dsub_rn, __dmul_rn, __fma_rn),
// which nvcc never contracts or reassociates (and the library is built with
// --fmad=false besides).
//
// Level bins.  A sum of many md terms is kept in G = L+1 bins B[0..L]: a
// value of order o (magnitude ~2^(-53 o) relative to the leading term) is
// deposited with TwoSum into B[o]; the exact error cascades by TwoSum into
// B[o+1], ..., B[L-1] and is added plainly into the guard bin B[L].  Bins
// 0..L-1 are therefore exact and all rounding happens one order below the
// last limb.  md_renorm turns the bins into L limbs at the end.
//
// This file shares no code with the CPU oracle (oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mdps {

__device__ __forceinline__ void two_sum(double a, double b, double &s, double &e) {
    s = __dadd_rn(a, b);
    double bb = __dsub_rn(s, a);
    e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

__device__ __forceinline__ void two_prod(double a, double b, double &p, double &e) {
    p = __dmul_rn(a, b);
    e = __fma_rn(a, b, -p);
}

// deposit v at static level O of an (L+1)-bin accumulator
template <int L, int O>
__device__ __forceinline__ void bins_dep(double (&B)[L + 1], double v) {
#pragma unroll
    for (int t = O; t < L; t++) two_sum(B[t], v, B[t], v);
    B[L] = __dadd_rn(B[L], v);
}

// B += a * b for L-limb a, b.  Partial products a_p b_q with p+q <= L-1 as
// TwoProd (hi at level p+q, lo at level p+q+1), p+q = L as FMAs into the
// guard bin, p+q > L dropped (<= 2^(-53(L+1)) |a||b| each).
template <int L>
__device__ __forceinline__ void bins_fma(double (&B)[L + 1], const double (&a)[L], const double (&b)[L]) {
#pragma unroll
    for (int o = 0; o <= L - 1; o++) {
#pragma unroll
        for (int p = 0; p <= o; p++) {
            double h, l;
            two_prod(a[p], b[o - p], h, l);
#pragma unroll
            for (int t = o; t < L; t++) two_sum(B[t], h, B[t], h);
            B[L] = __dadd_rn(B[L], h);
#pragma unroll
            for (int t = o + 1; t < L; t++) two_sum(B[t], l, B[t], l);
            B[L] = __dadd_rn(B[L], l);
        }
    }
#pragma unroll
    for (int p = 1; p <= L - 1; p++) B[L] = __fma_rn(a[p], b[L - p], B[L]);
}

// B += a (limb p at level p)
template <int L>
__device__ __forceinline__ void bins_add(double (&B)[L + 1], const double (&a)[L]) {
#pragma unroll
    for (int p = 0; p < L; p++) {
        double v = a[p];
#pragma unroll
        for (int t = p; t < L; t++) two_sum(B[t], v, B[t], v);
        B[L] = __dadd_rn(B[L], v);
    }
}

// B += w * a (w an integer weight, exact products via TwoProd)
template <int L>
__device__ __forceinline__ void bins_add_scaled(double (&B)[L + 1], const double (&a)[L], double w) {
#pragma unroll
    for (int p = 0; p < L; p++) {
        double h, l;
        two_prod(a[p], w, h, l);
#pragma unroll
        for (int t = p; t < L; t++) two_sum(B[t], h, B[t], h);
        B[L] = __dadd_rn(B[L], h);
#pragma unroll
        for (int t = p + 1; t < L; t++) two_sum(B[t], l, B[t], l);
        B[L] = __dadd_rn(B[L], l);
    }
}

// Renormalise N values (roughly decreasing magnitude, possibly overlapping)
// into their leading L limbs: pass l runs a bottom-up VecSum over v[l..N-1],
// leaving the rounded sum of the remainder in v[l] and the exact errors
// below it (the sum of v is preserved until the final truncation to L).
// The result is non-overlapping up to a few ulps of each limb.
template <int N, int L>
__device__ __forceinline__ void md_renorm(double (&v)[N], double (&out)[L]) {
#pragma unroll
    for (int l = 0; l < L; l++) {
        double s = v[N - 1];
#pragma unroll
        for (int i = N - 2; i >= l; i--) two_sum(v[i], s, s, v[i + 1]);
        v[l] = s;
        out[l] = s;
    }
}

template <int N>
__device__ __forceinline__ void md_zero(double (&v)[N]) {
#pragma unroll
    for (int i = 0; i < N; i++) v[i] = 0.0;
}

// ---- number-level operations ------------------------------------------------
template <int L>
__device__ __forceinline__ void md_add(const double (&a)[L], const double (&b)[L], double (&c)[L]) {
    double B[L + 1];
    md_zero(B);
    bins_add<L>(B, a);
    bins_add<L>(B, b);
    md_renorm(B, c);
}

template <int L>
__device__ __forceinline__ void md_mul(const double (&a)[L], const double (&b)[L], double (&c)[L]) {
    double B[L + 1];
    md_zero(B);
    bins_fma<L>(B, a, b);
    md_renorm(B, c);
}

// ---- frozen FP64 instruction counts (DADD/DSUB/DMUL/DFMA, 1 each) -------------
// c(L) of the EFT path, counted from the code above.
__host__ __device__ constexpr long long ops_bins_fma(int L) {
    long long ops = 0;
    for (int o = 0; o <= L - 1; o++)
        for (int p = 0; p <= o; p++) ops += 2 + 6 * (L - o) + 1 + 6 * (L - o - 1) + 1;
    return ops + (L - 1);
}
__host__ __device__ constexpr long long ops_bins_add(int L) {
    long long ops = 0;
    for (int p = 0; p < L; p++) ops += 6 * (L - p) + 1;
    return ops;
}
__host__ __device__ constexpr long long ops_bins_add_scaled(int L) {
    long long ops = 0;
    for (int p = 0; p < L; p++) ops += 2 + 6 * (L - p) + 1 + 6 * (L - p - 1) + 1;
    return ops;
}
__host__ __device__ constexpr long long ops_renorm(int N, int L) {
    long long ops = 0;
    for (int l = 0; l < L; l++) ops += 6 * (N - 1 - l);
    return ops;
}

}  // namespace mdps
