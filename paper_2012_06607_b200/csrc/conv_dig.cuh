// conv_dig.cuh — the product-job kernel on digit planes (MDPS_ALGO_DIGITS):
// z = x * y mod t^D for every job of one DAG level.
//
// See kernels_dig.cuh for the digit representation.  Mapping:
//  * P jobs per block; per job T = ceil(D/2) output pairs x F splits x NP
//    part lanes.  Thread (part lane, t, f) owns outputs k1 = t and k2 = D-1-t
//    — the folded triangle has exactly D+1 terms per pair, so no lane idles —
//    and the fold iterations j = f, f+F, ... (the F lanes of a pair are
//    adjacent lanes of one warp).
//  * Two passes (real part, imaginary part), one after the other on the same
//    thread (NP = 1) or one per part lane (NP = 2: twice the threads per job,
//    half its latency, no extra reduction — the parts are separate outputs;
//    for small levels and short bodies).  Each pass keeps S digit accumulators
//    and the 2S digits of the operand x_i in registers and streams the 2S
//    digits of y_{k-i} from shared memory: per digit pair one DFMA.
//  * Alignment: a term whose exponent is delta digits below the accumulator
//    anchor reads y's digit plane l - delta.  Shared memory holds PADZ zero
//    planes in front of y's planes, so for delta <= PADZ (the common case,
//    checked warp-uniformly) every load is base + compile-time offset; larger
//    shifts take a select-based path.  A term with a zero operand part is
//    read at delta = 0 (its product is zero anyway).
//  * Partials: a copy of the k1 partial is parked in shared memory when a
//    lane crosses the fold (lanes cross at different iterations) and the k2
//    terms go on top of it; k2 = A - park after the loop.  The F lanes'
//    partials are added with warp shuffles.  All additions are exact
//    (integer digits).
//  * Shared memory per job: x planes [2][S][D] (the pool's own layout, one
//    TMA bulk copy), y planes [2][PADZ+S][D] (PADZ zero planes in front of
//    each part, one bulk copy per part), exponents [2][2][D]; per thread a
//    parking slot of S doubles.
#pragma once
#include "kernels_dig.cuh"

namespace mdps {

constexpr int PADZ = 4;

__host__ __device__ inline size_t conv_dig_smem(int S, int D, int P, int threads) {
    const size_t per_job = (size_t)2 * S * D + (size_t)2 * (PADZ + S) * D;  // doubles
    return (size_t)P * per_job * sizeof(double) + (size_t)threads * (S + 2) * sizeof(double) +
           (size_t)P * 4 * D * sizeof(int) + 16;  // + mbarrier
}

// ---- TMA bulk copies (cp.async.bulk) with an mbarrier, single CTA ----------
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// one product pass over this thread's fold iterations.  REAL: real series
// (imaginary parts zero and never read): one product per term.
template <int L, int DT, bool REAL = false>
__device__ __forceinline__ void conv_dig_pass(const double *__restrict__ sx, const double *__restrict__ sy,
                                              const int *__restrict__ ex, const int *__restrict__ ey, int Drt,
                                              int part, int t, int f, int F, int eacc1, int eacc2,
                                              double (&A)[digits_for(L)], double *park) {
    constexpr int S = digits_for(L);
    constexpr int NORM = norm_every(S);
    const int D = DT > 0 ? DT : Drt;
    constexpr int P2 = PADZ + S;
    // part 0 (re): Ur*Wr - Ui*Wi ;  part 1 (im): Ur*Wi + Ui*Wr.  One code
    // copy serves both passes (instruction-cache footprint): the part only
    // selects the y planes and the sign applied to Wi (a sign-bit flip).
    const int w1part = part, w2part = 1 - part;
    const long long sgn = part == 0 ? (long long)0x8000000000000000ULL : 0LL;
    md_zero(A);
    bool switched = false;
    // Software pipeline, one term ahead.  Everything the next term needs
    // (its x digits, its y offset kk and its alignment shifts d1, d2, read
    // from the exponents) is prepared INSIDE the current term's body, where
    // the integer work and the shared-memory latency hide behind the DFMAs:
    // after digit row l the operand digit u = S-1-l has had its last use, so
    // its register takes the next term's digit u (no extra registers).  The
    // per-term preamble shrinks to the warp vote on the fast path.
    // fold iteration j -> term (i, kk = k - i): j <= t is term i = j of k1 = t,
    // j > t is term i = D - j of k2 = D-1-t (descending), so the x index is
    // j or D - j — the same for every pair of the warp at a given j (a
    // shared-memory broadcast) — and kk = t - j or j - t - 1 is consecutive
    // over the warp's pairs (one contiguous window), for both outputs
    auto term_index = [&](int j) { return j <= t ? j : D - j; };
    auto term_meta = [&](int j, int &kk, int &d1, int &d2) {
        const bool first = j <= t;
        const int i = term_index(j);
        kk = first ? t - j : j - t - 1;
        const int eacc = first ? eacc1 : eacc2;
        const int exr = ex[i], exi = REAL ? ZERO_E : ex[D + i];
        const int ey1 = ey[w1part * D + kk], ey2 = REAL ? 0 : ey[w2part * D + kk];
        d1 = eacc - exr - ey1;
        d2 = eacc - exi - ey2;
        if (exr + ey1 <= ZERO_E / 2) d1 = 0;  // zero product: any plane will do
        if (REAL || exi + ey2 <= ZERO_E / 2) d2 = 0;
    };
    double Ur[S], Ui[S];
    int kk, d1, d2;
    {
        const int j0 = min(f, D);  // a lane with f > D has no terms (clamped reads only)
        term_meta(j0, kk, d1, d2);
        const double *ux = sx + term_index(j0);
#pragma unroll
        for (int s = 0; s < S; s++) {
            Ur[s] = ux[s * D];
            Ui[s] = REAL ? 0.0 : ux[(S + s) * D];
        }
    }
    // part 0's sign (-Ui*Wi) is applied to the streamed y digit w2 (one flip
    // per digit row, inside the body) rather than to the S held x digits
    auto neg = [&](double w) { return __longlong_as_double(__double_as_longlong(w) ^ sgn); };
    // blocks of at most NORM terms, each closed by a carry pass: one loop
    // test per term (no per-term counter test and branch), and the carries
    // stay warp-uniform (every lane's block ends at the same iteration count
    // but for a shorter last one)
    for (int j = f; j <= D;) {
    const int jstop = min(D, j + (NORM - 1) * F);
    for (; j <= jstop; j += F) {
        // k1 partial complete: park a copy (raw) and keep accumulating — the
        // k2 terms go on top of it, and k2 = A - park after the loop (exact:
        // integer digits).  Not zeroing A keeps the in-loop work at S/2
        // stores, which the compiler predicates onto every term (a lane
        // crosses the fold once, at a lane-dependent iteration); zeroing
        // cost S more predicated moves per term (measured at qd: the park
        // was ~14% of the kernel's instructions).  No carry here: anything
        // done at the crossing runs divergently.  The raw partial is below
        // 2^53 (< NORM terms since the last carry) and is carried after the
        // loop, by all lanes at once; the block carries of A go on.
        if (j > t && !switched) {
            switched = true;
#pragma unroll
            for (int s = 0; s < S; s++) park[s] = A[s];
        }
        // the next term (this term again on the last iteration: harmless)
        const int jn = j + F <= D ? j + F : j;
        const double *uxn = sx + term_index(jn);
        int kkn, d1n, d2n;
        auto ahead = [&](int l) {  // called after digit row l of the body
            if (l == 1) term_meta(jn, kkn, d1n, d2n);
            const int u = S - 1 - l;
            Ur[u] = uxn[u * D];
            if (!REAL) Ui[u] = uxn[(S + u) * D];
        };
        const bool fast = d1 <= PADZ && d2 <= PADZ;
        if (__all_sync(__activemask(), fast)) {
            const double *W1 = sy + (w1part * P2 + PADZ - d1) * D + kk;
            const double *W2 = sy + (w2part * P2 + PADZ - d2) * D + kk;
            // software pipelined: row l+1's two digits load while row l's FMAs run
            double w1 = W1[0], w2 = REAL ? 0.0 : neg(W2[0]);
#pragma unroll
            for (int l = 0; l < S; l++) {
                double w1n = 0.0, w2n = 0.0;
                if (l + 1 < S) {
                    w1n = W1[(l + 1) * D];
                    if (!REAL) w2n = neg(W2[(l + 1) * D]);
                }
#pragma unroll
                for (int u = 0; u < S - l; u++) {
                    A[u + l] = __fma_rn(Ur[u], w1, A[u + l]);
                    if (!REAL) A[u + l] = __fma_rn(Ui[u], w2, A[u + l]);
                }
                ahead(l);
                w1 = w1n;
                w2 = w2n;
            }
        } else {
            const double *W1 = sy + w1part * P2 * D + kk;
            const double *W2 = sy + w2part * P2 * D + kk;
#pragma unroll
            for (int l = 0; l < S; l++) {
                const double w1 = (l >= d1) ? W1[(PADZ + l - d1) * D] : 0.0;
                const double w2 = (!REAL && l >= d2) ? neg(W2[(PADZ + l - d2) * D]) : 0.0;
#pragma unroll
                for (int u = 0; u < S - l; u++) {
                    A[u + l] = __fma_rn(Ur[u], w1, A[u + l]);
                    if (!REAL) A[u + l] = __fma_rn(Ui[u], w2, A[u + l]);
                }
                ahead(l);
            }
        }
        kk = kkn;
        d1 = d1n;
        d2 = d2n;
    }
    carry_pass(A);
    }
    if (!switched) {  // no k2 iterations on this lane: everything belongs to k1
#pragma unroll
        for (int s = 0; s < S; s++) park[s] = A[s];
    }
    // on return: park = the k1 partial (|digit| < 2^53), A = the k1 + k2
    // partials (carried, |digit| <= R/2 + 2^31)
}

template <int L>
__device__ __forceinline__ void conv_dig_emit_digits(const double (&A)[digits_for(L)], int eacc, double *zd, int *ze,
                                                     int D, int k, int part, double *scratch);

// normalise and write one output (k, part): limbs (zl != null) for the
// addition jobs and/or digits with their exponent (zd != null) for later
// products.  scratch: S+2 doubles of this thread's shared-memory slot (the
// leading-zero shift by the data-dependent z0 goes through a store/reload).
template <int L>
__device__ __forceinline__ void conv_dig_emit(double (&A)[digits_for(L)], int eacc, double *zd, int *ze, double *zl,
                                              int D, int k, int part, double *scratch) {
    constexpr int S = digits_for(L);
    // inputs: carry-passed partials (|A_t| <= R/2 + 2^31) summed over <= 8
    // lanes, so two parallel carry passes balance every digit to R/2 + 1
    carry_pass(A);
    carry_pass(A);
    if (zd) conv_dig_emit_digits<L>(A, eacc, zd, ze, D, k, part, scratch);
    if (zl) {  // limbs for the addition jobs: the exact accumulator rounded to L limbs
        double out[L];
        digits_to_limbs<L, S, true>(A, eacc - 1, out);  // A_t has weight R^(eacc-2-t); consumes A
#pragma unroll
        for (int p = 0; p < L; p++) zl[(part * L + p) * D + k] = out[p];
    }
}

// digits of a normalised accumulator with the leading-zero shift
template <int L>
__device__ __forceinline__ void conv_dig_emit_digits(const double (&A)[digits_for(L)], int eacc, double *zd, int *ze,
                                                     int D, int k, int part, double *scratch) {
    constexpr int S = digits_for(L);
    // Z = [c2, c1, c0, A_1 .. A_{S-1}], Z_u has weight R^(eacc - u)
    double a0 = A[0];
    const double c2 = rint_magic(__dmul_rn(a0, INV_RADIX * INV_RADIX));
    a0 = __fma_rn(-c2, RADIX * RADIX, a0);
    const double c1 = rint_magic(__dmul_rn(a0, INV_RADIX));
    const double c0 = __fma_rn(-c1, RADIX, a0);
    scratch[0] = c2;
    scratch[1] = c1;
    scratch[2] = c0;
    int z0 = S + 2;
#pragma unroll
    for (int s = S - 1; s >= 1; s--) {
        scratch[s + 2] = A[s];
        if (A[s] != 0.0) z0 = s + 2;
    }
    if (c0 != 0.0) z0 = 2;
    if (c1 != 0.0) z0 = 1;
    if (c2 != 0.0) z0 = 0;
    const int e = (z0 >= S + 2 || eacc <= ZERO_E / 2) ? ZERO_E : eacc + 1 - z0;
    const double *src = scratch + z0;
    const int avail = S + 2 - z0;
#pragma unroll
    for (int s = 0; s < S; s++) zd[(part * S + s) * D + k] = (s < avail && e != ZERO_E) ? src[s] : 0.0;
    ze[part * D + k] = e;
}

template <int L, int DT, bool REAL = false>
// register budget per SM: 4 blocks of 128 up to L = 4 (<= 128 registers),
// 3 up to L = 8 (<= 170), 2 above; 256-thread blocks for D = 128 and the
// generic-D build.  REAL: real systems (mdps_options.real): only the real
// part is computed; the imaginary limbs of the limb outputs are written as 0.
__global__ void __launch_bounds__(DT == 128 || DT == 0 ? 256 : 128,
                                  DT == 128 || DT == 0 ? 1 : (L <= 4 ? 4 : (L <= 8 ? 3 : 2)))
    conv_dig_kernel(double *__restrict__ dpool, int *__restrict__ epool, double *__restrict__ lpool,
                    const int *__restrict__ jobs, int njobs, int Drt, int T, int F, int P, int NPrt) {
    constexpr int S = digits_for(L);
    const int D = DT > 0 ? DT : Drt;
    const int SX = 2 * S * D, SY = 2 * (PADZ + S) * D;
    const int NP = REAL ? 1 : NPrt;  // part lanes per output pair (1 or 2)
    const int threads_per_job = T * F * NP;
    extern __shared__ __align__(16) double sm[];
    double *sdig = sm;                                        // [P][SX + SY]
    double *spark = sm + (size_t)P * (SX + SY);               // [threads][S]
    constexpr int PSTR = S + 2;                               // parking / emit scratch slot
    int *sexp = (int *)(spark + (size_t)blockDim.x * PSTR);   // [P][2 series][2][D]

    const int job0 = blockIdx.x * P;
    // stage: x planes -> [part][s][D] (the pool layout), y planes ->
    // [part][PADZ + s][D], zero planes.  Even D: three 16-byte aligned
    // contiguous runs per job (x whole, y per part), so one thread issues
    // three TMA bulk copies (cp.async.bulk) per job against an mbarrier while
    // the other warps write the zero planes and exponents.  Odd D: one warp
    // per plane row, scalar loads.
    uint64_t *bar = reinterpret_cast<uint64_t *>(sexp + (size_t)P * 4 * D);
    const bool use_tma = (D & 1) == 0;
    if (use_tma) {
        if (threadIdx.x == 0) mbar_init(bar, 1);
        __syncthreads();
        if (threadIdx.x < 32) {
            if (threadIdx.x == 0) mbar_expect_tx(bar, (unsigned)(P * 4 * S * D * 8));
            __syncwarp();
            for (int c = threadIdx.x; c < 3 * P; c += 32) {  // (job, copy): x | y re | y im
                const int jl = c / 3, which = c - jl * 3;
                const int job = min(job0 + jl, njobs - 1);
                double *base = sdig + (size_t)jl * (SX + SY);
                if (which == 0)
                    bulk_g2s(base, dpool + (size_t)jobs[4 * job] * dig_slot_stride(S, D), (unsigned)(2 * S * D * 8),
                             bar);
                else
                    bulk_g2s(base + SX + ((which - 1) * (PADZ + S) + PADZ) * D,
                             dpool + (size_t)jobs[4 * job + 1] * dig_slot_stride(S, D) + (size_t)(which - 1) * S * D,
                             (unsigned)(S * D * 8), bar);
            }
        }
    } else {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
        const int nrows = P * 4 * S;  // (job, which, part*S + s)
#pragma unroll 2
        for (int row = warp; row < nrows; row += nwarps) {
            const int jl = row / (4 * S), rem = row - jl * 4 * S;
            const int which = rem / (2 * S), ps = rem - which * 2 * S;
            const int part = ps / S, s = ps - part * S;
            const int job = min(job0 + jl, njobs - 1);
            const double *g = dpool + (size_t)jobs[4 * job + which] * dig_slot_stride(S, D) + (size_t)ps * D;
            double *dst = sdig + (size_t)jl * (SX + SY) + (which ? SX + (part * (PADZ + S) + PADZ + s) * D
                                                                   : (size_t)ps * D);
            if ((D & 1) == 0) {
                for (int k = 2 * lane; k < D; k += 64)
                    *reinterpret_cast<double2 *>(dst + k) = __ldg(reinterpret_cast<const double2 *>(g + k));
            } else {
                for (int k = lane; k < D; k += 32) dst[k] = __ldg(g + k);
            }
        }
    }
    for (int idx = threadIdx.x; idx < P * 2 * PADZ * D; idx += blockDim.x) {  // zero planes of both parts
        const int jl = idx / (2 * PADZ * D), r = idx - jl * 2 * PADZ * D;
        const int part = r / (PADZ * D), rr = r - part * PADZ * D;
        sdig[(size_t)jl * (SX + SY) + SX + part * (PADZ + S) * D + rr] = 0.0;
    }
    for (int idx = threadIdx.x; idx < P * 2 * 2 * D; idx += blockDim.x) {
        const int jl = idx / (4 * D), r = idx - jl * 4 * D;
        const int which = r / (2 * D), r2 = r - which * 2 * D;
        const int job = min(job0 + jl, njobs - 1);
        sexp[idx] = epool[(size_t)jobs[4 * job + which] * 2 * D + r2];
    }
    if (use_tma) mbar_wait(bar, 0);
    __syncthreads();

    const int jl = threadIdx.x / threads_per_job;
    const int r0 = threadIdx.x - jl * threads_per_job;
    const int pl = NP == 2 ? r0 / (T * F) : 0;  // part lane (NP = 2: this thread's part)
    const int r = r0 - pl * T * F;
    const int t = r / F, f = r - t * F;
    const int jlc = min(jl, P - 1);  // padding lanes (blockDim rounded to whole warps) shadow the last job
    const double *sx = sdig + (size_t)jlc * (SX + SY), *sy = sx + SX;
    const int *ex = sexp + jlc * 4 * D, *ey = ex + 2 * D;

    // exponent pre-pass (split over the F lanes, max-reduced by shuffles):
    // anchors e_acc of (k1, k2) x (re, im) over ALL terms of each output
    int ea1r = ZERO_E, ea1i = ZERO_E, ea2r = ZERO_E, ea2i = ZERO_E;
    if (NP == 2) {  // one part per thread: only its own anchors
        const int *ey1 = ey + pl * D, *ey2 = ey + (1 - pl) * D;
        for (int j = f; j <= D; j += F) {
            const bool first = j <= t;
            const int i = first ? j : D - j;  // the pass's term order (conv_dig_pass)
            const int kk = first ? t - j : j - t - 1;
            const int e = max(ex[i] + ey1[kk], ex[D + i] + ey2[kk]);
            if (first) ea1r = max(ea1r, e);
            else ea2r = max(ea2r, e);
        }
        ea1i = ea1r;
        ea2i = ea2r;
    } else {
        for (int j = f; j <= D; j += F) {
            const bool first = j <= t;
            const int i = first ? j : D - j;  // the pass's term order (conv_dig_pass)
            const int kk = first ? t - j : j - t - 1;
            const int xr = ex[i], xi = REAL ? ZERO_E : ex[D + i], yr = ey[kk], yi = REAL ? ZERO_E : ey[D + kk];
            const int er = max(xr + yr, xi + yi), ei = max(xr + yi, xi + yr);
            if (first) {
                ea1r = max(ea1r, er);
                ea1i = max(ea1i, ei);
            } else {
                ea2r = max(ea2r, er);
                ea2i = max(ea2i, ei);
            }
        }
    }
    for (int off = F >> 1; off > 0; off >>= 1) {
        ea1r = max(ea1r, __shfl_xor_sync(0xffffffffu, ea1r, off));
        ea1i = max(ea1i, __shfl_xor_sync(0xffffffffu, ea1i, off));
        ea2r = max(ea2r, __shfl_xor_sync(0xffffffffu, ea2r, off));
        ea2i = max(ea2i, __shfl_xor_sync(0xffffffffu, ea2i, off));
    }
    ea1r = max(ea1r, ZERO_E);
    ea1i = max(ea1i, ZERO_E);
    ea2r = max(ea2r, ZERO_E);
    ea2i = max(ea2i, ZERO_E);

    double *park = spark + (size_t)threadIdx.x * PSTR;
    const int job = job0 + jl;
    const bool writer = jl < P && job < njobs;
    double *zd = dpool;
    int *ze = epool;
    double *zl = nullptr;  // limb output (the series is summed by the addition jobs)
    int wdig = 0;          // digit output (the series is a product input)
    if (writer) {
        const int out = jobs[4 * job + 2];
        const int code = jobs[4 * job + 3];
        zd = dpool + (size_t)out * dig_slot_stride(S, D);
        ze = epool + (size_t)out * 2 * D;
        wdig = code & 1;
        if (code & 2) zl = lpool + (size_t)(code >> 2) * 2 * L * D;
    }
    const int k1 = t, k2 = D - 1 - t;
    if (REAL && zl) {  // real system: the imaginary limbs of the outputs are exactly 0
        if (F == 1 || f < 2)
            for (int p = 0; p < L; p++) {
                if (F == 1 || f == 0) zl[(L + p) * D + k1] = 0.0;
                if (F == 1 || f == 1) zl[(L + p) * D + k2] = 0.0;
            }
    }
#pragma unroll 1
    for (int part = pl; part < (REAL ? 1 : (NP == 2 ? pl + 1 : 2)); part++) {
        double A[S];
        const int e1 = part ? ea1i : ea1r, e2 = part ? ea2i : ea2r;
        conv_dig_pass<L, DT, REAL>(sx, sy, ex, ey, D, part, t, f, F, e1, e2, A, park);
        // k1: every lane carries its parked (raw) partial — warp-uniform work,
        // no lane sums alone — and takes it off A, which leaves the k2 partial
        // (|digit| <= R + 2^32: exact)
        double B[S];
#pragma unroll
        for (int s = 0; s < S; s++) B[s] = park[s];
        carry_pass(B);
#pragma unroll
        for (int s = 0; s < S; s++) A[s] = __dsub_rn(A[s], B[s]);
        // k2: sum the F lanes' partials (exact) with shuffles; every lane has it
        for (int off = F >> 1; off > 0; off >>= 1) {
#pragma unroll
            for (int s = 0; s < S; s++) A[s] = __dadd_rn(A[s], __shfl_xor_sync(0xffffffffu, A[s], off));
        }
        // k1: the same shuffle reduction
        for (int off = F >> 1; off > 0; off >>= 1) {
#pragma unroll
            for (int s = 0; s < S; s++) B[s] = __dadd_rn(B[s], __shfl_xor_sync(0xffffffffu, B[s], off));
        }
        __syncwarp();  // parked partials consumed before the emit scratch reuses them
        if (F == 1) {
            if (writer && k2 != k1) conv_dig_emit<L>(A, e2, wdig ? zd : nullptr, ze, zl, D, k2, part, park);
            if (writer) conv_dig_emit<L>(B, e1, wdig ? zd : nullptr, ze, zl, D, k1, part, park);
        } else if (writer && f < 2 && (f == 0 || k2 != k1)) {
            // lanes 0 and 1 emit k1 and k2 in one (lane-dependent) call
            if (f == 0) {
#pragma unroll
                for (int s = 0; s < S; s++) A[s] = B[s];
            }
            conv_dig_emit<L>(A, f == 0 ? e1 : e2, wdig ? zd : nullptr, ze, zl, D, f == 0 ? k1 : k2, part, park);
        }
        __syncwarp();
    }
}

}  // namespace mdps
