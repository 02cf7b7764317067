// conv_dig.cuh — the product-job kernel on digit planes (MDPS_ALGO_DIGITS):
// z = x * y mod t^D for every job of one DAG level.
//
// See kernels_dig.cuh for the digit representation (pool slot: digits
// [S][D][2] — digit, coefficient, part — and one exponent per complex
// coefficient, both parts on one grid).  Mapping:
//  * P jobs per block; per job T = ceil(D/2) output pairs x F splits, and
//    per part one lane set (NP = 2 part lanes for complex systems, one for
//    real ones).  The block's threads are [part][job][pair t][lane f] with
//    each part's set padded to whole warps, so a warp computes ONE part and
//    runs that part's code copy (no per-row selects or sign flips).  Thread
//    (part, t, f) owns outputs k1 = t and k2 = D-1-t — the folded triangle
//    has exactly D+1 terms per pair, so no lane idles — and the fold
//    iterations j = f, f+F, ... (the F lanes of a pair are adjacent lanes).
//  * Per term x_i y_{k-i} the S (re, im) digit pairs of x_i are held in
//    registers (one 16-byte load each) and y's digit rows stream from shared
//    memory, one 16-byte (re, im) pair per row feeding both real products of
//    the part: re += xr yr - xi yi, im += xr yi + xi yr.  Per digit pair one
//    DFMA (exact: integer digits).
//  * Alignment: a term whose exponent (one per complex coefficient) is delta
//    digits below the accumulator anchor reads y's digit row l - delta.
//    Shared memory holds PADZ zero rows in front of y's rows, so for delta
//    <= PADZ (the common case, checked warp-uniformly) every load is base +
//    compile-time offset; larger shifts take a select-based path.  A term
//    with a zero operand is read at delta = 0 (its product is zero anyway).
//  * Partials: a copy of the k1 partial is parked in shared memory when a
//    lane crosses the fold (lanes cross at different iterations) and the k2
//    terms go on top of it; k2 = A - park after the loop.  The F lanes'
//    partials are added with warp shuffles.  All additions are exact
//    (integer digits).
//  * Output digits: the two parts of a coefficient share the exponent of
//    the larger: each part lane finds its leading digit, the part lanes
//    exchange it through shared memory (one block barrier), and both store
//    on the common grid.
//  * Shared memory per job: x [S][D][2] (the pool's own layout, one TMA bulk
//    copy), y [PADZ + S][D][2] (PADZ zero rows in front, one bulk copy),
//    exponents [2][D]; per thread a parking slot of S + 2 doubles; the
//    leading-digit exchange [2][P][D][2] ints.
#pragma once
#include "kernels_dig.cuh"

namespace mdps {

constexpr int PADZ = 4;

__host__ __device__ inline size_t conv_dig_smem(int S, int D, int P, int threads) {
    const size_t per_job = (size_t)2 * S * D + (size_t)2 * (PADZ + S) * D;  // doubles
    return (size_t)P * per_job * sizeof(double) + (size_t)threads * (S + 2) * sizeof(double) +
           (size_t)P * 2 * D * sizeof(int) + (size_t)2 * P * D * 2 * sizeof(int) +
           (size_t)P * (2 * D + 4) * sizeof(int) + 16;  // + anchor exchange, mbarrier
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

// programmatic dependent launch (griddepcontrol): no-ops in a launch without
// the programmatic-serialization attribute
__device__ __forceinline__ void grid_dep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// one product pass over this thread's fold iterations for part PART (0: re,
// 1: im).  REAL: real series (imaginary digits zero and never read): one
// product per term.
template <int L, int DT, int PART, bool REAL = false>
__device__ __forceinline__ void conv_dig_pass(const double *__restrict__ sx, const double *__restrict__ sy,
                                              const int *__restrict__ ex, const int *__restrict__ ey, int Drt,
                                              int t, int f, int F, int eacc1, int eacc2, double (&A)[digits_for(L)],
                                              double *park) {
    constexpr int S = digits_for(L);
    constexpr int NORM = norm_every(S);
    const int D = DT > 0 ? DT : Drt;
    const int D2 = 2 * D;  // doubles per digit row
    md_zero(A);
    bool switched = false;
    // Software pipeline, one term ahead.  Everything the next term needs
    // (its x digits, its y offset kk and its alignment shift d, read from
    // the exponents) is prepared INSIDE the current term's body, where the
    // integer work and the shared-memory latency hide behind the DFMAs:
    // after digit row l the operand digit u = S-1-l has had its last use, so
    // its registers take the next term's digit u (no extra registers).  The
    // per-term preamble shrinks to the warp vote on the fast path.
    // fold iteration j -> term (i, kk = k - i): j <= t is term i = j of k1 = t,
    // j > t is term i = D - j of k2 = D-1-t (descending), so the x index is
    // j or D - j — the same for every pair of the warp at a given j (a
    // shared-memory broadcast) — and kk = t - j or j - t - 1 is consecutive
    // over the warp's pairs (one contiguous window), for both outputs
    auto term_index = [&](int j) { return j <= t ? j : D - j; };
    auto term_meta = [&](int j, int &kk, int &d) {
        const bool first = j <= t;
        const int i = term_index(j);
        kk = first ? t - j : j - t - 1;
        const int e = ex[i] + ey[kk];
        d = e <= ZERO_E / 2 ? 0 : (first ? eacc1 : eacc2) - e;  // zero product: any row will do
    };
    double Ur[S], Ui[S];
    auto load_x = [&](const double *ux, int u) {
        if (REAL) {
            Ur[u] = ux[u * D2];
        } else {
            const double2 v = *reinterpret_cast<const double2 *>(ux + u * D2);
            Ur[u] = v.x;
            Ui[u] = v.y;
        }
    };
    int kk, d;
    {
        const int j0 = min(f, D);  // a lane with f > D has no terms (clamped reads only)
        term_meta(j0, kk, d);
        const double *ux = sx + 2 * term_index(j0);
#pragma unroll
        for (int u = 0; u < S; u++) load_x(ux, u);
    }
    // every lane of the warp within the PADZ window: voted one term ahead,
    // inside the body (the lanes of the next iteration are among the voters;
    // a lane that drops out votes with its last term's shift, and any lane
    // outside the window only sends the warp down the select path, which is
    // always right)
    // (VA: where measured faster — L = 8: od -0.4%, the L = 8 cells -0.5..3.6%;
    // L = 10: +1.4..2.3%, so there the vote stays at the term's start)
    constexpr bool VA = L == 8;
    bool fast = __all_sync(__activemask(), d <= PADZ);
    // the two real products of digit row l: w = (y re, y im) of that row
    auto row = [&](int l, double wr, double wi) {
#pragma unroll
        for (int u = 0; u < S - l; u++) {
            if (REAL) {
                A[u + l] = __fma_rn(Ur[u], wr, A[u + l]);
            } else if (PART == 0) {
                A[u + l] = __fma_rn(Ur[u], wr, A[u + l]);
                A[u + l] = __fma_rn(-Ui[u], wi, A[u + l]);
            } else {
                A[u + l] = __fma_rn(Ur[u], wi, A[u + l]);
                A[u + l] = __fma_rn(Ui[u], wr, A[u + l]);
            }
        }
    };
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
        const double *uxn = sx + 2 * term_index(jn);
        int kkn, dn;
        bool fastn = false;
        auto ahead = [&](int l) {  // called after digit row l of the body
            if (l == 1) term_meta(jn, kkn, dn);
            if (VA && l == 2) fastn = __all_sync(__activemask(), dn <= PADZ);
            load_x(uxn, S - 1 - l);
        };
        if (!VA) fast = __all_sync(__activemask(), d <= PADZ);
        if (fast) {
            const double *W = sy + (PADZ - d) * D2 + 2 * kk;
            // software pipelined: row l+1's digit pair loads while row l's FMAs run
            double2 w = REAL ? make_double2(W[0], 0.0) : *reinterpret_cast<const double2 *>(W);
#pragma unroll
            for (int l = 0; l < S; l++) {
                double2 wn = make_double2(0.0, 0.0);
                if (l + 1 < S)
                    wn = REAL ? make_double2(W[(l + 1) * D2], 0.0)
                              : *reinterpret_cast<const double2 *>(W + (l + 1) * D2);
                row(l, w.x, w.y);
                ahead(l);
                w = wn;
            }
        } else {
            const double *W = sy + 2 * kk;
#pragma unroll
            for (int l = 0; l < S; l++) {
                double2 w = make_double2(0.0, 0.0);
                if (l >= d)
                    w = REAL ? make_double2(W[(PADZ + l - d) * D2], 0.0)
                             : *reinterpret_cast<const double2 *>(W + (PADZ + l - d) * D2);
                row(l, w.x, w.y);
                ahead(l);
            }
        }
        kk = kkn;
        d = dn;
        fast = fastn;
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

// Z = [c2, c1, c0, A_1 .. A_{S-1}] of a balanced accumulator (Z_u has weight
// R^(eacc - u)) into shared memory; returns the index of its first nonzero
// entry (S + 2 if none)
template <int S>
__device__ __forceinline__ int conv_dig_z(const double (&A)[S], double *scratch) {
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
    return z0;
}

// The work of one block: P product jobs starting at job0.  NP = 2: complex
// (part lanes), NP = 1: REAL systems.
template <int L, int DT, bool REAL>
__device__ __forceinline__ void conv_dig_block(double *__restrict__ dpool, int *__restrict__ epool,
                                               double *__restrict__ lpool, const int *__restrict__ jobs, int job0,
                                               int njobs, int Drt, int T, int F, int P, double *sm) {
    constexpr int S = digits_for(L);
    constexpr int NP = REAL ? 1 : 2;
    const int D = DT > 0 ? DT : Drt;
    const int SX = 2 * S * D, SY = 2 * (PADZ + S) * D;
    const int half = (P * T * F + 31) / 32 * 32;               // threads per part lane set
    double *sdig = sm;                                        // [P][SX + SY]
    double *spark = sm + (size_t)P * (SX + SY);               // [threads][S + 2]
    constexpr int PSTR = S + 2;                               // parking / emit scratch slot
    int *sexp = (int *)(spark + (size_t)blockDim.x * PSTR);   // [P][2 series][D]
    int *szx = sexp + (size_t)P * 2 * D;                      // [2 rounds][P][D][2 parts]
    int *sanc = szx + (size_t)2 * P * D * 2;                  // [P][T][2 outputs][2 parts]
    uint64_t *bar = reinterpret_cast<uint64_t *>(sanc + (size_t)P * (2 * D + 4));

    // stage: x -> [S][D][2] (the pool layout), y -> [PADZ + S][D][2] behind
    // PADZ zero rows: two 16-byte aligned contiguous runs per job (every
    // slot and row is a multiple of 16 bytes), so one thread issues two TMA
    // bulk copies (cp.async.bulk) per job against an mbarrier while the
    // other warps write the zero rows and exponents
    // programmatic dependent launch: the next level's blocks may be scheduled
    // as this level's blocks drain; nothing a previous launch wrote (digit and
    // exponent pools) is read before grid_dep_wait() — the job list is static
    grid_dep_launch_dependents();
    // (the job table is static: the slot indices this thread needs first —
    // bulk copy c = threadIdx.x, exponent idx = threadIdx.x — are read here,
    // under the zero rows and the wait on the previous launch)
    int copy_slot = 0, exp_slot = 0;
    if (threadIdx.x < 32 && (int)threadIdx.x < 2 * P)
        copy_slot = jobs[4 * min(job0 + ((int)threadIdx.x >> 1), njobs - 1) + (threadIdx.x & 1)];
    if ((int)threadIdx.x < P * 2 * D) {
        const int jl = threadIdx.x / (2 * D), r = threadIdx.x - jl * 2 * D;
        exp_slot = jobs[4 * min(job0 + jl, njobs - 1) + r / D];
    }
    if (threadIdx.x == 0) mbar_init(bar, 1);
    for (int idx = threadIdx.x; idx < P * 2 * PADZ * D; idx += blockDim.x) {  // zero rows
        const int jl = idx / (2 * PADZ * D), r = idx - jl * 2 * PADZ * D;
        sdig[(size_t)jl * (SX + SY) + SX + r] = 0.0;
    }
    grid_dep_wait();
    __syncthreads();
    if (threadIdx.x < 32) {
        if (threadIdx.x == 0) mbar_expect_tx(bar, (unsigned)(P * 2 * SX * 8));
        __syncwarp();
        for (int c = threadIdx.x; c < 2 * P; c += 32) {  // (job, copy): x | y
            const int jl = c >> 1, which = c & 1;
            const int job = min(job0 + jl, njobs - 1);
            double *base = sdig + (size_t)jl * (SX + SY) + (which ? SX + 2 * PADZ * D : 0);
            const int slot = c < 32 ? copy_slot : jobs[4 * job + which];
            bulk_g2s(base, dpool + (size_t)slot * dig_slot_stride(S, D), (unsigned)(SX * 8), bar);
        }
    }
    for (int idx = threadIdx.x; idx < P * 2 * D; idx += blockDim.x) {
        const int jl = idx / (2 * D), r = idx - jl * 2 * D;
        const int which = r / D, k = r - which * D;
        const int job = min(job0 + jl, njobs - 1);
        const int slot = idx < (int)blockDim.x ? exp_slot : jobs[4 * job + which];
        sexp[idx] = epool[(size_t)slot * dig_exp_stride(D) + k];
    }
    __syncthreads();  // exponents staged; the operand digits are still in flight

    const int part = NP == 2 ? (int)threadIdx.x / half : 0;  // warp-uniform (half is whole warps)
    const int r0 = threadIdx.x - part * half;
    const int jl = r0 / (T * F);
    const int r = r0 - jl * T * F;
    const int t = r / F, f = r - t * F;
    const int jlc = min(jl, P - 1);  // padding lanes (sets rounded to whole warps) shadow the last job
    const double *sx = sdig + (size_t)jlc * (SX + SY), *sy = sx + SX;
    const int *ex = sexp + jlc * 2 * D, *ey = ex + D;

    // exponent pre-pass (split over the F lanes, max-reduced by shuffles):
    // anchors e_acc of k1 and k2 over ALL their terms (one exponent per
    // complex coefficient: the same anchors for both parts)
    // complex systems up to L = 8: the two part lanes of a pair take every
    // other term each and exchange their maxima through shared memory (one
    // barrier; measured: od -1.4%, qd -2.6%; at L = 10, two blocks per SM,
    // the barrier costs more than the halved pre-pass saves)
    constexpr int SPLIT = (NP == 2 && L <= 8) ? 2 : 1;
    int ea1 = ZERO_E, ea2 = ZERO_E;
#pragma unroll 2
    for (int j = f + (SPLIT == 2 ? part : 0) * F; j <= D; j += SPLIT * F) {
        const bool first = j <= t;
        const int e = ex[first ? j : D - j] + ey[first ? t - j : j - t - 1];  // the pass's term order
        ea1 = max(ea1, first ? e : ZERO_E);
        ea2 = max(ea2, first ? ZERO_E : e);
    }
    for (int off = F >> 1; off > 0; off >>= 1) {
        ea1 = max(ea1, __shfl_xor_sync(0xffffffffu, ea1, off));
        ea2 = max(ea2, __shfl_xor_sync(0xffffffffu, ea2, off));
    }
    if (SPLIT == 2) {
        if (f == 0 && jl < P) {
            sanc[((jl * T + t) * 2 + 0) * 2 + part] = ea1;
            sanc[((jl * T + t) * 2 + 1) * 2 + part] = ea2;
        }
        __syncthreads();
        ea1 = max(ea1, sanc[((jlc * T + t) * 2 + 0) * 2 + 1 - part]);
        ea2 = max(ea2, sanc[((jlc * T + t) * 2 + 1) * 2 + 1 - part]);
    }
    ea1 = max(ea1, ZERO_E);
    ea2 = max(ea2, ZERO_E);

    mbar_wait(bar, 0);  // operand digits landed (the pre-pass above ran under the bulk copies)

    double *park = spark + (size_t)threadIdx.x * PSTR;
    const int job = job0 + jl;
    const bool writer = jl < P && job < njobs;
    double *zd = nullptr;  // digit output (the series is a product input)
    int *ze = nullptr;
    double *zl = nullptr;  // limb output (the series is summed by the addition jobs)
    if (writer) {
        const int out = jobs[4 * job + 2];
        const int code = jobs[4 * job + 3];
        if (code & 1) {
            zd = dpool + (size_t)out * dig_slot_stride(S, D);
            ze = epool + (size_t)out * dig_exp_stride(D);
        }
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
    double A[S];
    if (part == 0)
        conv_dig_pass<L, DT, 0, REAL>(sx, sy, ex, ey, D, t, f, F, ea1, ea2, A, park);
    else
        conv_dig_pass<L, DT, 1, false>(sx, sy, ex, ey, D, t, f, F, ea1, ea2, A, park);
    // k1: every lane carries its parked (raw) partial — warp-uniform work,
    // no lane sums alone — and takes it off A, which leaves the k2 partial
    // (|digit| <= R + 2^32: exact)
    double B[S];
#pragma unroll
    for (int s = 0; s < S; s++) B[s] = park[s];
    carry_pass(B);
#pragma unroll
    for (int s = 0; s < S; s++) A[s] = __dsub_rn(A[s], B[s]);
    // sum the F lanes' partials of k2 (A) and k1 (B), exact, with shuffles
    for (int off = F >> 1; off > 0; off >>= 1) {
#pragma unroll
        for (int s = 0; s < S; s++) {
            A[s] = __dadd_rn(A[s], __shfl_xor_sync(0xffffffffu, A[s], off));
            B[s] = __dadd_rn(B[s], __shfl_xor_sync(0xffffffffu, B[s], off));
        }
    }
    __syncwarp();  // parked partials consumed before the emit scratch reuses them
    // emit: F = 1 — every lane emits k2 (round 0) then k1 (round 1); F >= 2 —
    // lane f = 0 emits k1, lane f = 1 emits k2 (one round).  Per round: the
    // accumulator balanced (two carry passes: partial sums of <= 8 lanes),
    // its Z vector parked, the leading digit exchanged with the other part
    // lane of the output (block barrier), then digits on the common grid
    // and/or limbs.
    const int rounds = F == 1 ? 2 : 1;
    for (int rd = 0; rd < rounds; rd++) {
        const bool use_b = F == 1 ? rd == 1 : f == 0;
        const int k = use_b ? k1 : k2;
        const int eacc = use_b ? ea1 : ea2;
        const bool mine = writer && (F == 1 || f < 2) && (use_b || k2 != k1);
        double Z[S];
#pragma unroll
        for (int s = 0; s < S; s++) Z[s] = use_b ? B[s] : A[s];
        carry_pass(Z);
        carry_pass(Z);
        const int z0 = conv_dig_z<S>(Z, park);
        int *zx = szx + (size_t)rd * P * D * 2;
        if (NP == 2 && mine) zx[(jl * D + k) * 2 + part] = z0;
        if (NP == 2) __syncthreads();
        if (mine) {
            if (zd) {  // digits on the grid of the larger part
                const int zc = NP == 2 ? min(z0, zx[(jl * D + k) * 2 + 1 - part]) : z0;
                const int e = (zc >= S + 2 || eacc <= ZERO_E / 2) ? ZERO_E : eacc + 1 - zc;
                const double *src = park + zc;
                const int avail = S + 2 - zc;
#pragma unroll
                for (int s = 0; s < S; s++) zd[((size_t)s * D + k) * 2 + part] = (s < avail && e != ZERO_E) ? src[s] : 0.0;
                if (part == 0) ze[k] = e;
            }
            if (zl) {  // limbs for the addition jobs: the exact accumulator rounded to L limbs
                double out[L];
                digits_to_limbs<L, S, true>(Z, eacc - 1, out);  // Z_t has weight R^(eacc-2-t); consumes Z
#pragma unroll
                for (int p = 0; p < L; p++) zl[(part * L + p) * D + k] = out[p];
            }
        }
        __syncwarp();  // the scratch is free again before the next round parks into it
    }
}

template <int L, int DT, bool REAL = false>
// register budget per SM: 4 blocks of 128 up to L = 4 (<= 128 registers),
// 3 up to L = 8 (<= 170), 2 above; 256-thread blocks for D = 128 and the
// generic-D build.  REAL: real systems (mdps_options.real): only the real
// part is computed; the imaginary limbs of the limb outputs are written as 0.
__global__ void __launch_bounds__(DT == 128 || DT == 0 ? 256 : 128,
                                  DT == 128 || DT == 0 ? 1 : (L <= 4 ? 4 : (L <= 8 ? 3 : 2)))
    conv_dig_kernel(double *__restrict__ dpool, int *__restrict__ epool, double *__restrict__ lpool,
                    const int *__restrict__ jobs, int njobs, int Drt, int T, int F, int P) {
    extern __shared__ __align__(16) double sm[];
    conv_dig_block<L, DT, REAL>(dpool, epool, lpool, jobs, blockIdx.x * P, njobs, Drt, T, F, P, sm);
}

}  // namespace mdps
