// conv_dig_fused.cuh — the product-job kernel on digit planes with BOTH parts
// of an output on one thread (complex systems, small digit counts):
// z = x * y mod t^D for every job of one DAG level.
//
// Same representation, staging, fold, alignment and exact accumulation as
// conv_dig.cuh (read that header first).  What differs: conv_dig_kernel gives
// each part (re, im) of an output pair its own lane, so the two part lanes
// load the same x digits (registers) and y digit rows (shared memory) and
// each issue two DFMAs per loaded digit pair.  At S <= 14 digits (L <= 5) a
// term is short — S(S+1) DFMAs for 2S 16-byte loads per part lane — and the
// shared-memory pipe is the co-limit (~3 wavefronts per 16-byte
// load, 92% of its bandwidth at a full FP64 pipe at S = 12).  Here one thread
// keeps the accumulators of both parts (2S doubles) next to the x digits (2S)
// and issues all four DFMAs of a digit pair from one x load and one y load:
//     re += xr yr - xi yi,   im += xr yi + xi yr
// — half the shared-memory traffic, half the per-term code (pre-pass, fold
// crossing, fast-path vote) and half the operand registers per DFMA, and no
// exchange between part lanes (the common output exponent and the anchors
// are thread-local).  At S = 21, 26 the 4S doubles do not fit the register
// file at a useful occupancy, so L >= 8 stays on conv_dig_kernel (a build
// that re-read the x digits from shared memory at every use instead of
// holding them — 2S doubles per thread — was 1.6x (od) to 3.5x (deca) slower:
// DESIGN.md §7.4).
//
// Threads of a block: [job][pair t][lane f], padded to whole warps.  Shared
// memory per job as in conv_dig.cuh.  Parking at the fold and the emit
// scratch: LPARK = false — a per-thread shared-memory slot of PS (re, im)
// pairs, PS = S + 2 rounded up to odd (16-byte accesses at an odd multiple of
// 16 bytes between lanes are bank-conflict free); LPARK = true (the default
// wherever measured faster, libmdps.cu fused_lpark_default) — the parked
// partial in local memory and the emit scratch in the job's own operand
// buffers, so that the operand buffers alone set the resident blocks.
#pragma once
#include "conv_dig.cuh"

namespace mdps {

__host__ __device__ constexpr int fused_park_slot(int S) { return (S + 2) | 1; }  // double2 entries

// lpark: the fold parks in local memory and the emit scratch reuses the job's
// operand buffers (no per-thread shared-memory slot)
__host__ __device__ inline size_t conv_fused_smem(int S, int D, int P, int threads, bool lpark = false) {
    const size_t per_job = (size_t)2 * S * D + (size_t)2 * (PADZ + S) * D;  // doubles
    return (size_t)P * per_job * sizeof(double) +
           (lpark ? 0 : (size_t)threads * fused_park_slot(S) * 2 * sizeof(double)) +
           (size_t)P * 2 * D * sizeof(int) + 16;  // + exponents, mbarrier
}

// one pass over this thread's fold iterations, both parts.  On return: park =
// the k1 partials (raw, |digit| < 2^53), (Ar, Ai) = the k1 + k2 partials
// (carried).
// park(s, v): stores entry s of the parked k1 partial.
template <int L, int DT, bool PRE, class ParkFn>
__device__ __forceinline__ void conv_fused_pass(const double *__restrict__ sx, const double *__restrict__ sy,
                                                const int *__restrict__ ex, const int *__restrict__ ey, int Drt,
                                                int t, int f, int F, int eacc1, int eacc2,
                                                double (&Ar)[digits_for(L)], double (&Ai)[digits_for(L)],
                                                ParkFn park) {
    constexpr int S = digits_for(L);
    constexpr int NORM = norm_every(S);
    const int D = DT > 0 ? DT : Drt;
    const int D2 = 2 * D;  // doubles per digit row
    md_zero(Ar);
    md_zero(Ai);
    bool switched = false;
    // term order, software pipeline and fast path: as conv_dig_pass
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
        const double2 v = *reinterpret_cast<const double2 *>(ux + u * D2);
        Ur[u] = v.x;
        Ui[u] = v.y;
    };
    // Row 0 of the NEXT term's y operand is loaded inside the current body too
    // (at row PF, once the next term's offset and shift are known): at S <= 14 a
    // body is short and the first DFMA of every term otherwise waits out that
    // load (ncu at qd: 10% of the kernel's stall samples on that one
    // instruction).  The row is read through the fast-path base with the shift
    // clamped to PADZ, which is also the right value on the select path: a
    // lane with d > PADZ reads a zero row there, as its row 0 must be.
    // PRE = false (the shared-memory-slot build, kept for L = 5 at degree 127,
    // where the prefetch measured +3.9%): row 0 is loaded at the term's start.
    constexpr int PF = S > 6 ? S - 5 : 2;
    auto fast_base = [&](int kk_, int d_) { return sy + (PADZ - min(d_, PADZ)) * D2 + 2 * kk_; };
    int kk, d;
    const double *Wf;  // y's digit row 0 moved down by min(d, PADZ) rows
    double2 w0;        // its (re, im) pair
    // every lane of the warp within the PADZ window: voted one term ahead,
    // inside the body (the lanes of the next iteration are among the voters;
    // a lane that drops out votes with its last term's shift, and any lane
    // outside the window only sends the warp down the select path, which is
    // always right)
    // (VA: where measured faster — L = 3: -0.7..2.3%; L = 5: +0.5..2.8%, L = 4:
    // +-0.5%, so there the vote stays at the term's start)
    constexpr bool VA = L == 3;
    bool fast;
    {
        const int j0 = min(f, D);  // a lane with f > D has no terms (clamped reads only)
        term_meta(j0, kk, d);
        Wf = fast_base(kk, d);
        w0 = *reinterpret_cast<const double2 *>(Wf);
        fast = __all_sync(__activemask(), d <= PADZ);
        const double *ux = sx + 2 * term_index(j0);
#pragma unroll
        for (int u = 0; u < S; u++) load_x(ux, u);
    }
    // the four real products of digit row l: w = (y re, y im) of that row
    auto row = [&](int l, double wr, double wi) {
#pragma unroll
        for (int u = 0; u < S - l; u++) {
            Ar[u + l] = __fma_rn(Ur[u], wr, Ar[u + l]);
            Ai[u + l] = __fma_rn(Ur[u], wi, Ai[u + l]);
            Ar[u + l] = __fma_rn(-Ui[u], wi, Ar[u + l]);
            Ai[u + l] = __fma_rn(Ui[u], wr, Ai[u + l]);
        }
    };
    for (int j = f; j <= D;) {
        const int jstop = min(D, j + (NORM - 1) * F);
        for (; j <= jstop; j += F) {
            if (j > t && !switched) {  // k1 partial complete: park a copy (raw), keep accumulating
                switched = true;
#pragma unroll
                for (int s = 0; s < S; s++) park(s, make_double2(Ar[s], Ai[s]));
            }
            const int jn = j + F <= D ? j + F : j;
            const double *uxn = sx + 2 * term_index(jn);
            int kkn, dn;
            const double *Wfn;
            double2 w0n = make_double2(0.0, 0.0);
            bool fastn = false;
            auto ahead = [&](int l) {  // called after digit row l of the body
                if (l == 1) {
                    term_meta(jn, kkn, dn);
                    Wfn = fast_base(kkn, dn);
                }
                if (VA && l == 2) fastn = __all_sync(__activemask(), dn <= PADZ);
                if (PRE && l == PF) w0n = *reinterpret_cast<const double2 *>(Wfn);
                load_x(uxn, S - 1 - l);
            };
            if (!VA) fast = __all_sync(__activemask(), d <= PADZ);
            if (fast) {
                const double *W = Wf;
                if (!PRE) w0 = *reinterpret_cast<const double2 *>(Wf);
                double2 w = w0;
#pragma unroll
                for (int l = 0; l < S; l++) {
                    double2 wn = make_double2(0.0, 0.0);
                    if (l + 1 < S) wn = *reinterpret_cast<const double2 *>(W + (l + 1) * D2);
                    row(l, w.x, w.y);
                    ahead(l);
                    w = wn;
                }
            } else {
                const double *W = sy + 2 * kk;
                if (!PRE) w0 = *reinterpret_cast<const double2 *>(Wf);
#pragma unroll
                for (int l = 0; l < S; l++) {
                    double2 w = l == 0 ? w0 : make_double2(0.0, 0.0);
                    if (l > 0 && l >= d) w = *reinterpret_cast<const double2 *>(W + (PADZ + l - d) * D2);
                    row(l, w.x, w.y);
                    ahead(l);
                }
            }
            kk = kkn;
            d = dn;
            Wf = Wfn;
            w0 = w0n;
            fast = fastn;
        }
        carry_pass(Ar);
        carry_pass(Ai);
    }
    if (!switched) {  // no k2 iterations on this lane: everything belongs to k1
#pragma unroll
        for (int s = 0; s < S; s++) park(s, make_double2(Ar[s], Ai[s]));
    }
}

// Z = [c2, c1, c0, A_1 .. A_{S-1}] of one part of a balanced accumulator into
// the .x (PART 0) or .y (PART 1) halves of the scratch pairs; returns the
// index of its first nonzero entry (S + 2 if none)
template <int S, int PART>
__device__ __forceinline__ int conv_fused_z(const double (&A)[S], double2 *scratch) {
    double *sc = reinterpret_cast<double *>(scratch) + PART;
    double a0 = A[0];
    const double c2 = rint_magic(__dmul_rn(a0, INV_RADIX * INV_RADIX));
    a0 = __fma_rn(-c2, RADIX * RADIX, a0);
    const double c1 = rint_magic(__dmul_rn(a0, INV_RADIX));
    const double c0 = __fma_rn(-c1, RADIX, a0);
    sc[0] = c2;
    sc[2] = c1;
    sc[4] = c0;
    int z0 = S + 2;
#pragma unroll
    for (int s = S - 1; s >= 1; s--) {
        sc[2 * (s + 2)] = A[s];
        if (A[s] != 0.0) z0 = s + 2;
    }
    if (c0 != 0.0) z0 = 2;
    if (c1 != 0.0) z0 = 1;
    if (c2 != 0.0) z0 = 0;
    return z0;
}

// LPARK: the parked k1 partial goes to LOCAL memory (a per-thread array
// indexed through a run-time zero, so it is not promoted to registers; written
// once at the fold and read once after the loop, through L1/L2) and the emit
// scratch reuses the job's operand buffers once all of the job's lanes have
// finished their pass — no per-thread shared-memory slot, so the operand
// buffers alone set the resident blocks (qd: 7 instead of 5 blocks of two
// jobs per SM).
template <int L, int DT, bool LPARK>
__device__ __forceinline__ void conv_fused_block(double *__restrict__ dpool, int *__restrict__ epool,
                                                 double *__restrict__ lpool, const int *__restrict__ jobs, int job0,
                                                 int njobs, int Drt, int T, int F, int P, double *sm) {
    constexpr int S = digits_for(L);
    constexpr int PS = fused_park_slot(S);
    const int D = DT > 0 ? DT : Drt;
    const int SX = 2 * S * D, SY = 2 * (PADZ + S) * D;
    double *sdig = sm;                                                  // [P][SX + SY]
    double2 *spark = reinterpret_cast<double2 *>(sm + (size_t)P * (SX + SY));  // [threads][PS] (not LPARK)
    int *sexp = (int *)(spark + (LPARK ? 0 : (size_t)blockDim.x * PS));  // [P][2 series][D]
    uint64_t *bar = reinterpret_cast<uint64_t *>(sexp + (size_t)P * 2 * D);

    // stage (as conv_dig_block): two TMA bulk copies per job against an
    // mbarrier while the other threads write the zero rows and exponents
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

    const int jl = threadIdx.x / (T * F);
    const int r = threadIdx.x - jl * T * F;
    const int t = r / F, f = r - t * F;
    const int jlc = min(jl, P - 1);  // padding lanes (block rounded to whole warps) shadow the last job
    const double *sx = sdig + (size_t)jlc * (SX + SY), *sy = sx + SX;
    const int *ex = sexp + jlc * 2 * D, *ey = ex + D;

    // exponent pre-pass (split over the F lanes, max-reduced by shuffles):
    // anchors e_acc of k1 and k2 over ALL their terms
    int ea1 = ZERO_E, ea2 = ZERO_E;
#pragma unroll 2
    for (int j = f; j <= D; j += F) {
        const bool first = j <= t;
        const int e = ex[first ? j : D - j] + ey[first ? t - j : j - t - 1];  // the pass's term order
        ea1 = max(ea1, first ? e : ZERO_E);
        ea2 = max(ea2, first ? ZERO_E : e);
    }
    for (int off = F >> 1; off > 0; off >>= 1) {
        ea1 = max(ea1, __shfl_xor_sync(0xffffffffu, ea1, off));
        ea2 = max(ea2, __shfl_xor_sync(0xffffffffu, ea2, off));
    }

    mbar_wait(bar, 0);  // operand digits landed (the pre-pass above ran under the bulk copies)

    double2 *park = LPARK ? nullptr : spark + (size_t)threadIdx.x * PS;  // parking + emit scratch slot
    double2 lpark[LPARK ? S : 1];
    const int zero = Drt >> 30;  // 0 at run time (D <= 128), unknown to the compiler
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
    double Ar[S], Ai[S];
    conv_fused_pass<L, DT, LPARK>(sx, sy, ex, ey, D, t, f, F, ea1, ea2, Ar, Ai, [&](int s, double2 v) {
        if (LPARK) lpark[s + zero] = v;
        else park[s] = v;
    });
    // k1: every lane carries its parked (raw) partial and takes it off A,
    // which leaves the k2 partial (|digit| <= R + 2^32: exact)
    double Br[S], Bi[S];
#pragma unroll
    for (int s = 0; s < S; s++) {
        const double2 v = LPARK ? lpark[s + zero] : park[s];
        Br[s] = v.x;
        Bi[s] = v.y;
    }
    carry_pass(Br);
    carry_pass(Bi);
#pragma unroll
    for (int s = 0; s < S; s++) {
        Ar[s] = __dsub_rn(Ar[s], Br[s]);
        Ai[s] = __dsub_rn(Ai[s], Bi[s]);
    }
    // sum the F lanes' partials (exact) with shuffles; afterwards lane f = 0
    // keeps k1 and the others k2 in (Ar, Ai) — F = 1 keeps both and emits
    // k2 then k1
    for (int off = F >> 1; off > 0; off >>= 1) {
#pragma unroll
        for (int s = 0; s < S; s++) {
            Ar[s] = __dadd_rn(Ar[s], __shfl_xor_sync(0xffffffffu, Ar[s], off));
            Ai[s] = __dadd_rn(Ai[s], __shfl_xor_sync(0xffffffffu, Ai[s], off));
            Br[s] = __dadd_rn(Br[s], __shfl_xor_sync(0xffffffffu, Br[s], off));
            Bi[s] = __dadd_rn(Bi[s], __shfl_xor_sync(0xffffffffu, Bi[s], off));
        }
    }
    if (F > 1 && f == 0) {
#pragma unroll
        for (int s = 0; s < S; s++) {
            Ar[s] = Br[s];
            Ai[s] = Bi[s];
        }
    }
    bool emits = true;
    if (LPARK) {
        // the emit scratch of lane (t, f < 2) lies in its job's operand
        // buffers: every lane of the job must be done with them (a job's lanes
        // share a warp, or the block holds whole jobs only)
        if (T * F <= 32 && 32 % (T * F) == 0) __syncwarp();
        else __syncthreads();
        emits = jl < P && (F == 1 || f < 2);
        park = reinterpret_cast<double2 *>(sdig + (size_t)jlc * (SX + SY)) + (size_t)(F == 1 ? t : 2 * t + f) * PS;
    } else {
        __syncwarp();  // parked partials consumed before the emit scratch reuses them
    }
    const int rounds = F == 1 ? 2 : 1;
    for (int rd = 0; rd < rounds; rd++) {
        const bool is_k1 = F == 1 ? rd == 1 : f == 0;
        if (rd == 1) {
#pragma unroll
            for (int s = 0; s < S; s++) {
                Ar[s] = Br[s];
                Ai[s] = Bi[s];
            }
        }
        const int k = is_k1 ? k1 : k2;
        const int eacc = max(is_k1 ? ea1 : ea2, ZERO_E);
        const bool mine = writer && (F == 1 || f < 2) && (is_k1 || k2 != k1);
        int z0r = S + 2, z0i = S + 2;
        if (emits) {
            carry_pass(Ar);
            carry_pass(Ar);
            carry_pass(Ai);
            carry_pass(Ai);
            z0r = conv_fused_z<S, 0>(Ar, park);
            z0i = conv_fused_z<S, 1>(Ai, park);
        }
        if (mine) {
            if (zd) {  // digits of both parts on the grid of the larger part
                const int zc = min(z0r, z0i);
                const int e = (zc >= S + 2 || eacc <= ZERO_E / 2) ? ZERO_E : eacc + 1 - zc;
                const double2 *src = park + zc;
                const int avail = S + 2 - zc;
#pragma unroll
                for (int s = 0; s < S; s++) {
                    double2 v = make_double2(0.0, 0.0);
                    if (s < avail && e != ZERO_E) v = src[s];
                    *reinterpret_cast<double2 *>(zd + ((size_t)s * D + k) * 2) = v;
                }
                ze[k] = e;
            }
            if (zl) {  // limbs for the addition jobs: the exact accumulators rounded to L limbs
                double out[L];
                digits_to_limbs<L, S, true>(Ar, eacc - 1, out);  // Z_t has weight R^(eacc-2-t); consumes Ar
#pragma unroll
                for (int p = 0; p < L; p++) zl[p * D + k] = out[p];
                digits_to_limbs<L, S, true>(Ai, eacc - 1, out);
#pragma unroll
                for (int p = 0; p < L; p++) zl[(L + p) * D + k] = out[p];
            }
        }
        __syncwarp();  // the scratch is free again before the next round parks into it
    }
}

// register budget per SM: 128-thread blocks, 4 resident up to S = 10 (<= 128
// registers), 3 above (<= 168); 256-thread blocks for D = 128 and the
// generic-D build
template <int L, int DT, bool LPARK = false>
__global__ void __launch_bounds__(DT == 128 || DT == 0 ? 256 : 128, DT == 128 || DT == 0 ? 1 : (L <= 3 ? 4 : 3))
    conv_fused_kernel(double *__restrict__ dpool, int *__restrict__ epool, double *__restrict__ lpool,
                      const int *__restrict__ jobs, int njobs, int Drt, int T, int F, int P) {
    static_assert(L <= 5, "the fused-parts kernel holds 4 S doubles per thread: L <= 5");
    extern __shared__ __align__(16) double sm[];
    conv_fused_block<L, DT, LPARK>(dpool, epool, lpool, jobs, blockIdx.x * P, njobs, Drt, T, F, P, sm);
}

}  // namespace mdps
