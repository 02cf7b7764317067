// conv_quad.cuh — product-job kernel variant for small digit counts
// (MDPS_CONV_KERNEL=3; complex systems, D a multiple of 4): two output
// coefficients per lane and phase share the x operand.
//
// Same digit representation, staging, alignment and carry scheme as
// conv_dig.cuh; what changes is the mapping.  Quad q of a job owns the four
// outputs {2q, 2q+1} (low phase, terms i = 0..2q+1) and {D-2-2q, D-1-2q}
// (high phase, terms i = 0..D-1-2q): D+2 term slots per quad, every quad the
// same (the folded triangle, two outputs at a time).  At term i of a phase
// with outputs a (the larger) and b = a-1 the lane forms x_i y_{a-i} -> A_a
// and x_i y_{a-1-i} -> A_b: the 2S x digits held in registers feed twice the
// DFMAs, so a term costs 2S x loads + 4S y loads for 2 S(S+1) DFMAs instead of
// 4S loads for S(S+1) — at small S (L <= 5) the digit kernel is bound by
// these loads and by the per-term work, not by the FP64 pipe.
//
// This file shares no code with the CPU oracle (oracle/).
#pragma once
#include "conv_dig.cuh"

namespace mdps {

__host__ __device__ inline size_t conv_q_smem(int S, int D, int P, int threads) {
    const size_t per_job = (size_t)2 * S * D + (size_t)2 * (PADZ + S) * D;  // doubles
    return (size_t)P * per_job * sizeof(double) + (size_t)threads * (2 * S + 2) * sizeof(double) +
           (size_t)P * 4 * D * sizeof(int) + 16;  // + mbarrier
}

// one pass (part) over this lane's term slots: Aa, Ab accumulate the high
// phase's outputs; the low phase's are parked raw in park[0..2S) at the switch
template <int L, int DT>
__device__ __forceinline__ void conv_q_pass(const double *__restrict__ sx, const double *__restrict__ sy,
                                            const int *__restrict__ ex, const int *__restrict__ ey, int Drt,
                                            int part, int q, int f, int F, const int (&eacc)[4],
                                            double (&Aa)[digits_for(L)], double (&Ab)[digits_for(L)],
                                            double *park) {
    constexpr int S = digits_for(L);
    constexpr int NORM = norm_every(S);  // each accumulator takes one term (two real products) per slot
    const int D = DT > 0 ? DT : Drt;
    constexpr int P2 = PADZ + S;
    const int w1part = part, w2part = 1 - part;
    const long long sgn = part == 0 ? (long long)0x8000000000000000ULL : 0LL;
    auto neg = [&](double w) { return __longlong_as_double(__double_as_longlong(w) ^ sgn); };
    md_zero(Aa);
    md_zero(Ab);
    const int nlow = 2 * q + 2, nslots = D + 2;
    int cnt = 0;
    bool switched = false;
    // term metadata of slot j: x index i, y offsets of outputs a and b, the
    // alignment shifts (d1: the w1 plane, d2: the w2 plane) and whether b has
    // this term
    struct Meta {
        int i, kka, d1a, d2a, d1b, d2b;
        bool vb;
    };
    auto meta = [&](int j) {
        Meta m;
        const bool low = j < nlow;
        m.i = low ? j : j - nlow;
        const int a = low ? 2 * q + 1 : D - 1 - 2 * q;
        m.kka = a - m.i;
        m.vb = m.kka >= 1;
        const int kkb = m.vb ? m.kka - 1 : m.kka;
        const int ea = eacc[low ? 0 : 2], eb = eacc[low ? 1 : 3];
        const int exr = ex[m.i], exi = ex[D + m.i];
        auto shift = [&](int e, int ex_, int ey_) { return ex_ + ey_ <= ZERO_E / 2 ? 0 : e - ex_ - ey_; };
        m.d1a = shift(ea, exr, ey[w1part * D + m.kka]);
        m.d2a = shift(ea, exi, ey[w2part * D + m.kka]);
        m.d1b = m.vb ? shift(eb, exr, ey[w1part * D + kkb]) : 0;
        m.d2b = m.vb ? shift(eb, exi, ey[w2part * D + kkb]) : 0;
        return m;
    };
    double Ur[S], Ui[S];
    Meta cur = meta(min(f, nslots - 1));
    {
        const double *ux = sx + cur.i;
#pragma unroll
        for (int s = 0; s < S; s++) {
            Ur[s] = ux[s * D];
            Ui[s] = ux[(S + s) * D];
        }
    }
    for (int j = f; j < nslots; j += F) {
        const bool sw = j >= nlow && !switched;
        if (__any_sync(__activemask(), sw) && sw) {  // low outputs complete: park them raw
            switched = true;
#pragma unroll
            for (int s = 0; s < S; s++) {
                park[s] = Aa[s];
                park[S + s] = Ab[s];
                Aa[s] = 0.0;
                Ab[s] = 0.0;
            }
        }
        const int jn = j + F < nslots ? j + F : j;
        Meta nxt;
        const double *uxn = sx + (jn < nlow ? jn : jn - nlow);
        auto ahead = [&](int l) {  // after digit row l: the next slot's metadata and x digit S-1-l
            if (l == 1) nxt = meta(jn);
            const int u = S - 1 - l;
            Ur[u] = uxn[u * D];
            Ui[u] = uxn[(S + u) * D];
        };
        const bool fast = cur.d1a <= PADZ && cur.d2a <= PADZ && cur.d1b <= PADZ && cur.d2b <= PADZ;
        const int kkb = cur.vb ? cur.kka - 1 : cur.kka;
        if (__all_sync(__activemask(), fast)) {
            const double *W1a = sy + (w1part * P2 + PADZ - cur.d1a) * D + cur.kka;
            const double *W2a = sy + (w2part * P2 + PADZ - cur.d2a) * D + cur.kka;
            const double *W1b = sy + (w1part * P2 + PADZ - cur.d1b) * D + kkb;
            const double *W2b = sy + (w2part * P2 + PADZ - cur.d2b) * D + kkb;
            const bool vb = cur.vb;
            double w1a = W1a[0], w2a = neg(W2a[0]);
            double w1b = vb ? W1b[0] : 0.0, w2b = vb ? neg(W2b[0]) : 0.0;
#pragma unroll
            for (int l = 0; l < S; l++) {
                double n1a = 0.0, n2a = 0.0, n1b = 0.0, n2b = 0.0;
                if (l + 1 < S) {
                    n1a = W1a[(l + 1) * D];
                    n2a = neg(W2a[(l + 1) * D]);
                    n1b = vb ? W1b[(l + 1) * D] : 0.0;
                    n2b = vb ? neg(W2b[(l + 1) * D]) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < S - l; u++) {
                    Aa[u + l] = __fma_rn(Ur[u], w1a, Aa[u + l]);
                    Ab[u + l] = __fma_rn(Ur[u], w1b, Ab[u + l]);
                    Aa[u + l] = __fma_rn(Ui[u], w2a, Aa[u + l]);
                    Ab[u + l] = __fma_rn(Ui[u], w2b, Ab[u + l]);
                }
                ahead(l);
                w1a = n1a;
                w2a = n2a;
                w1b = n1b;
                w2b = n2b;
            }
        } else {
            const double *W1a = sy + w1part * P2 * D + cur.kka, *W2a = sy + w2part * P2 * D + cur.kka;
            const double *W1b = sy + w1part * P2 * D + kkb, *W2b = sy + w2part * P2 * D + kkb;
#pragma unroll
            for (int l = 0; l < S; l++) {
                const double w1a = (l >= cur.d1a) ? W1a[(PADZ + l - cur.d1a) * D] : 0.0;
                const double w2a = (l >= cur.d2a) ? neg(W2a[(PADZ + l - cur.d2a) * D]) : 0.0;
                const double w1b = (cur.vb && l >= cur.d1b) ? W1b[(PADZ + l - cur.d1b) * D] : 0.0;
                const double w2b = (cur.vb && l >= cur.d2b) ? neg(W2b[(PADZ + l - cur.d2b) * D]) : 0.0;
#pragma unroll
                for (int u = 0; u < S - l; u++) {
                    Aa[u + l] = __fma_rn(Ur[u], w1a, Aa[u + l]);
                    Ab[u + l] = __fma_rn(Ur[u], w1b, Ab[u + l]);
                    Aa[u + l] = __fma_rn(Ui[u], w2a, Aa[u + l]);
                    Ab[u + l] = __fma_rn(Ui[u], w2b, Ab[u + l]);
                }
                ahead(l);
            }
        }
        cur = nxt;
        if (++cnt == NORM) {
            carry_pass(Aa);
            carry_pass(Ab);
            cnt = 0;
        }
    }
    carry_pass(Aa);
    carry_pass(Ab);
    if (!switched) {  // no high-phase slots on this lane: everything belongs to the low outputs
#pragma unroll
        for (int s = 0; s < S; s++) {
            park[s] = Aa[s];
            park[S + s] = Ab[s];
            Aa[s] = 0.0;
            Ab[s] = 0.0;
        }
    }
}

template <int L, int DT>
__global__ void __launch_bounds__(DT == 128 || DT == 0 ? 256 : 128, DT == 128 || DT == 0 ? 1 : (L <= 5 ? 3 : 2))
    conv_q_kernel(double *__restrict__ dpool, int *__restrict__ epool, double *__restrict__ lpool,
                  const int *__restrict__ jobs, int njobs, int Drt, int Q, int F, int P) {
    constexpr int S = digits_for(L);
    const int D = DT > 0 ? DT : Drt;
    const int SX = 2 * S * D, SY = 2 * (PADZ + S) * D;
    const int threads_per_job = Q * F;
    extern __shared__ __align__(16) double sm[];
    double *sdig = sm;                                       // [P][SX + SY]
    double *spark = sm + (size_t)P * (SX + SY);              // [threads][2S + 2]
    constexpr int PSTR = 2 * S + 2;
    int *sexp = (int *)(spark + (size_t)blockDim.x * PSTR);  // [P][2 series][2][D]

    const int job0 = blockIdx.x * P;
    // staging as in conv_dig_kernel (D is even: TMA bulk copies)
    uint64_t *bar = reinterpret_cast<uint64_t *>(sexp + (size_t)P * 4 * D);
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
                bulk_g2s(base, dpool + (size_t)jobs[4 * job] * dig_slot_stride(S, D), (unsigned)(2 * S * D * 8), bar);
            else
                bulk_g2s(base + SX + ((which - 1) * (PADZ + S) + PADZ) * D,
                         dpool + (size_t)jobs[4 * job + 1] * dig_slot_stride(S, D) + (size_t)(which - 1) * S * D,
                         (unsigned)(S * D * 8), bar);
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
    mbar_wait(bar, 0);
    __syncthreads();

    const int jl = threadIdx.x / threads_per_job;
    const int r = threadIdx.x - jl * threads_per_job;
    const int q = r / F, f = r - q * F;
    const int jlc = min(jl, P - 1);
    const double *sx = sdig + (size_t)jlc * (SX + SY), *sy = sx + SX;
    const int *ex = sexp + jlc * 4 * D, *ey = ex + 2 * D;
    // the four outputs: 0 = 2q+1, 1 = 2q (low phase), 2 = D-1-2q, 3 = D-2-2q (high)
    const int kout[4] = {2 * q + 1, 2 * q, D - 1 - 2 * q, D - 2 - 2 * q};

    // exponent pre-pass: anchors of the four outputs x (re, im) over all their terms
    int ea[2][4];
#pragma unroll
    for (int p = 0; p < 2; p++)
#pragma unroll
        for (int o = 0; o < 4; o++) ea[p][o] = ZERO_E;
    const int nlow = 2 * q + 2;
    for (int j = f; j < D + 2; j += F) {
        const bool low = j < nlow;
        const int i = low ? j : j - nlow;
        const int a = low ? 2 * q + 1 : D - 1 - 2 * q;
        const int oa = low ? 0 : 2;
        const int xr = ex[i], xi = ex[D + i];
        {
            const int yr = ey[a - i], yi = ey[D + a - i];
            const int er = max(xr + yr, xi + yi), ei = max(xr + yi, xi + yr);
            if (low) {
                ea[0][0] = max(ea[0][0], er);
                ea[1][0] = max(ea[1][0], ei);
            } else {
                ea[0][2] = max(ea[0][2], er);
                ea[1][2] = max(ea[1][2], ei);
            }
        }
        if (a - 1 - i >= 0) {
            const int yr = ey[a - 1 - i], yi = ey[D + a - 1 - i];
            const int er = max(xr + yr, xi + yi), ei = max(xr + yi, xi + yr);
            if (low) {
                ea[0][1] = max(ea[0][1], er);
                ea[1][1] = max(ea[1][1], ei);
            } else {
                ea[0][3] = max(ea[0][3], er);
                ea[1][3] = max(ea[1][3], ei);
            }
        }
        (void)oa;
    }
#pragma unroll
    for (int p = 0; p < 2; p++)
#pragma unroll
        for (int o = 0; o < 4; o++) {
            for (int off = F >> 1; off > 0; off >>= 1) ea[p][o] = max(ea[p][o], __shfl_xor_sync(0xffffffffu, ea[p][o], off));
            ea[p][o] = max(ea[p][o], ZERO_E);
        }

    double *park = spark + (size_t)threadIdx.x * PSTR;
    const int job = job0 + jl;
    const bool writer = jl < P && job < njobs;
    double *zd = dpool;
    int *ze = epool;
    double *zl = nullptr;
    int wdig = 0;
    if (writer) {
        const int out = jobs[4 * job + 2];
        const int code = jobs[4 * job + 3];
        zd = dpool + (size_t)out * dig_slot_stride(S, D);
        ze = epool + (size_t)out * 2 * D;
        wdig = code & 1;
        if (code & 2) zl = lpool + (size_t)(code >> 2) * 2 * L * D;
    }
#pragma unroll 1
    for (int part = 0; part < 2; part++) {
        double Aa[S], Ab[S];
        const int eacc[4] = {ea[part][0], ea[part][1], ea[part][2], ea[part][3]};
        conv_q_pass<L, DT>(sx, sy, ex, ey, D, part, q, f, F, eacc, Aa, Ab, park);
        // high outputs: shuffle sums over the F lanes (exact; every lane has them)
        for (int off = F >> 1; off > 0; off >>= 1) {
#pragma unroll
            for (int s = 0; s < S; s++) {
                Aa[s] = __dadd_rn(Aa[s], __shfl_xor_sync(0xffffffffu, Aa[s], off));
                Ab[s] = __dadd_rn(Ab[s], __shfl_xor_sync(0xffffffffu, Ab[s], off));
            }
        }
        // low outputs: every lane carries its parked raw partials, then the same sums
        double Pa[S], Pb[S];
#pragma unroll
        for (int s = 0; s < S; s++) {
            Pa[s] = park[s];
            Pb[s] = park[S + s];
        }
        carry_pass(Pa);
        carry_pass(Pb);
        for (int off = F >> 1; off > 0; off >>= 1) {
#pragma unroll
            for (int s = 0; s < S; s++) {
                Pa[s] = __dadd_rn(Pa[s], __shfl_xor_sync(0xffffffffu, Pa[s], off));
                Pb[s] = __dadd_rn(Pb[s], __shfl_xor_sync(0xffffffffu, Pb[s], off));
            }
        }
        __syncwarp();  // parked partials consumed before the emit scratch reuses them
        // the four outputs over the F lanes (lane f emits outputs o = f, f+F, ...)
        if (writer)
            for (int o = f; o < 4; o += F) {
                double C[S];
#pragma unroll
                for (int s = 0; s < S; s++) C[s] = o == 0 ? Pa[s] : o == 1 ? Pb[s] : o == 2 ? Aa[s] : Ab[s];
                conv_dig_emit<L>(C, ea[part][o], wdig ? zd : nullptr, ze, zl, D, kout[o], part, park);
            }
        __syncwarp();
    }
}

}  // namespace mdps
