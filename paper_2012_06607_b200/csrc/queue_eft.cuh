// queue_eft.cuh — the device-side job queue: ONE persistent
// launch runs every product job and every addition job of an evaluation.
//
// The paper's multitasking (§5, Fig. 1) lets tasks take the
// next job index from a counter guarded by a binary semaphore and separates
// the stages by barriers.  Here the counter is a global
// atomic, a "task" is a thread block, and the stage barriers are replaced by
// per-series ready flags: a product job starts as soon as ITS two input
// series are final, not when their whole level is done.  Job indices are
// handed out in topological order (level by level, then the addition jobs),
// so a job only ever waits on jobs with smaller indices, all of which were
// claimed by running blocks — no deadlock, whatever the grid size.
//
// Flags hold the evaluation's epoch (ctl->epoch + 1 during a launch), so they
// need no reset between evaluations; the block taking the last ticket resets
// the counter and advances the epoch.  Pool series written inside the launch
// are read with ld.global.cg (L2, never a stale L1 line) after a gpu-scope
// acquire of their flag; the producer stores, fences, then releases the flag.
//
// Arithmetic: the paper's md arithmetic (md.cuh level bins, as
// conv_eft_kernel), with one job spread over the whole block for latency:
// thread (t, part, f) accumulates the real or imaginary part of the folded
// output pair (t, D-1-t) over the fold iterations j = f, f+F, ... (F lanes per
// pair and part), and the F partial bin sets are merged by shuffles in a fixed
// order (lane 0 of the group merges 1, then 2-3, ...), so every evaluation is
// bitwise identical.  Addition jobs: one thread per (output series, k) as in
// accum_eft_kernel, each entry acquired before it is read.
#pragma once
#include "md.cuh"

namespace mdps {

// diagnostics (mdps_test_queue_trace): globaltimer stamps per ticket — claimed,
// inputs ready, staged, computed, released (addition tickets: 0, 1, 4)
constexpr int QUEUE_TRACE_STAMPS = 5;

struct QueueCtl {
    unsigned int counter;  // next ticket (reset to 0 by the last block)
    unsigned int epoch;    // evaluations completed; flags of this launch hold epoch + 1
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u32(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// wait until series `slot` is final (slots below nready are inputs: always).
// Relaxed polling; the caller issues one acquire fence after its waits.
__device__ __forceinline__ void queue_wait(const unsigned *flags, int slot, int nready, unsigned cur) {
    if (slot < nready) return;
    if (ld_relaxed_u32(flags + slot) == cur) return;
    unsigned ns = 8;
    while (ld_relaxed_u32(flags + slot) != cur) {
        __nanosleep(ns);
        ns = ns < 128 ? 2 * ns : ns;
    }
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// wait until the NS series slot[0..NS) are final: the flags are polled
// together (one L2 round trip per poll, not one per series)
template <int NS>
__device__ __forceinline__ void queue_wait_all(const unsigned *flags, const int (&slot)[NS], const bool (&need)[NS],
                                               unsigned cur) {
    unsigned ns = 8;
    for (;;) {
        bool ok = true;
#pragma unroll
        for (int u = 0; u < NS; u++)
            if (need[u]) ok &= ld_relaxed_u32(flags + slot[u]) == cur;
        if (ok) return;
        __nanosleep(ns);
        ns = ns < 128 ? 2 * ns : ns;
    }
}

// threads per job for the queue kernel: 2 parts x T pairs x F lanes, F the
// largest power of two <= fmax with 2 T F <= 256 (default 4: measured on dd,
// scripts/queue_tune.py — 8 and 16 lanes cost more in merges than they save)
__host__ __device__ inline int queue_lanes(int D, int fmax = 4) {
    const int T = (D + 1) / 2;
    int F = fmax;
    while (F > 1 && 2 * T * F > 256) F >>= 1;
    return F;
}

template <int L>
__global__ void __launch_bounds__(256) queue_eft_kernel(
    const double *__restrict__ x_in,  // [nx][2][L][D]: the evaluation's input series (slots 0..nx-1)
    double *pool,                     // [slot][2][L][D] (slots nx..: coefficients, then products)
    unsigned *flags,                  // [slot]: epoch of the evaluation that finished the series
    QueueCtl *ctl, const int *__restrict__ jobs, int njobs,  // (in1, in2, out, code), topological
    const int *__restrict__ task_ptr, const int *__restrict__ ent_slot, const int *__restrict__ ent_w,
    int ntasks, int nvals, int tasks_per_ticket, int nx, int nready, int D, int F, double *__restrict__ values,
    double *__restrict__ jac, long long *__restrict__ trace) {  // trace: NULL, or [ticket][QUEUE_TRACE_STAMPS] ns
    extern __shared__ double sq[];
    __shared__ unsigned s_ticket;
    constexpr int TS = QUEUE_TRACE_STAMPS;
    const int LD2 = 2 * L * D;
    const int T = (D + 1) / 2;
    const unsigned cur = ctl->epoch + 1u;
    const unsigned nticket_add = (unsigned)((ntasks + tasks_per_ticket - 1) / tasks_per_ticket);
    const unsigned total = (unsigned)njobs + nticket_add;
    auto series = [&](int slot) -> const double * {
        return slot < nx ? x_in + (size_t)slot * LD2 : pool + (size_t)slot * LD2;
    };
    // lane mapping of a product job: groups of F adjacent lanes per (t, part)
    const int g = threadIdx.x / F, f = threadIdx.x - g * F;
    const int t = g >> 1, part = g & 1;
    for (;;) {
        if (threadIdx.x == 0) s_ticket = atomicAdd(&ctl->counter, 1u);
        __syncthreads();
        const unsigned tk = s_ticket;
        __syncthreads();
        if (tk >= total) {
            // every block takes exactly one ticket past the end, when it has
            // no more work: the last of those resets the queue for the next call
            if (threadIdx.x == 0 && tk == total + gridDim.x - 1) {
                ctl->counter = 0u;
                ctl->epoch = cur;
                __threadfence();
            }
            return;
        }
        if (trace && threadIdx.x == 0) trace[TS * tk] = (long long)globaltimer_ns();
        if (tk < (unsigned)njobs) {
            // ---- product job z = x * y mod t^D
            const int in1 = __ldg(jobs + 4 * tk), in2 = __ldg(jobs + 4 * tk + 1), out = __ldg(jobs + 4 * tk + 2);
            // one thread waits for both inputs (acquire), the barrier passes
            // the ordering on to the block; the loads bypass L1
            if (threadIdx.x == 0) {
                const int sl[2] = {in1, in2};
                const bool nd[2] = {in1 >= nready, in2 >= nready};
                if (nd[0] || nd[1]) {
                    queue_wait_all<2>(flags, sl, nd, cur);
                    fence_acquire_gpu();
                }
                if (trace) trace[TS * tk + 1] = (long long)globaltimer_ns();
            }
            __syncthreads();
            const double *s1 = series(in1), *s2 = series(in2);
            // staging: up to 4 loads per thread in flight before the stores
            for (int base = threadIdx.x; base < 2 * LD2; base += 4 * blockDim.x) {
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int idx = base + u * blockDim.x;
                    v[u] = idx < LD2 ? __ldcg(s1 + idx) : (idx < 2 * LD2 ? __ldcg(s2 + idx - LD2) : 0.0);
                }
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int idx = base + u * blockDim.x;
                    if (idx < 2 * LD2) sq[idx] = v[u];
                }
            }
            __syncthreads();
            if (trace && threadIdx.x == 0) trace[TS * tk + 2] = (long long)globaltimer_ns();
            const double *sx = sq, *sy = sq + LD2;
            double B1[L + 1], B2[L + 1];
            md_zero(B1);
            md_zero(B2);
            const int tt = t < T ? t : T - 1;  // padding lanes shadow the last pair (not written)
            // part 0: re = ar br - ai bi ; part 1: im = ar bi + ai br
            const int pb1 = part, pb2 = 1 - part;
            for (int j = f; j <= D; j += F) {
                const bool first = j <= tt;
                const int i = first ? j : j - tt - 1;
                const int k = first ? tt : D - 1 - tt;
                double ar[L], a2[L], b1[L], b2[L];
#pragma unroll
                for (int p = 0; p < L; p++) {
                    ar[p] = sx[p * D + i];
                    const double ai = sx[(L + p) * D + i];
                    a2[p] = part == 0 ? -ai : ai;
                    b1[p] = sy[(pb1 * L + p) * D + (k - i)];
                    b2[p] = sy[(pb2 * L + p) * D + (k - i)];
                }
                if (first) {
                    bins_fma<L>(B1, ar, b1);
                    bins_fma<L>(B1, a2, b2);
                } else {
                    bins_fma<L>(B2, ar, b1);
                    bins_fma<L>(B2, a2, b2);
                }
            }
            // fixed-order merge of the F lanes' partial sums into lane f = 0
            for (int off = 1; off < F; off <<= 1) {
                double C1[L + 1], C2[L + 1];
#pragma unroll
                for (int p = 0; p <= L; p++) {
                    C1[p] = __shfl_down_sync(0xffffffffu, B1[p], off, F);
                    C2[p] = __shfl_down_sync(0xffffffffu, B2[p], off, F);
                }
                if ((f & (2 * off - 1)) == 0) {
                    bins_merge<L>(B1, C1);
                    bins_merge<L>(B2, C2);
                }
            }
            if (f == 0 && t < T) {
                double *z = pool + (size_t)out * LD2;
                double r[L];
                md_renorm(B1, r);
#pragma unroll
                for (int p = 0; p < L; p++) z[(part * L + p) * D + t] = r[p];
                md_renorm(B2, r);
#pragma unroll
                for (int p = 0; p < L; p++) z[(part * L + p) * D + (D - 1 - t)] = r[p];
            }
            // the block's stores, then one gpu-scope fence and the release of
            // the output's flag by thread 0 (the barrier orders the stores first)
            __syncthreads();
            if (threadIdx.x == 0) {
                if (trace) trace[TS * tk + 3] = (long long)globaltimer_ns();
                __threadfence();
                st_release_u32(flags + out, cur);
                if (trace) trace[TS * tk + 4] = (long long)globaltimer_ns();
            }
        } else {
            // ---- addition jobs: values and Jacobian entries
            const int a0 = (int)(tk - (unsigned)njobs) * tasks_per_ticket;
            // every thread waits for the entries of its own batch as it goes
            // (sums start on the entries that are final), an acquire load
            // after each wait; the loads bypass L1
            if (trace && threadIdx.x == 0) trace[TS * tk + 1] = (long long)globaltimer_ns();
            for (int e = threadIdx.x; e < tasks_per_ticket * D; e += blockDim.x) {
                const int task = a0 + e / D, k = e - (e / D) * D;
                if (task >= ntasks) break;
                double Br[L + 1], Bi[L + 1];
                md_zero(Br);
                md_zero(Bi);
                // entries in batches of QB: the loads of a batch are in flight
                // together (a serial load per entry costs an L2 round trip
                // each), then summed in entry order (the same bins as one by one)
                constexpr int QB = L <= 2 ? 8 : (L <= 5 ? 4 : 2);
                const int q1 = __ldg(task_ptr + task + 1);
                for (int qb = __ldg(task_ptr + task); qb < q1; qb += QB) {
                    double ar[QB][L], ai[QB][L];
                    int w[QB];
                    int slots[QB];
#pragma unroll
                    for (int u = 0; u < QB; u++) slots[u] = qb + u < q1 ? __ldg(ent_slot + qb + u) : 0;
                    bool need[QB], any = false;
#pragma unroll
                    for (int u = 0; u < QB; u++) {
                        need[u] = qb + u < q1 && slots[u] >= nready;
                        any |= need[u];
                    }
                    if (any) {
                        queue_wait_all<QB>(flags, slots, need, cur);
                        fence_acquire_gpu();
                    }
#pragma unroll
                    for (int u = 0; u < QB; u++) {
                        const bool in = qb + u < q1;
                        const int slot = slots[u];
                        w[u] = in ? __ldg(ent_w + qb + u) : 0;
                        const double *sp = series(slot);
#pragma unroll
                        for (int p = 0; p < L; p++) {
                            ar[u][p] = in ? __ldcg(sp + p * D + k) : 0.0;
                            ai[u][p] = in ? __ldcg(sp + (L + p) * D + k) : 0.0;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < QB; u++) {
                        if (w[u] == 1) {
                            bins_add<L>(Br, ar[u]);
                            bins_add<L>(Bi, ai[u]);
                        } else if (w[u] != 0) {
                            bins_add_scaled<L>(Br, ar[u], (double)w[u]);
                            bins_add_scaled<L>(Bi, ai[u], (double)w[u]);
                        }
                    }
                }
                double zr[L], zi[L];
                md_renorm(Br, zr);
                md_renorm(Bi, zi);
                double *o = task < nvals ? values + (size_t)task * LD2 : jac + (size_t)(task - nvals) * LD2;
#pragma unroll
                for (int p = 0; p < L; p++) {
                    o[p * D + k] = zr[p];
                    o[(L + p) * D + k] = zi[p];
                }
            }
            if (trace) {
                __syncthreads();
                if (threadIdx.x == 0) trace[TS * tk + 4] = (long long)globaltimer_ns();
            }
        }
    }
}

}  // namespace mdps
