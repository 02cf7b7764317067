// queue_dig.cuh — the device-side job queue (PAPER.md:367-378
// Fig. 1, 411-424) for the digit algorithm: one persistent launch runs every
// product job (P per ticket, the block work of conv_dig_kernel) and every
// addition job of an evaluation.  A ticket waits only for the input series
// of its own jobs (per-series ready flags holding the evaluation's epoch, as
// in queue_eft.cuh), so the jobs of consecutive DAG levels overlap: no level
// ends with a partial wave, no launch gap, and the GPU holds as many jobs as
// fit instead of one level's.  The x series are converted to digits by
// to_digits_kernel before the launch (stream order makes them ready).
#pragma once
#include "conv_dig.cuh"
#include "queue_eft.cuh"

namespace mdps {

template <int L, int DT>
__global__ void __launch_bounds__(DT == 128 || DT == 0 ? 256 : 128,
                                  DT == 128 || DT == 0 ? 1 : (L <= 4 ? 4 : (L <= 8 ? 3 : 2)))
    queue_dig_kernel(double *dpool, int *epool, double *lpool, unsigned *flags, QueueCtl *ctl,
                     const int *__restrict__ jobs, int njobs, int Drt, int T, int F, int P,
                     const int *__restrict__ task_ptr, const int *__restrict__ ent_flag,
                     const int *__restrict__ ent_lslot, const int *__restrict__ ent_w, int ntasks, int nvals,
                     int tasks_per_ticket, int nready, double *__restrict__ values, double *__restrict__ jac) {
    extern __shared__ __align__(16) double sm[];
    __shared__ unsigned s_ticket;
    const int D = DT > 0 ? DT : Drt;
    const unsigned cur = ctl->epoch + 1u;
    const unsigned nprod = (unsigned)((njobs + P - 1) / P);
    const unsigned total = nprod + (unsigned)((ntasks + tasks_per_ticket - 1) / tasks_per_ticket);
    for (;;) {
        if (threadIdx.x == 0) s_ticket = atomicAdd(&ctl->counter, 1u);
        __syncthreads();
        const unsigned tk = s_ticket;
        __syncthreads();
        if (tk >= total) {
            if (threadIdx.x == 0 && tk == total + gridDim.x - 1) {
                ctl->counter = 0u;
                ctl->epoch = cur;
                __threadfence();
            }
            return;
        }
        if (tk < nprod) {
            const int job0 = (int)tk * P;
            // warp 0: one lane per input series of the ticket's jobs
            if (threadIdx.x < 32) {
                for (int i = threadIdx.x; i < 2 * P; i += 32) {
                    const int job = min(job0 + i / 2, njobs - 1);
                    queue_wait(flags, __ldg(jobs + 4 * job + (i & 1)), nready, cur);
                }
                fence_acquire_gpu();
            }
            __syncthreads();
            conv_dig_block<L, DT, false, true>(dpool, epool, lpool, jobs, job0, njobs, Drt, T, F, P, sm, nullptr, 0u);
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                for (int jl = 0; jl < P && job0 + jl < njobs; jl++) st_release_u32(flags + __ldg(jobs + 4 * (job0 + jl) + 2), cur);
            }
        } else {
            queue_add_ticket<L>(flags, cur, nready, task_ptr, ent_flag, ent_lslot, ent_w,
                                (int)(tk - nprod) * tasks_per_ticket, tasks_per_ticket, ntasks, nvals, D, nullptr, 0,
                                lpool, values, jac);
        }
    }
}

}  // namespace mdps
