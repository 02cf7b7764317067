/*
 * mdps_test.h — diagnostic entry points of libmdps: the device kernels of the
 * hot path exposed one at a time for unit parity tests and measurement.
 * Same conventions as libmdps.h (layouts, error codes, asynchronous on
 * `stream`, DEVICE pointers unless stated).
 */
#ifndef MDPS_TEST_H
#define MDPS_TEST_H

#include "libmdps.h"

#ifdef __cplusplus
extern "C" {
#endif

/* count independent truncated products z[c] = x[c] * y[c] mod t^(degree+1)
 * with the product kernel of `algo` (MDPS_ALGO_EFT or
 * MDPS_ALGO_DIGITS), the same launch configuration as mdps_eval_diff.
 * x, y, z: [count][2][limbs][degree+1]; z must not alias x or y. */
int mdps_test_series_mul(const double *x, const double *y, double *z, int32_t count,
                         int32_t degree, int32_t limbs, int32_t algo, mdps_stream_t stream);

/* Device md arithmetic on arrays of real md numbers a[count][limbs],
 * b[count][limbs] -> c[count][limbs]: op 0 = add, 1 = mul (md.cuh). */
int mdps_test_md_op(int32_t op, const double *a, const double *b, double *c, int32_t count,
                    int32_t limbs, mdps_stream_t stream);

/* Device sum of squares of a complex md vector v[count][2][limbs]:
 * out[limbs] = sum_j re_j^2 + im_j^2 (PAPER.md:82-95 without the sqrt). */
int mdps_test_norm2sq(const double *v, int32_t count, int32_t limbs, double *out,
                      mdps_stream_t stream);

/* Round trip through the digit format: limbs -> digits -> limbs for
 * count series [count][2][limbs][degree+1] (digits algo staging). */
int mdps_test_digits_roundtrip(const double *x, double *y, int32_t count, int32_t degree,
                               int32_t limbs, mdps_stream_t stream);

/* FP64 peak microbenchmark: independent DFMA chains on every SM for about
 * `iters` iterations; writes the measured FP64 instructions per second
 * (host pointer) — the roofline denominator measured in the same run. */
int mdps_fp64_peak(int64_t iters, double *inst_per_s, mdps_stream_t stream);

/* Launch-geometry override of the digit product kernel (tuning only): F
 * lanes per output pair, P jobs per block and NP lane sets per job of a
 * complex system (1: both parts of an output on one thread, the fused-parts
 * kernel, where it exists — L <= 5, else ignored; 3: the same with the fold
 * parked in local memory; 2: one lane set per part, twice the threads per job) for every later launch in this process; 0 =
 * the model's / the tuned table's choice (the default).  F in {0,1,2,4,8}, P
 * a power of two <= 32, NP in {0,1,2,3}; MDPS_EINVAL otherwise, and at launch
 * when the geometry does not fit the kernel's thread / shared-memory limits.
 * Real systems always run one lane set.  Not thread-safe. */
int mdps_test_force_geometry(int32_t F, int32_t P, int32_t NP);

/* Programmatic dependent launch of the digit product levels (measurement
 * only): 1 (default) = each level's kernel is launched with the
 * programmatic-stream-serialization attribute, so its blocks are scheduled
 * while the previous level drains and wait for it (griddepcontrol.wait)
 * before reading the pools; 0 = plain stream order.  Bit 1 set (2, 3): also
 * run every level on the default launch geometry (no wider geometry for
 * levels below one wave).  Bit 2 set (4..7): systems created afterwards keep
 * every product in its earliest level (no level balancing).  Results are
 * identical.  Applies to later launches in this process.  Not thread-safe. */
int mdps_test_set_pdl(int32_t enable);

/* Per-kernel timing of mdps_eval_diff (measurement only): when enabled, each
 * launch group is bracketed by CUDA events on the caller's stream (the CUDA
 * graph path is bypassed while enabled).  mdps_system_timing synchronises
 * the recorded events and returns the summed device durations since the
 * last reset. */
typedef struct {
    double conv_ms;         /* product kernels (all levels) */
    double accum_ms;        /* addition-job kernel */
    double convert_ms;      /* input staging (copy or limbs -> digits) */
    int64_t conv_launches;
    int64_t accum_launches;
    int64_t convert_launches;
    int64_t evals;
} mdps_timing;

int mdps_system_set_timing(mdps_system *sys, int32_t enable);
int mdps_system_timing(mdps_system *sys, mdps_timing *out, int32_t reset);

/* Phase trace of the last solve (synchronises): globaltimer nanoseconds at the
 * start of the persistent solver kernel and at the completion of each of its
 * grid barriers (refinement phases, then one per coefficient pair of the
 * substitution loop, two where the dx step cannot overlap the updates).  Returns the
 * number of stamps written to ns (<= max) or < 0; refine_steps (optional) =
 * Newton-Schulz steps run. */
int mdps_solver_trace(mdps_solver *solver, int64_t *ns, int32_t max, int32_t *refine_steps);

/* Job-queue diagnostics (MDPS_SCHED_QUEUE systems).  enable = 1 allocates a
 * per-ticket trace that every later evaluation fills with five globaltimer
 * stamps (ticket claimed, inputs ready, inputs staged, computed, flag
 * released; addition tickets fill 0, 1 and 4), enable = 0 frees it, < 0
 * leaves it as is.  With out != NULL (after an evaluation) copies
 * min(tickets, max_tickets) x 5 stamps, synchronising the device.  Returns
 * the ticket count (or the count copied), < 0 on error. */
int mdps_test_queue_trace(mdps_system *sys, int32_t enable, int64_t *out, int32_t max_tickets);

/* Tuning only: queue-kernel geometry for systems created afterwards — grid
 * cap (max_blocks > 0; 0 = occupancy x SMs) and lanes per output pair and part
 * (a power of two; 0 = the default rule).  Returns MDPS_OK or MDPS_EINVAL. */
int mdps_test_queue_config(int32_t max_blocks, int32_t lanes);

/* Host-only (no GPU): level balancing of a system's schedule (a product whose
 * output is only summed may run in any later level; such jobs move from the
 * earlier levels above `min_jobs` jobs into later levels below it), then the
 * schedule check and the memory plan of mdps_test_plan.  before / after:
 * product jobs per level (max_levels entries each, zero-filled); *moved: jobs
 * moved; *same_jobs: 1 if the balanced levels hold exactly the original
 * jobs, none moved to an earlier level.  Returns the number of levels, or
 * MDPS_EINVAL (a failed check included). */
int mdps_test_balance(const mdps_supports *supports, const int32_t *exponents, int32_t n, int64_t min_jobs,
                      int64_t *before, int64_t *after, int32_t max_levels, int64_t *moved, int32_t *same_jobs);

/* Host-only (no GPU): build the job schedule of a system, check it (every
 * slot in range, every input written by an earlier launch, no slot read and
 * written in one launch, no live slot overwritten — schedule.hpp
 * check_schedule), plan its memory (liveness reuse, `chunks` row chunks) and
 * check the plan.  out[0] pool bytes without reuse, out[1] with the plan,
 * out[2] chunks used, out[3] launches per evaluation.  corrupt in {1,2,3}
 * damages the plan first (same-launch read/write, overwrite of a live slot,
 * slot out of range): then MDPS_EINVAL means the check caught it, 1 that it
 * did not. */
int mdps_test_plan(const mdps_supports *supports, const int32_t *exponents, int32_t n, int32_t degree,
                   int32_t limbs, int32_t eft, int32_t batch, int32_t chunks, int32_t corrupt, int64_t *out);

#ifdef __cplusplus
}
#endif
#endif /* MDPS_TEST_H */
