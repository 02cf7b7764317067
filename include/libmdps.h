/*
 * libmdps.h — C ABI of the B200-native evaluation and differentiation of a
 * polynomial system at a vector of truncated power series in complex
 * multiple-double precision (arXiv 2012.06607, "Parallel Software to Offset
 * the Cost of Higher Precision", J. Verschelde).
 *
 * The operation (§4): given a system
 *   f = (f_0, ..., f_{N-1}) of polynomials in x = (x_0, ..., x_{n-1}) whose
 * coefficients are truncated power series in t, and a point x(t) whose
 * components are truncated power series, compute
 *   values[i]      = f_i(x(t))                 mod t^(degree+1)
 *   jacobian[i][j] = (d f_i / d x_j)(x(t))     mod t^(degree+1)
 * with every coefficient a complex multiple-double number of `limbs` doubles
 * (§2).  Series products are truncated convolutions
 * z_k = sum_{i<=k} x_i y_{k-i} (§3); the Jacobian is
 * computed by algorithmic differentiation at about 3x the cost of the
 * evaluation: forward, backward and cross products per
 * monomial.  N may differ from n (PAPER.md:258 allows N >= n; N < n is a
 * subset of the rows, e.g. one GPU's share of a system sharded by rows,
 * DESIGN.md §10).
 *
 * Series layout (all series arguments): float64, [part][limb][coefficient]
 * per series — part 0 = real, 1 = imaginary; limb 0 most significant
 * (non-overlapping expansion); coefficient k = 0..degree (D = degree+1).
 * One series is 2*limbs*D doubles; arrays of series are contiguous.
 *
 * Threading: calls on different systems are independent.  One eval_diff may
 * be in flight per system (the system owns its workspace).
 */
#ifndef LIBMDPS_H
#define LIBMDPS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MDPS_OK 0
#define MDPS_EINVAL (-1)   /* invalid argument (see mdps_last_error) */
#define MDPS_ENOMEM (-2)   /* device or host allocation failed */
#define MDPS_ECUDA (-3)    /* a CUDA call or kernel launch failed */

/* A cudaStream_t (the same handle type; this header needs no CUDA headers). */
typedef struct CUstream_st *mdps_stream_t;

typedef struct mdps_system mdps_system; /* opaque; owns device memory */

/* Supports of the system in CSR form (HOST pointers, read during create only).
 * Polynomial i has monomials r in [poly_ptr[i], poly_ptr[i+1]); monomial r has
 * variables vars[mono_ptr[r] .. mono_ptr[r+1]) — indices in [0, n), distinct
 * within a monomial, in any order.  An empty monomial is a constant term.
 * Duplicate monomials within a polynomial are allowed (they are summed). */
typedef struct {
    int32_t n_polys;          /* N >= 1 polynomials (rows); N = n for a square system */
    const int32_t *poly_ptr;  /* [n_polys+1], non-decreasing, poly_ptr[0] = 0 */
    const int32_t *mono_ptr;  /* [M+1], non-decreasing, mono_ptr[0] = 0, M = poly_ptr[n_polys] */
    const int32_t *vars;      /* [nnz], nnz = mono_ptr[M] */
} mdps_supports;

/* Convolution algorithm for the product jobs. */
#define MDPS_ALGO_AUTO 0     /* default: digits, except EFT above degree 127 and for limbs = 2
                                (faster there, measured) */
#define MDPS_ALGO_EFT 1      /* limb planes: TwoProd + TwoSum level bins */
#define MDPS_ALGO_DIGITS 2   /* 23-bit digit planes, exact FP64 FMA products */

typedef struct {
    int32_t algo;        /* MDPS_ALGO_* */
    int32_t use_graph;   /* 1: capture the launch sequence in a CUDA graph,
                            re-captured when the pointers or stream change */
    int32_t real;        /* 1: a real system — every coefficient and input series
                            has zero imaginary limbs (not checked); one real md
                            product per term (1/4 of the complex work), and the
                            imaginary limbs of values and Jacobian are 0 */
    int32_t batch;       /* >= 1 (0 = 1): evaluate the system at `batch` points per
                            call — series_in [batch][n][...], values_out
                            [batch][N][...], jacobian_out [batch][N][n][...] —
                            in one launch per level (small systems fill the GPU;
                            mdps_newton_step needs batch = 1) */
    int32_t schedule;    /* MDPS_SCHED_*: how the product and addition jobs are run */
    int32_t workspace_mb; /* LEVELS schedule: bound on the pool memory, MiB (0 = a quarter
                            of the device memory free at create).  Pool slots are reused
                            by liveness; when that is not enough the rows are split into
                            chunks evaluated one after the other (each its levels, then
                            its addition jobs), as few as fit (<= 64).  Measured: od
                            2.8 GB unbounded, 0.86 GB at 1000 MiB (4 chunks, +3.6% time);
                            deca 9.7 GB, 2.7 GB at 3000 MiB (+1.7%) */
} mdps_options;

/* Job scheduling (PAPER.md:367-378 job queue, 411-424 stages). */
#define MDPS_SCHED_AUTO 0    /* default: QUEUE for small systems on the EFT algorithm
                                (<= MDPS_QUEUE_MAX_PRODUCTS product jobs per call), else LEVELS */
#define MDPS_SCHED_LEVELS 1  /* one launch per DAG level, then one for the addition jobs */
#define MDPS_SCHED_QUEUE 2   /* one persistent launch: blocks claim jobs from a device
                                counter in topological order and wait on per-series ready
                                flags (EFT algorithm only) */
#define MDPS_QUEUE_MAX_PRODUCTS 8192

/* Create a system.  exponents: HOST [nnz] aligned with
 * vars, each >= 1.  coefficients: HOST [M][2][limbs][degree+1], the series
 * coefficient of each monomial.  n >= 1, 0 <= degree <= 255,
 * limbs in {2,3,4,5,8,10}.  All host arrays are deep-copied; the caller may
 * free them on return.  Returns NULL on error (mdps_last_error() says why):
 * invalid sizes, NULL pointers, n_polys < 1, non-monotone CSR, a variable
 * out of range or repeated within a monomial, an exponent < 1, or a failed
 * allocation.  Variables are sorted per monomial internally.  Requires a
 * current CUDA device (the device of the caller's current context). */
mdps_system *mdps_system_create(const mdps_supports *supports, const int32_t *exponents,
                                const double *coefficients, int32_t n, int32_t degree,
                                int32_t limbs);

/* As mdps_system_create, with options (NULL = defaults). */
mdps_system *mdps_system_create_ex(const mdps_supports *supports, const int32_t *exponents,
                                   const double *coefficients, int32_t n, int32_t degree,
                                   int32_t limbs, const mdps_options *options);

/* Evaluate and differentiate (the hot path).  DEVICE pointers:
 *   series_in    [n][2][limbs][D]      read only
 *   values_out   [N][2][limbs][D]      fully overwritten (N = supports->n_polys)
 *   jacobian_out [N][n][2][limbs][D]   fully overwritten; row i = polynomial,
 *                                      column j = variable; entries with no
 *                                      monomial of f_i containing x_j are 0.
 * Asynchronous: enqueues kernels on `stream` (NULL = legacy default stream)
 * and returns.  The outputs must not alias each other or series_in.
 * Returns MDPS_OK, MDPS_EINVAL (NULL/aliased pointers) or MDPS_ECUDA (a
 * launch failed); asynchronous faults surface at the caller's next
 * synchronisation.  Non-finite inputs propagate; nothing is checked on the
 * hot path. */
int mdps_eval_diff(mdps_system *sys, const double *series_in, double *values_out,
                   double *jacobian_out, mdps_stream_t stream);

/* End-to-end variant with HOST buffers (same layouts): copies series_in to the
 * device, evaluates, copies both outputs back and synchronises `stream`.
 * Host buffers may be pageable or pinned (pinned is faster). */
int mdps_eval_diff_host(mdps_system *sys, const double *series_in_host, double *values_host,
                        double *jacobian_host, mdps_stream_t stream);

/* Frees all device memory of the system (synchronises the device first). */
void mdps_system_destroy(mdps_system *sys);

/* Thread-local message for the last failure of a call on this thread. */
const char *mdps_last_error(void);

typedef struct {
    int64_t products;          /* series product jobs per eval (forward/backward/cross/common) */
    int64_t add_terms;         /* series added by the accumulation jobs */
    int64_t fp64_ops_conv;     /* algorithmic FP64 instructions of the product jobs */
    int64_t fp64_ops_total;    /* ... of the whole eval (conversions, products, sums) */
    int64_t compulsory_bytes;  /* inputs + coefficients + outputs, bytes */
    int32_t levels;            /* product levels (one launch each) */
    int32_t algo;              /* MDPS_ALGO_EFT or MDPS_ALGO_DIGITS */
    int32_t digits;            /* digits per part (digits algo), else 0 */
    int32_t launches;          /* kernel launches per eval */
    size_t workspace_bytes;    /* device memory owned by the system */
    int32_t n;                 /* variables (series_in holds batch * n series) */
    int32_t n_polys;           /* polynomials N (values_out: batch * N, jacobian_out: batch * N * n series) */
    int32_t degree;            /* truncation degree d (D = d + 1 coefficients) */
    int32_t limbs;             /* L */
    int32_t batch;             /* points per evaluation (mdps_options.batch) */
    int32_t schedule;          /* MDPS_SCHED_LEVELS or MDPS_SCHED_QUEUE (as resolved at create) */
    int32_t chunks;            /* row chunks evaluated one after the other (LEVELS; 1 = none) */
    int64_t pool_bytes;        /* of workspace_bytes: the slot pools (digits + limbs, or limbs) */
} mdps_stats;

/* Statistics of a system (for the measurement). */
int mdps_system_stats(const mdps_system *sys, mdps_stats *out);

/* Per-level job counts (levels entries) for diagnostics; returns levels or <0. */
int mdps_system_level_jobs(const mdps_system *sys, int64_t *jobs_per_level, int32_t max_levels);


/* ---------------------------------------------------------------------------
 * Block lower-triangular Toeplitz solver — the linear solve of one Newton step
 * on power series (§4).
 *
 * With linearisation A(t) = A_0 + A_1 t + ... + A_d t^d, A_k the n-by-n
 * matrix of coefficient k of the Jacobian series, solves
 *     A(t) dx(t) = b(t)   mod t^(d+1)
 * by forward substitution: A_0 dx_0 = b_0 and
 *     A_0 dx_j = b_j - sum_{i=1..j} A_i dx_{j-i},   j = 1..d,
 * factoring A_0 once (LU with partial pivoting, N = n: PAPER.md:260-262).
 * The GPU applies the factorisation as the explicit inverse A_0^-1 (formed
 * from the LU factors once), so that each of the d+1 solves is one parallel
 * matrix-vector product.
 *
 * Layouts are those of mdps_eval_diff: jacobian [n][n][2][limbs][D] (row p,
 * column q, series), rhs and dx [n][2][limbs][D]; D = degree + 1.
 * ------------------------------------------------------------------------- */
typedef struct mdps_solver mdps_solver; /* opaque; owns its device workspace */

/* n in [1, 128], degree in [0, 255], limbs in {2,3,4,5,8,10} (n <= 128 keeps
 * every exact digit accumulation of the solver below 2^53).  Allocates the
 * workspace (about 2x the Jacobian) on the current device.  NULL on error. */
mdps_solver *mdps_solver_create(int32_t n, int32_t degree, int32_t limbs);

/* A solver for N >= n equations in n unknowns, N <= 128 (least squares):
 * each dx_j minimises |A_0 dx_j - r_j| with r_j = b_j - sum_{i>=1} A_i dx_{j-i};
 * the GPU applies A_0^+ (refined to md precision from the normal equations'
 * double-precision solution).  Then jacobian is [N][n][...], rhs [N][...] and
 * dx_out [n][...] in mdps_solve; pivots (mdps_solver_status) are those of
 * A_0^H A_0.  N = n is mdps_solver_create.  Requires full column rank. */
mdps_solver *mdps_solver_create_ls(int32_t N, int32_t n, int32_t degree, int32_t limbs);

/* dx(t) with A(t) dx(t) = rhs(t) mod t^D (least squares for N > n).  DEVICE pointers: jacobian and rhs
 * read only, dx_out fully overwritten; dx_out must not alias the inputs.
 * Asynchronous on `stream`; one solve may be in flight per solver.  Returns
 * MDPS_OK, MDPS_EINVAL or MDPS_ECUDA.  A singular A_0 (a zero pivot column)
 * does not fail the call: it is reported by mdps_solver_status and dx_out is
 * then unspecified. */
int mdps_solve(mdps_solver *solver, const double *jacobian, const double *rhs, double *dx_out,
               mdps_stream_t stream);

/* After synchronising the last solve's stream: the pivot rows of the LU of
 * A_0 (HOST [n], row k swapped with pivots[k] at step k; NULL to skip) and
 * singular = 1 if some pivot column of A_0 was zero. */
int mdps_solver_status(mdps_solver *solver, int32_t *pivots, int32_t *singular);

/* After synchronising the last solve's stream: its outcome flags.
 * MDPS_SOLVE_SINGULAR: a zero pivot column of A_0 (as mdps_solver_status).
 * MDPS_SOLVE_NOT_CONVERGED: the md refinement of A_0's inverse (Newton-Schulz
 * from the double-precision Gauss-Jordan seed) missed ||I - W A_0||^2 <
 * 2^-(53 L + 16) after its step limit — A_0 is too ill-conditioned for a
 * double seed (kappa >~ 1e16; the paper's md LU, has no
 * such limit).  dx_out is unspecified when either flag is set. */
#define MDPS_SOLVE_SINGULAR 1
#define MDPS_SOLVE_NOT_CONVERGED 2
int mdps_solver_flags(mdps_solver *solver, int32_t *flags);

typedef struct {
    int64_t complex_fma;       /* complex md multiply-adds per solve (LU, inverse, substitution) */
    int64_t fp64_ops;          /* algorithmic FP64 instructions per solve */
    int32_t launches;          /* kernel launches per solve */
    int32_t grid_blocks;       /* co-resident blocks of the persistent kernels */
    size_t workspace_bytes;
} mdps_solver_info;

int mdps_solver_stats(const mdps_solver *solver, mdps_solver_info *out);

void mdps_solver_destroy(mdps_solver *solver);

/* One step of Newton's method on power series: f and its
 * Jacobian at x(t) (mdps_eval_diff), then J(t) dx(t) = -f(t) (the solver),
 * then x <- x + dx (md addition per coefficient).  `sys` and `solver` must
 * have the same n, degree and limbs.  DEVICE pointers: x [n][2][limbs][D]
 * in/out; dx_out (NULL: solver scratch) receives dx; update_norm (NULL: not
 * written) receives ||dx|| = max over components and coefficients of the
 * complex modulus of dx's leading limbs (reading R14).  The solver
 * owns the f and J workspace (allocated at the first step).  Asynchronous. */
int mdps_newton_step(mdps_system *sys, mdps_solver *solver, double *x, double *dx_out, double *update_norm,
                     mdps_stream_t stream);

/* Newton's method: steps from x until ||dx|| <= tol or max_iters steps (the
 * paper's stopping rule, §6: tolerance 1.0E-32 on ||dx||, at most
 * 8, 8, 12, 16 steps for degrees 8, 16, 24, 32).  Synchronises `stream` after
 * every step to read the norm.  Returns the number of steps taken (>= 1) or
 * < 0 on error; *last_norm (optional) = ||dx|| of the last step. */
int mdps_newton(mdps_system *sys, mdps_solver *solver, double *x, int32_t max_iters, double tol,
                double *last_norm, mdps_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* LIBMDPS_H */
