// libmdps.cu — the C ABI (include/libmdps.h): system creation, the leveled
// launcher of the product jobs and the addition jobs, statistics.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/libmdps.h"
#include "../../include/mdps_test.h"
#include "conv_dig.cuh"
#include "conv_dig_fused.cuh"
#include "kernels_dig.cuh"
#include "kernels_eft.cuh"
#include "queue_eft.cuh"
#include "schedule.hpp"

using namespace mdps;

static thread_local std::string g_err;

static void set_err(const std::string &s) { g_err = s; }

void mdps_internal_set_error(const std::string &s) { g_err = s; }  // solve.cu

#define CUDA_TRY(call, code)                                                          \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess) {                                                      \
            set_err(std::string(#call) + ": " + cudaGetErrorString(e_));              \
            return code;                                                              \
        }                                                                             \
    } while (0)

extern "C" const char *mdps_last_error(void) { return g_err.c_str(); }

static bool valid_limbs(int L) { return L == 2 || L == 3 || L == 4 || L == 5 || L == 8 || L == 10; }

// dispatch a templated functor on L
template <template <int> class Fn, typename... Args>
static int dispatch_L(int L, Args &&...args) {
    switch (L) {
        case 2: return Fn<2>::run(args...);
        case 3: return Fn<3>::run(args...);
        case 4: return Fn<4>::run(args...);
        case 5: return Fn<5>::run(args...);
        case 8: return Fn<8>::run(args...);
        case 10: return Fn<10>::run(args...);
    }
    set_err("unsupported limb count");
    return MDPS_EINVAL;
}

// ---------------------------------------------------------------------------
// launch geometry
struct EftGeom {
    int T, P, threads;
    size_t smem;
};
static EftGeom eft_geom(int L, int D) {
    EftGeom g;
    g.T = (D + 1) / 2;
    g.P = std::max(1, 128 / g.T);
    g.threads = g.P * g.T;
    const size_t JS = (size_t)2 * (2 * L * D) + 2;
    g.smem = ((size_t)g.P * JS + (size_t)g.threads * 2 * (L + 1)) * sizeof(double);
    return g;
}

struct DigGeom {
    int T, F, P, threads;
    size_t smem;
    int NP = 2;  // part lane sets: 2 for complex systems (one warp set per part), 1 for real ones
};
// Launch geometry of the product kernel: F lanes per output pair and P jobs
// per block, chosen by modelled throughput — resident warps per SM (limited
// by registers, shared memory and 64 warps), lane balance of the folded
// triangle ((D+1) terms over F lanes, each part's lane set padded to whole
// warps) and the per-lane term count that amortises the per-output epilogue
// — unless a measured table entry exists.
// forced geometry of the product kernel (mdps_test_force_geometry; tuning only)
static int g_force_F = 0, g_force_P = 0, g_force_NP = 0;
static int g_force_queue_blocks = 0;  // mdps_test_queue_config: grid cap of the queue kernel (0 = occupancy)
static int g_force_queue_F = 0;       // mdps_test_queue_config: lanes per output pair and part (0 = default)

// Measured best (F, P) of the complex digit kernel where it beats the model
// by > 1% (scripts/tune_table.py, every fitting (F, P) timed on the sweep
// cells and configs, L2 flushed; profiles/r02_tune_table_aligned.json):
// {L, D, F, P}.  At L = 4, D = 32 the qd config (-5%) wins over the d = 31
// sweep cell (+3.6%).
static const int kTunedGeom[][4] = {
    {2, 16, 2, 2}, {2, 32, 2, 1}, {3, 16, 2, 2}, {3, 32, 1, 4}, {3, 128, 1, 1}, {4, 32, 2, 1},
    {5, 16, 1, 4}, {5, 32, 1, 2}, {5, 64, 1, 1}, {8, 16, 2, 4}, {10, 16, 2, 4}, {10, 32, 2, 2},
};

// The same for the real-system kernel (mdps_options.real; TUNE_REAL=1,
// profiles/r01_tune_table_real.json).
static const int kTunedGeomReal[][4] = {
    {2, 32, 2, 2},  {3, 16, 2, 4},  {3, 64, 2, 1},  {3, 128, 2, 1}, {4, 16, 2, 2},  {4, 32, 2, 2},
    {5, 16, 2, 2},  {5, 32, 2, 1},  {5, 64, 2, 1},  {8, 16, 2, 2},  {10, 16, 2, 4}, {10, 32, 2, 2},
    {10, 64, 2, 1},
};

// The same for the fused-parts kernel (conv_dig_fused.cuh, complex systems).
// (profiles/r02_tune_fused.json; D = 128 runs the model's choice, F = 2, P = 1)
static const int kTunedGeomFused[][4] = {
    {2, 16, 2, 8}, {2, 32, 2, 4}, {2, 64, 2, 2}, {3, 16, 2, 2}, {3, 32, 2, 1}, {3, 64, 2, 1},
    {4, 16, 2, 4}, {4, 32, 2, 2}, {4, 64, 2, 1}, {5, 16, 2, 2}, {5, 32, 2, 1}, {5, 64, 2, 1},
};

// The same with the fold parked in local memory (conv_fused_kernel<.., true>).
// (profiles/r02_tune_lpark.json)
static const int kTunedGeomFusedLpark[][4] = {
    {3, 16, 2, 2}, {3, 32, 2, 2}, {3, 64, 2, 2}, {3, 128, 2, 1}, {4, 16, 2, 2}, {4, 32, 2, 1}, {4, 64, 2, 1},
    {4, 128, 2, 1}, {5, 16, 2, 2}, {5, 32, 2, 1}, {5, 64, 2, 1},
};

// real: the real-system kernel (one part lane set) and its table; tuned:
// use the table; forceF/P > 0 restrict the search to that F / P
static DigGeom dig_geom(int L, int D, int regs_per_thread, int max_threads, bool real, int forceF = 0,
                        int forceP = 0, bool tuned = false, bool fused = false, bool lpark = false) {
    const int S = digits_for(L);
    const int T = (D + 1) / 2;
    const int NP = (real || fused) ? 1 : 2;  // lane sets per job (fused: both parts on one thread)
    DigGeom best{T, 1, 1, 32, 0, NP};
    double best_score = -1.0;
    if (tuned && forceF == 0 && forceP == 0) {
        auto pick = [&](const auto &table) {
            for (const auto &t : table)
                if (t[0] == L && t[1] == D) {
                    forceF = t[2];
                    forceP = t[3];
                }
        };
        if (fused && lpark) pick(kTunedGeomFusedLpark);
        else if (fused) pick(kTunedGeomFused);
        else if (real) pick(kTunedGeomReal);
        else pick(kTunedGeom);
    }
    // resident warps count up to 16 per SM; measured (profiles/r01_sweep.json
    // history): at L = 4, D >= 32 more terms per lane beat the 16th warp
    // (qd 1.03 -> 0.97 ms, d = 31 -12%, d = 63 -7%), elsewhere 16 is right
    const int warp_cap = (L == 4 && D >= 32) ? 12 : 16;
    for (int F = 1; F <= 8; F *= 2) {
        if (forceF > 0 && forceF != F) continue;
        for (int P = 1; P <= 32; P *= 2) {
            if (forceP > 0 && forceP != P) continue;
            DigGeom g;
            g.T = T;
            g.F = F;
            g.P = P;
            g.NP = NP;
            g.threads = NP * ((P * T * F + 31) / 32 * 32);  // each part's lane set whole warps
            if (g.threads > max_threads) continue;
            g.smem = fused ? conv_fused_smem(S, D, P, g.threads, lpark) : conv_dig_smem(S, D, P, g.threads);
            if (g.smem > 227 * 1024) continue;
            const int blocks_smem = (int)(228 * 1024 / (g.smem + 1024));
            const int blocks_regs = 65536 / (std::max(regs_per_thread, 32) * g.threads);
            const int blocks = std::min(std::min(blocks_smem, blocks_regs), 32);
            if (blocks < 1) continue;
            const int warps = std::min(blocks * g.threads / 32, 64);
            const int iters = (D + 1 + F - 1) / F;
            const double balance = (double)(D + 1) / (F * iters) * (double)(NP * P * T * F) / g.threads;
            const double amort = (double)iters / (iters + 3.0);
            const double score = std::min(warps, warp_cap) * balance * amort;
            if (score > best_score) {
                best_score = score;
                best = g;
            }
        }
    }
    return best;
}

// ---------------------------------------------------------------------------
template <int L>
struct ConvEft {
    static int run(double *pool, const int *jobs, int njobs, int D, cudaStream_t st) {
        if (njobs <= 0) return MDPS_OK;
        EftGeom g = eft_geom(L, D);
        auto kern = conv_eft_kernel<L>;
        if (g.smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
        const int blocks = (njobs + g.P - 1) / g.P;
        kern<<<blocks, g.threads, g.smem, st>>>(pool, jobs, njobs, D, g.T, g.P);
        CUDA_TRY(cudaGetLastError(), MDPS_ECUDA);
        return MDPS_OK;
    }
};

// fused-parts kernel (conv_dig_fused.cuh): complex systems with few digits.
// mode: 0 = never (part lanes), 1 = where measured faster (default), 2 = always
// where the kernel exists (L <= 5), 3 = always, with the fold parked in local
// memory; mdps_test_force_geometry's NP = 2 / 0 / 1 / 3
static int g_fused_mode = 1;
// measured (profiles/r02_tune_lpark.json, best geometry each): L = 3 -3..6%,
// L = 5 -6..8% but +6% at D = 128, L = 4 -0..1%; L = 2 not measured (AUTO runs
// the EFT kernel there)
static bool fused_lpark_default(int L, int D) { return L == 3 || L == 4 || (L == 5 && D < 128); }
static int g_small_levels = 1;  // wider geometry for levels below one wave (mdps_test_set_pdl bit 1 clears it)
static int g_balance_levels = 1;  // level balancing at create (mdps_test_set_pdl bit 2 clears it)
static int g_pdl = 1;  // programmatic dependent launch of the digit product levels (mdps_test_set_pdl)
static bool fused_default(int L, int D) {
    (void)D;
    return L <= 5;
}

template <int L, bool HAS_FUSED = (L <= 5)>
struct FusedKern {
    using KernT = void (*)(double *, int *, double *, const int *, int, int, int, int, int);
    static KernT get(int, bool) { return nullptr; }
};
template <int L>
struct FusedKern<L, true> {
    using KernT = void (*)(double *, int *, double *, const int *, int, int, int, int, int);
    static KernT get(int D, bool lpark) {
        if (lpark)
            return D == 16 ? conv_fused_kernel<L, 16, true> : D == 32 ? conv_fused_kernel<L, 32, true>
                 : D == 64 ? conv_fused_kernel<L, 64, true> : D == 128 ? conv_fused_kernel<L, 128, true>
                 : conv_fused_kernel<L, 0, true>;
        return D == 16 ? conv_fused_kernel<L, 16> : D == 32 ? conv_fused_kernel<L, 32>
             : D == 64 ? conv_fused_kernel<L, 64> : D == 128 ? conv_fused_kernel<L, 128>
             : conv_fused_kernel<L, 0>;
    }
};

template <int L>
struct ConvDig {
    using KernT = void (*)(double *, int *, double *, const int *, int, int, int, int, int);
    // kernel, launch geometry and jobs per wave of resident blocks for a level of njobs jobs
    static int geom(int njobs, int D, int real, KernT &kern, DigGeom &g, long long &wave_jobs) {
        const bool fused = !real && L <= 5 && (g_fused_mode >= 2 || (g_fused_mode == 1 && fused_default(L, D)));
        // (D >= 2: the emit scratch of D + 1 lanes must fit the job's operand buffers)
        const bool lpark = fused && D >= 2 && (g_fused_mode == 3 || (g_fused_mode == 1 && fused_lpark_default(L, D)));
        if (fused)  // complex systems, few digits: both parts of an output on one thread
            kern = FusedKern<L>::get(D, lpark);
        else if (real)  // real systems: one part, one product per term
            kern = D == 16 ? conv_dig_kernel<L, 16, true> : D == 32 ? conv_dig_kernel<L, 32, true>
                 : D == 64 ? conv_dig_kernel<L, 64, true> : D == 128 ? conv_dig_kernel<L, 128, true>
                 : conv_dig_kernel<L, 0, true>;
        else
            kern = D == 16 ? conv_dig_kernel<L, 16> : D == 32 ? conv_dig_kernel<L, 32> : D == 64 ? conv_dig_kernel<L, 64>
                 : D == 128 ? conv_dig_kernel<L, 128> : conv_dig_kernel<L, 0>;
        // geometry per (D, kernel), computed once per process under a lock
        static std::mutex mu;
        static DigGeom cache[4 * 257];
        static int cregs[4 * 257], cmaxt[4 * 257];
        static bool cached[4 * 257];
        // small levels (a level that cannot fill the GPU: the last levels of a
        // system whose monomials differ in length): the same kernel with 2x
        // and 4x the lanes per output pair, one job per block, and the jobs
        // one wave of each geometry holds — a level runs on the widest
        // geometry that still takes all its jobs in one wave (the results do
        // not depend on the geometry: exact accumulation)
        static DigGeom wide[4 * 257][2];
        static long long cap[4 * 257][3];  // jobs per wave: default, 2x, 4x
        const int key = D + (lpark ? 3 * 257 : fused ? 2 * 257 : real ? 257 : 0);
        int regs, maxt;
        {
            std::lock_guard<std::mutex> lk(mu);
            if (!cached[key]) {
                cudaFuncAttributes fa;
                regs = 255;
                maxt = 128;
                if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess) {
                    regs = fa.numRegs;
                    maxt = std::min(fa.maxThreadsPerBlock, 256);
                }
                cregs[key] = regs;
                cmaxt[key] = maxt;
                cache[key] = dig_geom(L, D, regs, maxt, real != 0, 0, 0, true, fused, lpark);
                if (cache[key].smem == 0)  // tuned entry does not fit
                    cache[key] = dig_geom(L, D, regs, maxt, real != 0, 0, 0, false, fused, lpark);
                int dev = 0, sms = 1;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                auto wave = [&](const DigGeom &q) -> long long {
                    if (q.smem == 0) return 0;
                    if (q.smem > 48 * 1024)
                        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)q.smem);
                    int per = 0;
                    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, q.threads, q.smem) != cudaSuccess) {
                        cudaGetLastError();
                        return 0;
                    }
                    return (long long)per * sms * q.P;
                };
                cap[key][0] = wave(cache[key]);
                for (int w = 0; w < 2; w++) {
                    const int Fw = cache[key].F << (w + 1);
                    wide[key][w] = Fw <= 8 ? dig_geom(L, D, regs, maxt, real != 0, Fw, 1, false, fused, lpark)
                                           : DigGeom{0, 0, 0, 0, 0, 0};
                    cap[key][w + 1] = wave(wide[key][w]);
                }
                cached[key] = true;
            }
            g = cache[key];
            regs = cregs[key];
            maxt = cmaxt[key];
            wave_jobs = cap[key][0];
            if (g_small_levels && njobs < cap[key][0]) {
                for (int w = 1; w >= 0; w--)
                    if (njobs <= cap[key][w + 1]) {
                        g = wide[key][w];
                        break;
                    }
            }
        }
        if (g_force_F > 0 || g_force_P > 0) {  // tuning: a forced (F, P), checked
            g = dig_geom(L, D, regs, maxt, real != 0, g_force_F, g_force_P, false, fused, lpark);
            if (g.smem == 0) { set_err("forced geometry does not fit"); return MDPS_EINVAL; }
        }
        return MDPS_OK;
    }

    static int run(double *dpool, int *epool, double *lpool, const int *jobs, int njobs, int D, int real,
                   cudaStream_t st) {
        if (njobs <= 0) return MDPS_OK;
        KernT kern;
        DigGeom g;
        long long wave_jobs = 0;
        const int rc = geom(njobs, D, real, kern, g, wave_jobs);
        if (rc != MDPS_OK) return rc;
        if (g.smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
        const int blocks = (njobs + g.P - 1) / g.P;
        // programmatic dependent launch: this level's blocks may be scheduled
        // while the previous kernel of the stream drains (they wait for its
        // completion before touching the pools: grid_dep_wait in the kernel)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)blocks);
        cfg.blockDim = dim3((unsigned)g.threads);
        cfg.dynamicSmemBytes = g.smem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = g_pdl ? 1 : 0;
        int T = g.T, F = g.F, P = g.P;
        CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, dpool, epool, lpool, jobs, njobs, D, T, F, P), MDPS_ECUDA);
        CUDA_TRY(cudaGetLastError(), MDPS_ECUDA);
        return MDPS_OK;
    }
};

// jobs one wave of resident blocks of the digit product kernel holds (default geometry)
template <int L>
struct ConvDigWave {
    static int run(int D, int real, long long *out) {
        typename ConvDig<L>::KernT kern;
        DigGeom g;
        long long wave = 0;
        const int rc = ConvDig<L>::geom(1 << 30, D, real, kern, g, wave);
        *out = wave;
        return rc;
    }
};

// the device-side job queue (queue_eft.cuh): one persistent launch
struct QueueGeom {
    int F, threads, blocks, tasks_per_ticket;
    size_t smem;
};

template <int L>
struct QueueEft {
    static int geom(int D, int njobs, int ntasks, QueueGeom &g) {
        g.F = g_force_queue_F > 0 ? queue_lanes(D, g_force_queue_F) : queue_lanes(D);
        g.threads = (2 * ((D + 1) / 2) * g.F + 31) / 32 * 32;
        g.tasks_per_ticket = std::max(1, g.threads / D);
        g.smem = (size_t)2 * (2 * L * D) * sizeof(double);
        auto kern = queue_eft_kernel<L>;
        if (g.smem > 48 * 1024 &&
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem) != cudaSuccess) {
            cudaGetLastError();
            set_err("queue kernel: shared memory does not fit");
            return MDPS_EINVAL;
        }
        int dev = 0, sms = 0, per = 0;
        CUDA_TRY(cudaGetDevice(&dev), MDPS_ECUDA);
        CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), MDPS_ECUDA);
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, g.threads, g.smem), MDPS_ECUDA);
        if (per < 1) { set_err("queue kernel does not fit on an SM"); return MDPS_EINVAL; }
        const long long tickets = (long long)njobs + (ntasks + g.tasks_per_ticket - 1) / g.tasks_per_ticket;
        // at most 4 blocks per SM: more only lengthen the launch and the
        // ticket traffic (dd: 592 vs 1184 blocks, scripts/queue_tune.py)
        g.blocks = (int)std::max(1LL, std::min<long long>(tickets, (long long)sms * std::min(per, 4)));
        if (g_force_queue_blocks > 0) g.blocks = std::min(g.blocks, g_force_queue_blocks);
        return MDPS_OK;
    }
    static int run(const QueueGeom &g, const double *x_in, double *pool, unsigned *flags, QueueCtl *ctl,
                   const int *jobs, int njobs, const int *tp, const int *es, const int *ew, int ntasks, int nvals,
                   int nx, int nready, int D, double *values, double *jac, long long *trace, cudaStream_t st) {
        queue_eft_kernel<L><<<g.blocks, g.threads, g.smem, st>>>(x_in, pool, flags, ctl, jobs, njobs, tp, es, ew,
                                                                  ntasks, nvals, g.tasks_per_ticket, nx, nready, D,
                                                                  g.F, values, jac, trace);
        CUDA_TRY(cudaGetLastError(), MDPS_ECUDA);
        return MDPS_OK;
    }
};

template <int L>
struct QueueGeomFn {
    static int run(int D, int njobs, int ntasks, QueueGeom &g) { return QueueEft<L>::geom(D, njobs, ntasks, g); }
};

template <int L>
struct AccumEft {
    // addition jobs: values [v0, v0 + nv) and Jacobian entries [j0, j0 + nj), one launch
    static int run(const double *pool, const int *tp, const int *es, const int *ew, int v0, int nv, int j0, int nj,
                   int n, int D, double *values, double *jac, cudaStream_t st) {
        if (nv <= 0 && nj <= 0) return MDPS_OK;
        const int gj = accum_lanes_jac(L, D);
        const long long vb = ((long long)std::max(nv, 0) * D * ACCUM_LANES_VALUE + 127) / 128;
        const long long jb = ((long long)std::max(nj, 0) * D * gj + 127) / 128;
        auto kern = gj == 1 ? accum_eft_kernel<L, 1> : accum_eft_kernel<L, 2>;
        kern<<<(unsigned)(vb + jb), 128, 0, st>>>(pool, tp, es, ew, v0, std::max(nv, 0), (int)vb, j0, std::max(nj, 0),
                                                  n, D, values, jac);
        CUDA_TRY(cudaGetLastError(), MDPS_ECUDA);
        return MDPS_OK;
    }
};

template <int L>
struct ToDigits {
    static int run(const double *src, int count, int D, double *dpool, int *epool, int slot0, cudaStream_t st) {
        if (count <= 0) return MDPS_OK;
        const long long total = (long long)count * D;
        const int blocks = (int)((total + 127) / 128);
        to_digits_kernel<L><<<blocks, 128, 0, st>>>(src, count, D, dpool, epool, slot0);
        CUDA_TRY(cudaGetLastError(), MDPS_ECUDA);
        return MDPS_OK;
    }
};

// ---------------------------------------------------------------------------
struct mdps_system {
    int n = 0, N = 0, D = 0, L = 0, M = 0, algo = MDPS_ALGO_DIGITS, S = 0;  // n variables, N polynomials
    int real = 0;  // mdps_options.real: every series real, one product per term
    int batch = 1; // mdps_options.batch: points per evaluation (n, N are per point)
    int use_graph = 0;
    int schedule = MDPS_SCHED_LEVELS;  // resolved: LEVELS or QUEUE
    unsigned *qflags = nullptr;        // QUEUE: per-slot ready flags (epochs)
    QueueCtl *qctl = nullptr;          // QUEUE: ticket counter and epoch
    QueueGeom qgeom{};
    long long *qtrace = nullptr;       // QUEUE diagnostics: [ticket][QUEUE_TRACE_STAMPS] ns (mdps_test_queue_trace)
    int64_t qtickets = 0;
    int64_t njobs = 0;
    int64_t nslots = 0, products = 0, add_terms = 0, add_terms_w = 0;  // add_terms_w: weight != 1
    // LEVELS: row chunks run one after the other, each its levels then its
    // addition-job ranges (schedule.hpp plan_memory); one chunk normally
    struct ChunkRun {
        std::vector<int64_t> lv_off, lv_cnt;  // in jobs
        int32_t task0[2], ntask[2];
    };
    std::vector<ChunkRun> chunks;
    int64_t pool_bytes = 0;
    std::vector<int64_t> level_cnt;  // jobs per DAG level (diagnostics)
    int ntasks = 0;
    // device
    double *pool = nullptr;  // EFT: limb planes [slot][2][L][D]; DIGITS: digit planes [slot][2][S][D]
    int *epool = nullptr;    // DIGITS: exponents [slot][2][D]
    int *jobs = nullptr;     // all levels, (in1, in2, out) triples
    int *task_ptr = nullptr, *ent_slot = nullptr, *ent_w = nullptr;
    double *lpool = nullptr;  // DIGITS: limb planes of the series the addition jobs sum [lslot][2][L][D]
    std::vector<std::pair<int32_t, int32_t>> x_lslots;  // (x index, lslot) of inputs summed directly
    double *host_in = nullptr;  // staging for the _host variant (device buffers)
    double *dev_in = nullptr, *dev_vals = nullptr, *dev_jac = nullptr;
    size_t device_bytes = 0;
    // CUDA graph cache
    cudaGraphExec_t gexec = nullptr;
    cudaGraph_t graph = nullptr;
    cudaStream_t cap_stream = nullptr;  // capture stream of the graph
    const void *g_in = nullptr, *g_vals = nullptr, *g_jac = nullptr;
    cudaStream_t g_stream = nullptr;
    // measurement: event pairs per launch group (kind 0 conv, 1 accum, 2 convert)
    int timing = 0;
    struct Mark { cudaEvent_t a, b; int kind; };
    std::vector<Mark> marks;
    int64_t timed_evals = 0;
};

static void drop_marks(mdps_system *s) {
    for (auto &m : s->marks) {
        cudaEventDestroy(m.a);
        cudaEventDestroy(m.b);
    }
    s->marks.clear();
}

// begin/end a timed launch group (no-op unless timing is enabled)
struct TimedGroup {
    mdps_system *s;
    cudaStream_t st;
    int kind;
    cudaEvent_t a = nullptr, b = nullptr;
    TimedGroup(mdps_system *s_, cudaStream_t st_, int kind_) : s(s_), st(st_), kind(kind_) {
        if (s->timing && cudaEventCreate(&a) == cudaSuccess && cudaEventCreate(&b) == cudaSuccess)
            cudaEventRecord(a, st);
    }
    ~TimedGroup() {
        if (a && b) {
            cudaEventRecord(b, st);
            s->marks.push_back({a, b, kind});
        }
    }
};

static void free_system(mdps_system *s) {
    if (!s) return;
    drop_marks(s);
    if (s->gexec) cudaGraphExecDestroy(s->gexec);
    if (s->graph) cudaGraphDestroy(s->graph);
    if (s->cap_stream) cudaStreamDestroy(s->cap_stream);
    cudaFree(s->pool);
    cudaFree(s->epool);
    cudaFree(s->jobs);
    cudaFree(s->task_ptr);
    cudaFree(s->ent_slot);
    cudaFree(s->ent_w);
    cudaFree(s->lpool);
    cudaFree(s->dev_in);
    cudaFree(s->dev_vals);
    cudaFree(s->dev_jac);
    cudaFree(s->qflags);
    cudaFree(s->qctl);
    cudaFree(s->qtrace);
    delete s;
}

template <typename T>
static bool dalloc(mdps_system *s, T **p, size_t count) {
    if (count == 0) count = 1;
    if (cudaMalloc((void **)p, count * sizeof(T)) != cudaSuccess) {
        cudaGetLastError();
        set_err("cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed");
        return false;
    }
    s->device_bytes += count * sizeof(T);
    return true;
}

extern "C" mdps_system *mdps_system_create_ex(const mdps_supports *sup, const int32_t *exponents,
                                              const double *coefficients, int32_t n, int32_t degree,
                                              int32_t limbs, const mdps_options *opt) {
    if (!sup) { set_err("NULL supports"); return nullptr; }
    if (n < 1) { set_err("n must be >= 1"); return nullptr; }
    if (degree < 0 || degree > 255) { set_err("degree must be in [0, 255]"); return nullptr; }
    if (!valid_limbs(limbs)) { set_err("limbs must be one of 2, 3, 4, 5, 8, 10"); return nullptr; }
    int algo = opt ? opt->algo : MDPS_ALGO_AUTO;
    if (algo != MDPS_ALGO_AUTO && algo != MDPS_ALGO_EFT && algo != MDPS_ALGO_DIGITS) {
        set_err("unknown algo");
        return nullptr;
    }
    const int D = degree + 1;
    const int real = opt ? (opt->real != 0) : 0;
    if (real && algo == MDPS_ALGO_EFT) { set_err("real systems need the digits algorithm"); return nullptr; }
    if (real && D > 128) { set_err("real systems need degree <= 127"); return nullptr; }
    if (algo == MDPS_ALGO_DIGITS && D > 128) { set_err("the digits algorithm supports degree <= 127"); return nullptr; }

    Schedule S;
    std::string err;
    if (!build_schedule(sup->n_polys, sup->poly_ptr, sup->mono_ptr, sup->vars, exponents, n, S, err)) {
        set_err(err);
        return nullptr;
    }
    if (S.M > 0 && !coefficients) { set_err("NULL coefficients"); return nullptr; }
    const int B = opt && opt->batch > 1 ? opt->batch : 1;
    if (opt && opt->batch < 0) { set_err("batch must be >= 1"); return nullptr; }
    // MDPS_ALGO_AUTO (measured): digits, except above degree 127
    // (digits cap) and at L = 2 below degree 63: with S = 7 digits a term is
    // short, and up to D = 32 the EFT kernel, whose operands are 2 limbs, is
    // level or ahead (d = 15 a tie, d = 31 0.61 vs 0.62 ms; dd itself and
    // batches of dd points run the EFT job queue); from D = 64 on the
    // fused-parts digit kernel wins (d = 63 1.97 vs 2.04 ms, d = 127 7.05 vs
    // 7.61); at L = 3 digits win from degree 15 on
    if (algo == MDPS_ALGO_AUTO)
        algo = D > 128 || (!real && limbs == 2 && D < 64) ? MDPS_ALGO_EFT : MDPS_ALGO_DIGITS;
    const int sched_opt = opt ? opt->schedule : MDPS_SCHED_AUTO;
    if (sched_opt != MDPS_SCHED_AUTO && sched_opt != MDPS_SCHED_LEVELS && sched_opt != MDPS_SCHED_QUEUE) {
        set_err("unknown schedule");
        return nullptr;
    }
    if (sched_opt == MDPS_SCHED_QUEUE && algo != MDPS_ALGO_EFT) {
        set_err("the job queue (MDPS_SCHED_QUEUE) runs the EFT algorithm only");
        return nullptr;
    }
    // AUTO: the queue for small systems on the EFT algorithm, where one level's
    // jobs cannot fill the GPU and the per-level launch + tail dominate
    // (measured)
    const int sched = sched_opt == MDPS_SCHED_QUEUE ||
                              (sched_opt == MDPS_SCHED_AUTO && algo == MDPS_ALGO_EFT &&
                               S.products * (opt && opt->batch > 1 ? opt->batch : 1) <= MDPS_QUEUE_MAX_PRODUCTS)
                          ? MDPS_SCHED_QUEUE : MDPS_SCHED_LEVELS;
    if (sched == MDPS_SCHED_LEVELS && algo == MDPS_ALGO_DIGITS && B == 1 && g_balance_levels) {
        // level balancing (schedule.hpp): summed-only products move from the
        // full early levels into later levels below one wave of the kernel
        long long wave = 0;
        if (dispatch_L<ConvDigWave>(limbs, D, real, &wave) == MDPS_OK && wave > 0) balance_levels(S, wave);
    }
    if (B > 1 && !replicate_schedule(S, n, B, err)) {
        set_err(err);
        return nullptr;
    }
    const bool eft = algo == MDPS_ALGO_EFT;
    const int Sd = eft ? 0 : digits_for(limbs);
    if (sched == MDPS_SCHED_LEVELS) {
        // memory plan: liveness reuse; then as few row chunks as keep the
        // pools within the budget (none by default)
        if (opt && opt->workspace_mb < 0) { set_err("workspace_mb must be >= 0"); return nullptr; }
        int64_t budget = (opt && opt->workspace_mb > 0) ? (int64_t)opt->workspace_mb << 20 : 0;
        if (budget == 0) {  // default: a quarter of the device memory free now
            size_t fr = 0, tot = 0;
            if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) budget = (int64_t)(fr / 4);
            cudaGetLastError();
        }
        for (int C = 1;; C++) {
            if (!plan_memory(S, n, C, eft, err)) {
                set_err(err);
                return nullptr;
            }
            if (budget == 0 || plan_bytes(S, Sd, limbs, D, eft) <= budget || C >= 64 || (int)S.chunks.size() < C ||
                B > 1)
                break;
        }
    } else if (!check_schedule(S, n, eft, err)) {
        set_err(err);
        return nullptr;
    }

    mdps_system *s = new (std::nothrow) mdps_system();
    if (!s) { set_err("host allocation failed"); return nullptr; }
    s->n = n;
    s->N = S.N;
    s->D = D;
    s->L = limbs;
    s->M = S.M;
    s->algo = algo;
    s->S = Sd;
    s->use_graph = opt ? opt->use_graph : 0;
    s->real = real;
    s->batch = B;
    s->nslots = S.planned ? S.dig_slots : S.nslots;
    s->products = S.products;
    s->add_terms = (int64_t)S.ent_slot.size();
    for (int32_t w : S.ent_w) s->add_terms_w += w != 1;
    s->ntasks = B * (S.N + S.N * n);
    s->schedule = sched;
    const int64_t nlimb = S.planned ? S.plan_nlimb : S.nlimb;

    std::vector<int32_t> alljobs;  // (in1, in2, out, code) per job, launch by launch
    if (S.planned) {
        for (auto &ch : S.chunks) {
            mdps_system::ChunkRun cr;
            for (auto &lv : ch.levels4) {
                cr.lv_off.push_back((int64_t)alljobs.size() / 4);
                cr.lv_cnt.push_back((int64_t)lv.size() / 4);
                alljobs.insert(alljobs.end(), lv.begin(), lv.end());
            }
            for (int r = 0; r < 2; r++) {
                cr.task0[r] = ch.task0[r];
                cr.ntask[r] = ch.ntask[r];
            }
            s->chunks.push_back(std::move(cr));
        }
    } else {
        for (auto &lv : S.levels4) alljobs.insert(alljobs.end(), lv.begin(), lv.end());
    }
    for (auto &lv : S.levels4) s->level_cnt.push_back((int64_t)lv.size() / 4);  // per DAG level (diagnostics)
    s->njobs = (int64_t)alljobs.size() / 4;
    if (sched == MDPS_SCHED_QUEUE) {
        if (s->njobs + (int64_t)s->ntasks >= (int64_t)INT32_MAX / 2) { set_err("queue: too many jobs"); free_system(s); return nullptr; }
        const int rc = dispatch_L<QueueGeomFn>(limbs, D, (int)s->njobs, s->ntasks, s->qgeom);
        s->qtickets = s->njobs + (s->ntasks + s->qgeom.tasks_per_ticket - 1) / s->qgeom.tasks_per_ticket;
        if (rc != MDPS_OK || !dalloc(s, &s->qflags, (size_t)s->nslots) || !dalloc(s, &s->qctl, 1) ||
            cudaMemset(s->qflags, 0, sizeof(unsigned) * (size_t)std::max<int64_t>(1, s->nslots)) != cudaSuccess ||
            cudaMemset(s->qctl, 0, sizeof(QueueCtl)) != cudaSuccess) {
            if (g_err.empty()) set_err("queue setup failed");
            free_system(s);
            return nullptr;
        }
    }
    const size_t ser = algo == MDPS_ALGO_DIGITS ? dig_slot_stride(s->S, D) : (size_t)2 * limbs * D;  // doubles per slot
    const size_t before_pools = s->device_bytes;
    if (!dalloc(s, &s->pool, ser * (size_t)s->nslots) ||
        (algo == MDPS_ALGO_DIGITS && !dalloc(s, &s->epool, dig_exp_stride(D) * s->nslots)) ||
        (algo == MDPS_ALGO_DIGITS && !dalloc(s, &s->lpool, (size_t)2 * limbs * D * nlimb))) {
        free_system(s);
        return nullptr;
    }
    s->pool_bytes = (int64_t)(s->device_bytes - before_pools);
    const std::vector<int32_t> &ents = S.planned ? S.plan_ent : (eft ? S.ent_slot : S.ent_lslot);
    if (!dalloc(s, &s->jobs, alljobs.size()) || !dalloc(s, &s->task_ptr, S.task_ptr.size()) ||
        !dalloc(s, &s->ent_slot, ents.size()) || !dalloc(s, &s->ent_w, S.ent_w.size())) {
        free_system(s);
        return nullptr;
    }
    auto up = [&](void *dst, const void *src, size_t bytes) {
        return bytes == 0 || cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
    };
    const size_t limb_ser = (size_t)2 * limbs * D;
    bool ok = up(s->jobs, alljobs.data(), alljobs.size() * 4) &&
              up(s->task_ptr, S.task_ptr.data(), S.task_ptr.size() * 4) &&
              up(s->ent_slot, ents.data(), ents.size() * 4) &&
              up(s->ent_w, S.ent_w.data(), S.ent_w.size() * 4);
    if (ok && algo == MDPS_ALGO_DIGITS) {
        // summed coefficient series (constant terms, m = 1 without common
        // factor) are copied once into the limb pool; summed inputs x_j (none
        // with the current DAG) are copied at every eval
        const int64_t nx = (int64_t)B * n;
        for (auto &fl : S.fixed_limb) {
            if (fl.first < nx)
                s->x_lslots.emplace_back(fl.first, fl.second);
            else
                ok = ok && up(s->lpool + (size_t)fl.second * limb_ser, coefficients + (size_t)(fl.first - nx) * limb_ser,
                              limb_ser * 8);
        }
    }
    if (ok && S.M > 0) {
        if (algo == MDPS_ALGO_EFT) {
            ok = up(s->pool + (size_t)B * n * ser, coefficients, (size_t)S.M * limb_ser * 8);
        } else {
            double *tmp = nullptr;
            ok = cudaMalloc((void **)&tmp, (size_t)S.M * limb_ser * 8) == cudaSuccess &&
                 up(tmp, coefficients, (size_t)S.M * limb_ser * 8);
            if (ok) {
                const int rc = dispatch_L<ToDigits>(limbs, (const double *)tmp, S.M, D, s->pool, s->epool, B * n,
                                                    (cudaStream_t)0);
                ok = rc == MDPS_OK && cudaDeviceSynchronize() == cudaSuccess;
            }
            cudaFree(tmp);
        }
    }
    if (!ok) {
        cudaGetLastError();
        if (g_err.empty()) set_err("uploading the system to the device failed");
        free_system(s);
        return nullptr;
    }
    return s;
}

extern "C" mdps_system *mdps_system_create(const mdps_supports *sup, const int32_t *exponents,
                                           const double *coefficients, int32_t n, int32_t degree,
                                           int32_t limbs) {
    return mdps_system_create_ex(sup, exponents, coefficients, n, degree, limbs, nullptr);
}

extern "C" void mdps_system_destroy(mdps_system *s) {
    if (!s) return;
    cudaDeviceSynchronize();
    free_system(s);
}

template <int L>
struct QueueRun {
    static int run(mdps_system *s, const double *in, double *vals, double *jac, cudaStream_t st) {
        const int nx = s->n * s->batch;
        return QueueEft<L>::run(s->qgeom, in, s->pool, s->qflags, s->qctl, s->jobs, (int)s->njobs, s->task_ptr,
                                s->ent_slot, s->ent_w, s->ntasks, s->N * s->batch, nx, nx + s->M, s->D, vals, jac,
                                s->qtrace, st);
    }
};

// the launch sequence of one eval (also what the CUDA graph captures)
static int enqueue(mdps_system *s, const double *in, double *vals, double *jac, cudaStream_t st) {
    const int L = s->L, D = s->D, n = s->n * s->batch;  // input series of all points
    int rc;
    if (s->timing) s->timed_evals++;
    if (s->schedule == MDPS_SCHED_QUEUE) {
        // one persistent launch: products and additions, x read in place
        TimedGroup tg(s, st, 0);
        return dispatch_L<QueueRun>(L, s, in, vals, jac, st);
    }
    const bool eft = s->algo == MDPS_ALGO_EFT;
    {
        TimedGroup tg(s, st, 2);
        if (eft) {
            CUDA_TRY(cudaMemcpyAsync(s->pool, in, (size_t)n * 2 * L * D * 8, cudaMemcpyDeviceToDevice, st),
                     MDPS_ECUDA);
        } else {
            rc = dispatch_L<ToDigits>(L, in, n, D, s->pool, s->epool, 0, st);
            if (rc) return rc;
            for (auto &xl : s->x_lslots)
                CUDA_TRY(cudaMemcpyAsync(s->lpool + (size_t)xl.second * 2 * L * D, in + (size_t)xl.first * 2 * L * D,
                                         (size_t)2 * L * D * 8, cudaMemcpyDeviceToDevice, st),
                         MDPS_ECUDA);
        }
    }
    // chunk by chunk (normally one): its product levels, then its addition
    // jobs, which read the limb pool (EFT: the one pool) the products wrote
    for (const auto &ch : s->chunks) {
        for (size_t lv = 0; lv < ch.lv_cnt.size(); lv++) {
            TimedGroup tg(s, st, 0);
            const int *jb = (const int *)(s->jobs + 4 * ch.lv_off[lv]);
            rc = eft ? dispatch_L<ConvEft>(L, s->pool, jb, (int)ch.lv_cnt[lv], D, st)
                     : dispatch_L<ConvDig>(L, s->pool, s->epool, s->lpool, jb, (int)ch.lv_cnt[lv], D, s->real, st);
            if (rc) return rc;
        }
        TimedGroup tg(s, st, 1);
        {
            // the chunk's value jobs and Jacobian jobs (one chunk: task range 0
            // holds both kinds, values first)
            const int NB = s->N * s->batch;
            int v0 = ch.task0[0], nv = ch.ntask[0], j0 = ch.task0[1], nj = ch.ntask[1];
            if (s->chunks.size() == 1) {
                nv = std::min(ch.ntask[0], NB);
                j0 = NB;
                nj = ch.ntask[0] - nv;
            }
            rc = dispatch_L<AccumEft>(L, (const double *)(eft ? s->pool : s->lpool), (const int *)s->task_ptr,
                                      (const int *)s->ent_slot, (const int *)s->ent_w, v0, nv, j0, nj, NB, D, vals,
                                      jac, st);
            if (rc) return rc;
        }
    }
    return MDPS_OK;
}

extern "C" int mdps_system_set_timing(mdps_system *s, int32_t enable) {
    if (!s) {
        set_err("NULL argument");
        return MDPS_EINVAL;
    }
    s->timing = enable ? 1 : 0;
    return MDPS_OK;
}

extern "C" int mdps_system_timing(mdps_system *s, mdps_timing *out, int32_t reset) {
    if (!s || !out) {
        set_err("NULL argument");
        return MDPS_EINVAL;
    }
    memset(out, 0, sizeof *out);
    for (auto &m : s->marks) {
        CUDA_TRY(cudaEventSynchronize(m.b), MDPS_ECUDA);
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, m.a, m.b), MDPS_ECUDA);
        if (m.kind == 0) { out->conv_ms += ms; out->conv_launches++; }
        else if (m.kind == 1) { out->accum_ms += ms; out->accum_launches++; }
        else { out->convert_ms += ms; out->convert_launches++; }
    }
    out->evals = s->timed_evals;
    if (reset) {
        drop_marks(s);
        s->timed_evals = 0;
    }
    return MDPS_OK;
}

static bool overlaps(const void *a, size_t na, const void *b, size_t nb) {
    const char *x = (const char *)a, *y = (const char *)b;
    return x < y + nb && y < x + na;
}

extern "C" int mdps_eval_diff(mdps_system *s, const double *in, double *vals, double *jac, mdps_stream_t stream) {
    if (!s || !in || !vals || !jac) {
        set_err("NULL argument");
        return MDPS_EINVAL;
    }
    const size_t ser = (size_t)2 * s->L * s->D * 8;
    const size_t nin = ser * s->n * s->batch, nval = ser * s->N * s->batch, njac = ser * s->N * s->n * s->batch;
    if (overlaps(in, nin, vals, nval) || overlaps(in, nin, jac, njac) || overlaps(vals, nval, jac, njac)) {
        set_err("outputs alias each other or the input");
        return MDPS_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (!s->use_graph || s->timing) return enqueue(s, in, vals, jac, st);
    if (!s->gexec || s->g_in != in || s->g_vals != vals || s->g_jac != jac) {
        if (s->gexec) { cudaGraphExecDestroy(s->gexec); s->gexec = nullptr; }
        if (s->graph) { cudaGraphDestroy(s->graph); s->graph = nullptr; }
        // capture on the system's own stream (the caller's may be the legacy
        // default stream, which cannot be captured); the graph then launches
        // on the caller's stream
        if (!s->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking), MDPS_ECUDA);
        CUDA_TRY(cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal), MDPS_ECUDA);
        const int rc = enqueue(s, in, vals, jac, s->cap_stream);
        cudaGraph_t g = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(s->cap_stream, &g);
        if (rc != MDPS_OK) { if (g) cudaGraphDestroy(g); return rc; }
        if (ce != cudaSuccess) { set_err(std::string("graph capture: ") + cudaGetErrorString(ce)); return MDPS_ECUDA; }
        s->graph = g;
        CUDA_TRY(cudaGraphInstantiate(&s->gexec, g, 0), MDPS_ECUDA);
        s->g_in = in;
        s->g_vals = vals;
        s->g_jac = jac;
        s->g_stream = st;
    }
    CUDA_TRY(cudaGraphLaunch(s->gexec, st), MDPS_ECUDA);
    return MDPS_OK;
}

extern "C" int mdps_eval_diff_host(mdps_system *s, const double *in_h, double *vals_h, double *jac_h,
                                   mdps_stream_t stream) {
    if (!s || !in_h || !vals_h || !jac_h) {
        set_err("NULL argument");
        return MDPS_EINVAL;
    }
    const size_t ser = (size_t)2 * s->L * s->D;
    if (!s->dev_in) {
        if (!dalloc(s, &s->dev_in, ser * s->n * s->batch) || !dalloc(s, &s->dev_vals, ser * s->N * s->batch) ||
            !dalloc(s, &s->dev_jac, ser * s->N * s->n * s->batch))
            return MDPS_ENOMEM;
    }
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_TRY(cudaMemcpyAsync(s->dev_in, in_h, ser * s->n * s->batch * 8, cudaMemcpyHostToDevice, st), MDPS_ECUDA);
    int rc = mdps_eval_diff(s, s->dev_in, s->dev_vals, s->dev_jac, stream);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(vals_h, s->dev_vals, ser * s->N * s->batch * 8, cudaMemcpyDeviceToHost, st),
             MDPS_ECUDA);
    CUDA_TRY(cudaMemcpyAsync(jac_h, s->dev_jac, ser * s->N * s->n * s->batch * 8, cudaMemcpyDeviceToHost, st),
             MDPS_ECUDA);
    CUDA_TRY(cudaStreamSynchronize(st), MDPS_ECUDA);
    return MDPS_OK;
}

// FP64 instruction counts
static int64_t conv_ops_per_product(int algo, int L, int D) {
    const int64_t terms = (int64_t)D * (D + 1) / 2;
    if (algo == MDPS_ALGO_EFT) return terms * 4 * ops_bins_fma(L);
    const int64_t S = digits_for(L);
    return terms * 2 * S * (S + 1);  // one DFMA per digit pair, 2 real products per part
}

// shape of a system for solve.cu (the Newton step checks it against the solver)
int mdps_internal_system_shape(const mdps_system *s, int *N, int *n, int *D, int *L) {
    if (!s) return MDPS_EINVAL;
    *N = s->batch == 1 ? s->N : -1;  // the Newton step works on one point
    *n = s->n;
    *D = s->D;
    *L = s->L;
    return MDPS_OK;
}

extern "C" int mdps_system_stats(const mdps_system *s, mdps_stats *out) {
    if (!s || !out) {
        set_err("NULL argument");
        return MDPS_EINVAL;
    }
    memset(out, 0, sizeof *out);
    out->products = s->products;
    out->add_terms = s->add_terms;
    out->fp64_ops_conv = s->products * conv_ops_per_product(s->algo, s->L, s->D) / (s->real ? 4 : 1);
    // both algorithms sum with accum_eft_kernel (EFT bins over limb planes):
    // bins_add per unit-weight term, bins_add_scaled per weighted one (a_l >= 2)
    const int64_t add_ops = ((s->add_terms - s->add_terms_w) * ops_bins_add(s->L) +
                             s->add_terms_w * ops_bins_add_scaled(s->L)) * s->D * 2;
    out->fp64_ops_total = out->fp64_ops_conv + add_ops;
    const int64_t ser = (int64_t)2 * s->L * s->D * 8;
    out->compulsory_bytes = ser * (((int64_t)s->n + s->N + (int64_t)s->N * s->n) * s->batch + s->M);
    out->levels = (int32_t)s->level_cnt.size();
    out->algo = s->algo;
    out->digits = s->S;
    int32_t launches = 1;  // QUEUE: one persistent launch
    if (s->schedule != MDPS_SCHED_QUEUE) {
        launches = 1;  // input conversion / copy
        for (const auto &ch : s->chunks) launches += (int32_t)ch.lv_cnt.size() + (ch.ntask[0] > 0 || ch.ntask[1] > 0);
    }
    out->launches = launches;
    out->schedule = s->schedule;
    out->chunks = (int32_t)std::max<size_t>(1, s->chunks.size());
    out->pool_bytes = s->pool_bytes;
    out->workspace_bytes = s->device_bytes;
    out->n = s->n;
    out->n_polys = s->N;
    out->degree = s->D - 1;
    out->limbs = s->L;
    out->batch = s->batch;
    return MDPS_OK;
}

extern "C" int mdps_system_level_jobs(const mdps_system *s, int64_t *jobs, int32_t maxl) {
    if (!s || !jobs) {
        set_err("NULL argument");
        return MDPS_EINVAL;
    }
    const int nl = (int)s->level_cnt.size();
    for (int i = 0; i < nl && i < maxl; i++) jobs[i] = s->level_cnt[i];
    return nl;
}

// ---------------------------------------------------------------------------
// test entry points (include/mdps_test.h)
template <int L>
struct MdOp {
    static int run(int op, const double *a, const double *b, double *c, int count, cudaStream_t st);
};

template <int L>
__global__ void md_op_kernel(int op, const double *a, const double *b, double *c, int count) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= count) return;
    double x[L], y[L], z[L];
#pragma unroll
    for (int p = 0; p < L; p++) {
        x[p] = a[(size_t)g * L + p];
        y[p] = b[(size_t)g * L + p];
    }
    if (op == 0) md_add<L>(x, y, z);
    else md_mul<L>(x, y, z);
#pragma unroll
    for (int p = 0; p < L; p++) c[(size_t)g * L + p] = z[p];
}

template <int L>
int MdOp<L>::run(int op, const double *a, const double *b, double *c, int count, cudaStream_t st) {
    md_op_kernel<L><<<(count + 127) / 128, 128, 0, st>>>(op, a, b, c, count);
    CUDA_TRY(cudaGetLastError(), MDPS_ECUDA);
    return MDPS_OK;
}

template <int L>
__global__ void norm2sq_kernel(const double *v, int count, double *out) {
    // one warp: lane j accumulates entries j, j+32, ... in level bins, then
    // lane 0 merges the 32 partial bins in order (deterministic)
    __shared__ double part[32][L + 1];
    double B[L + 1];
    md_zero(B);
    for (int j = threadIdx.x; j < count; j += 32) {
        double re[L], im[L];
#pragma unroll
        for (int p = 0; p < L; p++) {
            re[p] = v[((size_t)j * 2 + 0) * L + p];
            im[p] = v[((size_t)j * 2 + 1) * L + p];
        }
        bins_fma<L>(B, re, re);
        bins_fma<L>(B, im, im);
    }
#pragma unroll
    for (int p = 0; p <= L; p++) part[threadIdx.x][p] = B[p];
    __syncwarp();
    if (threadIdx.x == 0) {
        double C[L + 1];
        md_zero(C);
        for (int w = 0; w < 32; w++) {
            double t[L + 1], lim[L];
#pragma unroll
            for (int p = 0; p <= L; p++) t[p] = part[w][p];
            md_renorm(t, lim);
            bins_add<L>(C, lim);
        }
        double r[L];
        md_renorm(C, r);
#pragma unroll
        for (int p = 0; p < L; p++) out[p] = r[p];
    }
}

template <int L>
struct Norm2sq {
    static int run(const double *v, int count, double *out, cudaStream_t st) {
        norm2sq_kernel<L><<<1, 32, 0, st>>>(v, count, out);
        CUDA_TRY(cudaGetLastError(), MDPS_ECUDA);
        return MDPS_OK;
    }
};

template <int L>
struct Roundtrip {
    static int run(const double *x, double *y, int count, int D, cudaStream_t st) {
        const long long total = (long long)count * D;
        digits_roundtrip_kernel<L><<<(int)((total + 127) / 128), 128, 0, st>>>(x, y, count, D);
        CUDA_TRY(cudaGetLastError(), MDPS_ECUDA);
        return MDPS_OK;
    }
};

template <int L>
struct SeriesMulDig {
    // stage x and y into a scratch digit pool; the product kernel writes the
    // limbs of each product straight into z (job code: limb slot c, no digits)
    static int run(const double *x, const double *y, double *z, int count, int D, cudaStream_t st) {
        constexpr int S = digits_for(L);
        double *dp = nullptr;
        int *ep = nullptr, *jobs = nullptr;
        const size_t slots = (size_t)3 * count;
        int rc = MDPS_OK;
        std::vector<int> hj(4 * (size_t)count);
        for (int c = 0; c < count; c++) {
            hj[4 * c] = c;
            hj[4 * c + 1] = count + c;
            hj[4 * c + 2] = 2 * count + c;
            hj[4 * c + 3] = (c << 2) | 2;
        }
        if (cudaMalloc((void **)&dp, slots * dig_slot_stride(S, D) * 8) != cudaSuccess ||
            cudaMalloc((void **)&ep, slots * dig_exp_stride(D) * 4) != cudaSuccess ||
            cudaMalloc((void **)&jobs, hj.size() * 4) != cudaSuccess) {
            cudaGetLastError();
            set_err("cudaMalloc failed");
            rc = MDPS_ENOMEM;
        }
        if (!rc) {
            cudaMemcpyAsync(jobs, hj.data(), hj.size() * 4, cudaMemcpyHostToDevice, st);
            rc = ToDigits<L>::run(x, count, D, dp, ep, 0, st);
            if (!rc) rc = ToDigits<L>::run(y, count, D, dp, ep, count, st);
            if (!rc) rc = ConvDig<L>::run(dp, ep, z, jobs, count, D, 0, st);
            if (!rc && cudaStreamSynchronize(st) != cudaSuccess) {
                set_err("series_mul kernel failed");
                rc = MDPS_ECUDA;
            }
        }
        cudaFree(dp);
        cudaFree(ep);
        cudaFree(jobs);
        return rc;
    }
};

template <int L>
struct SeriesMulEft {
    static int run(const double *x, const double *y, double *z, int count, int D, cudaStream_t st) {
        const size_t ser = (size_t)2 * L * D;
        double *pool = nullptr;
        int *jobs = nullptr;
        std::vector<int> hj(4 * (size_t)count);
        for (int c = 0; c < count; c++) {
            hj[4 * c] = c;
            hj[4 * c + 1] = count + c;
            hj[4 * c + 2] = 2 * count + c;
            hj[4 * c + 3] = 0;
        }
        if (cudaMalloc((void **)&pool, 3 * ser * count * 8) != cudaSuccess ||
            cudaMalloc((void **)&jobs, hj.size() * 4) != cudaSuccess) {
            cudaGetLastError();
            cudaFree(pool);
            set_err("cudaMalloc failed");
            return MDPS_ENOMEM;
        }
        cudaMemcpyAsync(jobs, hj.data(), hj.size() * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(pool, x, ser * count * 8, cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(pool + ser * count, y, ser * count * 8, cudaMemcpyDeviceToDevice, st);
        int rc = ConvEft<L>::run(pool, jobs, count, D, st);
        if (!rc) cudaMemcpyAsync(z, pool + 2 * ser * count, ser * count * 8, cudaMemcpyDeviceToDevice, st);
        if (!rc && cudaStreamSynchronize(st) != cudaSuccess) {
            set_err("series_mul kernel failed");
            rc = MDPS_ECUDA;
        }
        cudaFree(pool);
        cudaFree(jobs);
        return rc;
    }
};

extern "C" int mdps_test_series_mul(const double *x, const double *y, double *z, int32_t count, int32_t degree,
                                    int32_t limbs, int32_t algo, mdps_stream_t stream) {
    if (!x || !y || !z || count < 0 || degree < 0 || degree > 255 || !valid_limbs(limbs)) {
        set_err("invalid argument");
        return MDPS_EINVAL;
    }
    if (count == 0) return MDPS_OK;
    const int D = degree + 1;
    if (algo == MDPS_ALGO_EFT) return dispatch_L<SeriesMulEft>(limbs, x, y, z, (int)count, D, (cudaStream_t)stream);
    if (D > 128) { set_err("digits: degree <= 127"); return MDPS_EINVAL; }
    return dispatch_L<SeriesMulDig>(limbs, x, y, z, (int)count, D, (cudaStream_t)stream);
}

extern "C" int mdps_test_md_op(int32_t op, const double *a, const double *b, double *c, int32_t count,
                               int32_t limbs, mdps_stream_t stream) {
    if (!a || !b || !c || count < 0 || (op != 0 && op != 1) || !valid_limbs(limbs)) {
        set_err("invalid argument");
        return MDPS_EINVAL;
    }
    if (count == 0) return MDPS_OK;
    return dispatch_L<MdOp>(limbs, (int)op, a, b, c, (int)count, (cudaStream_t)stream);
}

extern "C" int mdps_test_norm2sq(const double *v, int32_t count, int32_t limbs, double *out, mdps_stream_t stream) {
    if (!v || !out || count < 0 || !valid_limbs(limbs)) {
        set_err("invalid argument");
        return MDPS_EINVAL;
    }
    return dispatch_L<Norm2sq>(limbs, v, (int)count, out, (cudaStream_t)stream);
}

extern "C" int mdps_test_digits_roundtrip(const double *x, double *y, int32_t count, int32_t degree, int32_t limbs,
                                          mdps_stream_t stream) {
    if (!x || !y || count < 0 || degree < 0 || !valid_limbs(limbs)) {
        set_err("invalid argument");
        return MDPS_EINVAL;
    }
    if (count == 0) return MDPS_OK;
    return dispatch_L<Roundtrip>(limbs, x, y, (int)count, (int)degree + 1, (cudaStream_t)stream);
}

// FP64 peak: 8 independent DFMA chains per thread, 4 blocks of 256 per SM
__global__ void fp64_peak_kernel(int64_t iters, double *sink) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
    double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
    const double m = 0.999999999, c = 1e-12;
    for (int64_t i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 16; u++) {
            a0 = __fma_rn(a0, m, c); a1 = __fma_rn(a1, m, c); a2 = __fma_rn(a2, m, c); a3 = __fma_rn(a3, m, c);
            a4 = __fma_rn(a4, m, c); a5 = __fma_rn(a5, m, c); a6 = __fma_rn(a6, m, c); a7 = __fma_rn(a7, m, c);
        }
    }
    const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678) sink[0] = s;
}

extern "C" int mdps_test_force_geometry(int32_t F, int32_t P, int32_t NP) {
    if (F < 0 || F > 8 || (F & (F - 1)) || P < 0 || P > 32 || (P & (P - 1)) || NP < 0 || NP > 3) {
        set_err("forced geometry: F in {0,1,2,4,8}, P in {0,1,...,32} (powers of two), NP in {0,1,2,3}");
        return MDPS_EINVAL;
    }
    g_force_F = F;
    g_force_P = P;
    g_force_NP = NP;
    g_fused_mode = NP == 1 ? 2 : NP == 3 ? 3 : (NP == 2 ? 0 : 1);
    return MDPS_OK;
}

extern "C" int mdps_test_set_pdl(int32_t enable) {
    g_pdl = (enable & 1) ? 1 : 0;
    g_small_levels = (enable & 2) ? 0 : 1;
    g_balance_levels = (enable & 4) ? 0 : 1;
    return MDPS_OK;
}

extern "C" int mdps_fp64_peak(int64_t iters, double *inst_per_s, mdps_stream_t stream) {
    if (!inst_per_s || iters < 1) {
        set_err("invalid argument");
        return MDPS_EINVAL;
    }
    int dev = 0, sms = 0;
    CUDA_TRY(cudaGetDevice(&dev), MDPS_ECUDA);
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), MDPS_ECUDA);
    double *sink = nullptr;
    CUDA_TRY(cudaMalloc((void **)&sink, 8), MDPS_ECUDA);
    cudaStream_t st = (cudaStream_t)stream;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 4, threads = 256;
    fp64_peak_kernel<<<blocks, threads, 0, st>>>(iters / 8 + 1, sink);  // warm-up
    cudaEventRecord(e0, st);
    fp64_peak_kernel<<<blocks, threads, 0, st>>>(iters, sink);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    CUDA_TRY(cudaGetLastError(), MDPS_ECUDA);
    const double inst = (double)blocks * threads * (double)iters * 16.0 * 8.0;
    *inst_per_s = inst / (ms * 1e-3);
    return MDPS_OK;
}

// queue diagnostics: enable the per-ticket trace, or read it back after a
// synchronize; the geometry knobs apply to systems created afterwards
extern "C" int mdps_test_queue_config(int32_t max_blocks, int32_t lanes) {
    if (max_blocks < 0 || lanes < 0 || lanes > 32 || (lanes & (lanes - 1))) {
        set_err("queue config: max_blocks >= 0, lanes a power of two <= 32 (0 = default)");
        return MDPS_EINVAL;
    }
    g_force_queue_blocks = max_blocks;
    g_force_queue_F = lanes;
    return MDPS_OK;
}

extern "C" int mdps_test_queue_trace(mdps_system *s, int32_t enable, int64_t *out, int32_t max_tickets) {
    if (!s) { set_err("NULL system"); return MDPS_EINVAL; }
    if (s->schedule != MDPS_SCHED_QUEUE) { set_err("not a queue-scheduled system"); return MDPS_EINVAL; }
    if (enable > 0 && !s->qtrace) {
        if (!dalloc(s, &s->qtrace, (size_t)QUEUE_TRACE_STAMPS * s->qtickets)) return MDPS_ENOMEM;
        CUDA_TRY(cudaMemset(s->qtrace, 0, sizeof(long long) * QUEUE_TRACE_STAMPS * (size_t)s->qtickets), MDPS_ECUDA);
    }
    if (enable == 0 && s->qtrace) {
        cudaDeviceSynchronize();
        cudaFree(s->qtrace);
        s->qtrace = nullptr;
    }
    if (out && s->qtrace) {
        const int64_t cnt = std::min<int64_t>(s->qtickets, max_tickets);
        CUDA_TRY(cudaDeviceSynchronize(), MDPS_ECUDA);
        CUDA_TRY(cudaMemcpy(out, s->qtrace, sizeof(long long) * QUEUE_TRACE_STAMPS * (size_t)cnt,
                            cudaMemcpyDeviceToHost), MDPS_ECUDA);
        return (int)cnt;
    }
    return (int)s->qtickets;
}

// Host-only: level balancing (schedule.hpp balance_levels) of a system's
// schedule with `min_jobs` jobs per level as the target, then the checks and
// the memory plan of mdps_test_plan.  before / after: product jobs per level
// (up to max_levels each); *moved: jobs moved; *same_jobs: 1 if the balanced
// levels hold exactly the jobs of the original ones, every moved job summed
// only, none moved to an earlier level.  Returns the number of levels, or
// MDPS_EINVAL (a failed check included).
extern "C" int mdps_test_balance(const mdps_supports *sup, const int32_t *exponents, int32_t n, int64_t min_jobs,
                                 int64_t *before, int64_t *after, int32_t max_levels, int64_t *moved,
                                 int32_t *same_jobs) {
    if (!sup || !before || !after || !moved || !same_jobs || n < 1 || max_levels < 1) {
        set_err("invalid argument");
        return MDPS_EINVAL;
    }
    Schedule S;
    std::string err;
    if (!build_schedule(sup->n_polys, sup->poly_ptr, sup->mono_ptr, sup->vars, exponents, n, S, err)) {
        set_err(err);
        return MDPS_EINVAL;
    }
    const auto old4 = S.levels4;
    *moved = balance_levels(S, min_jobs);
    const int nl = (int)S.levels4.size();
    // job -> level maps (a job is named by its output slot)
    std::vector<std::pair<int32_t, int32_t>> a, b;  // (out, level)
    for (int lv = 0; lv < (int)old4.size(); lv++)
        for (size_t q = 0; q < old4[(size_t)lv].size(); q += 4) a.push_back({old4[(size_t)lv][q + 2], lv});
    for (int lv = 0; lv < nl; lv++)
        for (size_t q = 0; q < S.levels4[(size_t)lv].size(); q += 4) b.push_back({S.levels4[(size_t)lv][q + 2], lv});
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    bool same = a.size() == b.size() && old4.size() == S.levels4.size() && S.levels.size() == S.levels4.size();
    int64_t changed = 0;
    for (size_t i = 0; same && i < a.size(); i++) {
        same = a[i].first == b[i].first && b[i].second >= a[i].second;
        changed += a[i].second != b[i].second;
    }
    for (int lv = 0; same && lv < nl; lv++) {
        same = S.levels[(size_t)lv].size() / 3 == S.levels4[(size_t)lv].size() / 4;
        for (size_t q = 0, r = 0; same && q < S.levels4[(size_t)lv].size(); q += 4, r += 3)
            same = S.levels4[(size_t)lv][q] == S.levels[(size_t)lv][r] &&
                   S.levels4[(size_t)lv][q + 1] == S.levels[(size_t)lv][r + 1] &&
                   S.levels4[(size_t)lv][q + 2] == S.levels[(size_t)lv][r + 2];
    }
    *same_jobs = same && changed == *moved ? 1 : 0;
    for (int lv = 0; lv < max_levels; lv++) {
        before[lv] = lv < (int)old4.size() ? (int64_t)(old4[(size_t)lv].size() / 4) : 0;
        after[lv] = lv < nl ? (int64_t)(S.levels4[(size_t)lv].size() / 4) : 0;
    }
    if (!check_schedule(S, n, false, err) || !plan_memory(S, n, 1, false, err)) {
        set_err(err);
        return MDPS_EINVAL;
    }
    return nl;
}

// host-only check of the job schedule and its memory plan (no GPU needed):
// out[0] pool bytes without reuse, out[1] with the plan, out[2] chunks,
// out[3] launches per evaluation.  corrupt > 0 damages the plan first (1: a
// job writes a slot another job of its launch reads; 2: a job overwrites a
// slot that a later launch still reads; 3: an input slot out of range) —
// the check must then fail (its own test).
extern "C" int mdps_test_plan(const mdps_supports *sup, const int32_t *exponents, int32_t n, int32_t degree,
                              int32_t limbs, int32_t eft, int32_t batch, int32_t chunks, int32_t corrupt,
                              int64_t *out) {
    if (!sup || !out || n < 1 || degree < 0 || !valid_limbs(limbs) || batch < 1 || chunks < 1) {
        set_err("invalid argument");
        return MDPS_EINVAL;
    }
    Schedule S;
    std::string err;
    if (!build_schedule(sup->n_polys, sup->poly_ptr, sup->mono_ptr, sup->vars, exponents, n, S, err) ||
        (batch > 1 && !replicate_schedule(S, n, batch, err))) {
        set_err(err);
        return MDPS_EINVAL;
    }
    const int D = degree + 1, Sd = eft ? 0 : digits_for(limbs);
    out[0] = plan_bytes(S, Sd, limbs, D, eft != 0);
    if (!check_schedule(S, n, eft != 0, err) || !plan_memory(S, n, chunks, eft != 0, err)) {
        set_err(err);
        return MDPS_EINVAL;
    }
    out[1] = plan_bytes(S, Sd, limbs, D, eft != 0);
    out[2] = (int64_t)S.chunks.size();
    int64_t launches = 1;
    for (auto &ch : S.chunks) launches += (int64_t)ch.levels4.size() + (ch.ntask[0] > 0 || ch.ntask[1] > 0);
    out[3] = launches;
    if (corrupt > 0) {
        const int64_t nfix = (int64_t)S.batch * n + S.M;
        bool done = false;
        for (auto &ch : S.chunks) {
            for (size_t lv = 0; lv < ch.levels4.size() && !done; lv++) {
                auto &v = ch.levels4[lv];
                if (corrupt == 1) {  // the last job writes the first dynamic input read in this launch
                    for (size_t q = 0; q < v.size() && !done; q += 4)
                        for (int k = 0; k < 2 && !done; k++)
                            if (v[q + k] >= nfix && v.size() >= 8) {
                                v[v.size() - 4 + 2] = v[q + k];
                                v[v.size() - 4 + 3] |= 1;
                                done = true;
                            }
                } else if (corrupt == 2 && lv + 2 < ch.levels4.size()) {
                    // a job of launch lv+1 overwrites an input that launch lv+2 reads and lv+1 does not write
                    auto &w = ch.levels4[lv + 2];
                    for (size_t q = 0; q < w.size() && !done; q += 4)
                        if (w[q] >= nfix) {
                            auto &u = ch.levels4[lv + 1];
                            bool produced_here = false;
                            for (size_t r = 0; r < u.size(); r += 4) produced_here |= u[r + 2] == w[q];
                            if (produced_here) continue;
                            u[2] = w[q];
                            u[3] |= 1;
                            done = true;
                        }
                } else if (corrupt == 3) {
                    v[0] = (int32_t)(S.dig_slots + 5);
                    done = true;
                }
            }
        }
        if (!done) {
            set_err("nothing to corrupt");
            return MDPS_EINVAL;
        }
        if (!check_schedule(S, n, eft != 0, err)) {
            set_err(err);
            return MDPS_EINVAL;  // detected
        }
        set_err("corruption not detected");
        return 1;
    }
    return MDPS_OK;
}
