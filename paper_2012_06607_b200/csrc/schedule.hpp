// schedule.hpp — host-side job DAG for mdps_eval_diff.
//
// Per monomial c * prod_l x_{v_l}^{a_l} (variables ascending)
// the product jobs of algorithmic differentiation (all n
// partials at ~3x the cost of one evaluation):
//   common factor  c' = c * prod_l x_{v_l}^{a_l - 1}     (only when some a_l >= 2;
//                  multiplied out as a tree, lowest levels first: depth
//                  ceil(log2(1 + sum(a_l - 1))), the same product count)
//   forward        f_1 = c' x_{v_1},  f_l = f_{l-1} x_{v_l};  value = f_m
//   backward       B_0 = x_{v_m} (alias),  B_k = B_{k-1} x_{v_{m-k}},  k = 1..m-2
//   cross          d_1 = c' B_{m-2},  d_l = f_{l-1} B_{m-l-1} (l = 2..m-1),  d_m = f_{m-1}
//   weights        J[i][v_l] += a_l * d_l                  (folded into the sums)
// 3(m-1) + sum_l (a_l - 1) products for m >= 2 (1 + sum for m = 1).  A job's
// level is 1 + the max level of its inputs (x and c are level 0); each level
// is one launch (the GPU analogue of the paper's stage synchronisation,
// PAPER.md:420-424).  The addition jobs are a CSR list per
// output series: N values then N*n Jacobian entries (row-major); N = n for a
// square system, any N >= 1 otherwise (a row subset, an over/under-determined
// system).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace mdps {

struct Schedule {
    int n = 0, N = 0, D = 0, L = 0, M = 0;  // n variables, N polynomials
    int64_t nslots = 0;                         // n + M + jobs
    std::vector<std::vector<int32_t>> levels;   // per level: (in1, in2, out) triples
    std::vector<int32_t> task_ptr;              // [N + N*n + 1]
    std::vector<int32_t> ent_slot, ent_w;       // addition terms
    int64_t products = 0;
    int32_t max_weight = 1;
    // form of each series: product inputs are read as digit planes, summed
    // series as limbs.  limb_slot[slot] = index in the limb pool or -1.
    std::vector<int32_t> limb_slot, ent_lslot;  // ent_lslot: ent_slot remapped to the limb pool
    int64_t nlimb = 0;
    // per level: (in1, in2, out, code) with code = lslot << 2 | 2 (write limbs)
    // | 1 (write digits: the output is a product input)
    std::vector<std::vector<int32_t>> levels4;
    // batch of B points (replicate_schedule): per-point limb slots of the
    // x and coefficient series and the per-point limb-pool size
    int batch = 1;
    std::vector<int32_t> limb_slot1;
    int64_t nlimb1 = 0;
    // row (polynomial) of every product job's output, slot - n - M (batch 1)
    std::vector<int32_t> job_row;
    // memory plan (plan_memory): chunks of rows run one after the other, each
    // its levels then its addition jobs; slots reused by liveness
    struct Chunk {
        std::vector<std::vector<int32_t>> levels4;  // non-empty levels, (in1, in2, out, code) per job
        std::vector<std::vector<int32_t>> orig3;    // the same jobs' unplanned (in1, in2, out) (checks)
        int32_t task0[2] = {0, 0}, ntask[2] = {0, 0};  // addition-job ranges (values, Jacobian rows)
    };
    std::vector<Chunk> chunks;
    bool planned = false;
    std::vector<std::pair<int32_t, int32_t>> fixed_limb;  // (slot < nx + M, limb slot) of summed inputs
    std::vector<int32_t> plan_ent;  // per addition entry: its planned slot (EFT pool) or limb slot (digits)
    int64_t dig_slots = 0;          // digit pool (or EFT pool) slots after planning
    int64_t plan_nlimb = 0;         // limb pool slots after planning (digits)
};

// Validates the inputs (libmdps.h) and builds the schedule.  Pool slots:
// [0, n) = x, [n, n+M) = coefficients, then one slot per product job.
bool build_schedule(int32_t n_polys, const int32_t *poly_ptr, const int32_t *mono_ptr,
                    const int32_t *vars, const int32_t *exps, int32_t n, Schedule &S,
                    std::string &err);

// Level balancing (leveled schedule): a product whose output is only summed by
// the addition jobs (never a product input) may run in any later level.  The
// levels of a system whose monomials differ in length shrink towards the end
// — the last ones cannot fill the GPU — so such jobs are moved, in order,
// from the earlier levels that hold more than min_jobs into every later
// level that holds fewer, until it holds min_jobs (one wave of the product
// kernel's resident blocks) or the donors run out.  Same jobs, same
// arithmetic: the outputs do not change.  Call before replicate_schedule /
// plan_memory.  Returns the number of jobs moved.
int64_t balance_levels(Schedule &S, int64_t min_jobs);

// The same system at B points in one schedule (mdps_options.batch): slots
// [0, B n) = the points' x, [B n, B n + M) = the shared coefficients, then B
// blocks of product slots; every level holds the B copies of its jobs, the
// addition jobs are the B N values then the B N n Jacobian entries, each
// point with its own limb-pool block.  The kernels are unchanged.
bool replicate_schedule(Schedule &S, int32_t n, int32_t B, std::string &err);

// Memory plan for the leveled launch order: the rows are split
// into `chunks` contiguous groups balanced by product count (batch 1 only),
// run one after the other (each: its levels, then its addition jobs), and
// every product output gets a pool slot only for its live range — from the
// launch that writes it to the last launch that reads it (a product input:
// digit slot; a summed series: limb slot, read by its chunk's addition jobs).
// A slot freed after launch t is reused from launch t + 1 on (launches are
// stream-ordered, so no two launches overlap).  eft: one pool of limb series
// for both roles.  Rewrites the job tuples and the addition entries.
bool plan_memory(Schedule &S, int32_t n, int32_t chunks, bool eft, std::string &err);

// Bytes of the plan's pools: digits (2 S D doubles + 2 D ints per slot) and
// limbs (2 L D doubles per slot), or one limb pool for eft.
int64_t plan_bytes(const Schedule &S, int S_digits, int L, int D, bool eft);

// Checks a schedule (planned or not): every slot index in range; every job
// output written exactly once per evaluation (unplanned) or, planned, no
// slot read after it was overwritten and no slot written while a launch
// still reads it; every input of a launch written by an EARLIER launch (or a
// fixed input); every summed series written before its addition jobs.  The
// race-freedom and bounds invariants of the kernels' reads and writes.
bool check_schedule(const Schedule &S, int32_t n, bool eft, std::string &err);

}  // namespace mdps
