// schedule.cpp — builds the leveled product DAG and the addition lists.
// See schedule.hpp for the scheme and its citations.
#include "schedule.hpp"

#include <algorithm>
#include <climits>
#include <utility>

namespace mdps {

namespace {

struct Builder {
    Schedule &S;
    std::vector<int32_t> level;  // per slot
    int32_t row = 0;             // the polynomial whose monomial is being built
    explicit Builder(Schedule &s) : S(s) {}

    int32_t job(int32_t a, int32_t b) {
        const int32_t out = (int32_t)level.size();
        const int32_t lev = 1 + std::max(level[a], level[b]);
        level.push_back(lev);
        if ((int)S.levels.size() < lev) S.levels.resize(lev);
        auto &v = S.levels[lev - 1];
        v.push_back(a);
        v.push_back(b);
        v.push_back(out);
        S.job_row.push_back(row);
        S.products++;
        return out;
    }
};

}  // namespace

bool build_schedule(int32_t n_polys, const int32_t *poly_ptr, const int32_t *mono_ptr,
                    const int32_t *vars, const int32_t *exps, int32_t n, Schedule &S,
                    std::string &err) {
    if (n < 1) { err = "n must be >= 1"; return false; }
    if (n_polys < 1) { err = "n_polys must be >= 1"; return false; }
    if (!poly_ptr || !mono_ptr) { err = "NULL poly_ptr or mono_ptr"; return false; }
    if (poly_ptr[0] != 0) { err = "poly_ptr[0] must be 0"; return false; }
    for (int i = 0; i < n_polys; i++)
        if (poly_ptr[i + 1] < poly_ptr[i]) { err = "poly_ptr is not non-decreasing"; return false; }
    const int32_t M = poly_ptr[n_polys];
    if (mono_ptr[0] != 0) { err = "mono_ptr[0] must be 0"; return false; }
    for (int r = 0; r < M; r++)
        if (mono_ptr[r + 1] < mono_ptr[r]) { err = "mono_ptr is not non-decreasing"; return false; }
    const int32_t nnz = mono_ptr[M];
    if (nnz > 0 && (!vars || !exps)) { err = "NULL vars or exponents"; return false; }
    if ((int64_t)n_polys + (int64_t)n_polys * n + 1 > INT32_MAX) { err = "n too large"; return false; }

    S.n = n;
    S.N = n_polys;
    S.M = M;
    S.levels.clear();
    S.products = 0;
    Builder B(S);
    B.level.assign((size_t)n + M, 0);
    const int64_t ntasks = (int64_t)n_polys + (int64_t)n_polys * n;
    std::vector<std::vector<std::pair<int32_t, int32_t>>> lists((size_t)ntasks);
    auto jac = [&](int i, int j) -> std::vector<std::pair<int32_t, int32_t>> & {
        return lists[(size_t)n_polys + (size_t)i * n + j];
    };

    std::vector<std::pair<int32_t, int32_t>> mono;
    std::vector<int32_t> f, Bk;
    S.job_row.clear();
    for (int i = 0; i < n_polys; i++) {
        B.row = i;
        for (int r = poly_ptr[i]; r < poly_ptr[i + 1]; r++) {
            mono.clear();
            for (int t = mono_ptr[r]; t < mono_ptr[r + 1]; t++) {
                if (vars[t] < 0 || vars[t] >= n) { err = "variable index out of range"; return false; }
                if (exps[t] < 1) { err = "exponent < 1"; return false; }
                if (exps[t] > (1 << 20)) { err = "exponent too large"; return false; }
                mono.emplace_back(vars[t], exps[t]);
            }
            std::sort(mono.begin(), mono.end());
            for (size_t t = 1; t < mono.size(); t++)
                if (mono[t].first == mono[t - 1].first) {
                    err = "variable repeated within a monomial";
                    return false;
                }
            const int m = (int)mono.size();
            const int32_t c = n + r;
            if (m == 0) {  // constant term
                lists[i].emplace_back(c, 1);
                continue;
            }
            // common factor c' = c * prod x^(a-1): the same sum(a-1) products as a
            // chain, multiplied out as a tree — always the two operands of lowest
            // level first (ties in creation order, deterministic) — so c' sits
            // at level ceil(log2(1 + sum(a-1))) instead of sum(a-1): the
            // forward chain and everything after it start earlier (qd's
            // exponent-2 monomials)
            int32_t cp = c;
            {
                std::vector<std::pair<int32_t, int32_t>> q;  // (level, slot), in creation order
                q.emplace_back(0, c);
                for (int l = 0; l < m; l++)
                    for (int a = 1; a < mono[l].second; a++) q.emplace_back(0, mono[l].first);
                while (q.size() > 1) {
                    // the two lowest levels (stable: earliest first)
                    size_t i0 = 0;
                    for (size_t t = 1; t < q.size(); t++)
                        if (q[t].first < q[i0].first) i0 = t;
                    const auto a0 = q[i0];
                    q.erase(q.begin() + (long)i0);
                    size_t i1 = 0;
                    for (size_t t = 1; t < q.size(); t++)
                        if (q[t].first < q[i1].first) i1 = t;
                    const auto a1 = q[i1];
                    q.erase(q.begin() + (long)i1);
                    const int32_t o = B.job(a0.second, a1.second);
                    q.emplace_back(B.level[(size_t)o], o);
                }
                cp = q[0].second;
            }
            for (int l = 0; l < m; l++) S.max_weight = std::max(S.max_weight, mono[l].second);
            if (m == 1) {
                lists[i].emplace_back(B.job(cp, mono[0].first), 1);
                jac(i, mono[0].first).emplace_back(cp, mono[0].second);
                continue;
            }
            f.assign(m + 1, -1);
            f[1] = B.job(cp, mono[0].first);
            for (int l = 2; l <= m; l++) f[l] = B.job(f[l - 1], mono[l - 1].first);
            lists[i].emplace_back(f[m], 1);
            Bk.assign(m - 1, -1);
            Bk[0] = mono[m - 1].first;  // B_0 = x_{v_m}
            for (int k = 1; k <= m - 2; k++) Bk[k] = B.job(Bk[k - 1], mono[m - 1 - k].first);
            // d_1 = c' * B_{m-2}
            jac(i, mono[0].first).emplace_back(B.job(cp, Bk[m - 2]), mono[0].second);
            for (int l = 2; l <= m - 1; l++)
                jac(i, mono[l - 1].first).emplace_back(B.job(f[l - 1], Bk[m - l - 1]), mono[l - 1].second);
            jac(i, mono[m - 1].first).emplace_back(f[m - 1], mono[m - 1].second);
        }
    }
    S.nslots = (int64_t)B.level.size();
    if (S.nslots > INT32_MAX / 4) { err = "too many series (slots overflow int32)"; return false; }
    S.task_ptr.assign((size_t)ntasks + 1, 0);
    S.ent_slot.clear();
    S.ent_w.clear();
    for (int64_t t = 0; t < ntasks; t++) {
        for (auto &e : lists[(size_t)t]) {
            S.ent_slot.push_back(e.first);
            S.ent_w.push_back(e.second);
        }
        if (S.ent_slot.size() > (size_t)INT32_MAX) { err = "too many addition terms"; return false; }
        S.task_ptr[(size_t)t + 1] = (int32_t)S.ent_slot.size();
    }
    // which series are product inputs (digit form) and which are summed by the
    // addition jobs (limb form); the limb pool holds only the latter
    std::vector<uint8_t> as_input((size_t)S.nslots, 0);
    for (auto &lv : S.levels)
        for (size_t q = 0; q < lv.size(); q += 3) {
            as_input[(size_t)lv[q]] = 1;
            as_input[(size_t)lv[q + 1]] = 1;
        }
    S.limb_slot.assign((size_t)S.nslots, -1);
    S.nlimb = 0;
    for (int32_t s : S.ent_slot)
        if (S.limb_slot[(size_t)s] < 0) S.limb_slot[(size_t)s] = (int32_t)S.nlimb++;
    S.ent_lslot.resize(S.ent_slot.size());
    for (size_t e = 0; e < S.ent_slot.size(); e++) S.ent_lslot[e] = S.limb_slot[(size_t)S.ent_slot[e]];
    S.levels4.clear();
    for (auto &lv : S.levels) {
        std::vector<int32_t> v;
        v.reserve(lv.size() / 3 * 4);
        for (size_t q = 0; q < lv.size(); q += 3) {
            const int32_t out = lv[q + 2];
            const int32_t ls = S.limb_slot[(size_t)out];
            const int32_t code = (ls >= 0 ? ((ls << 2) | 2) : 0) | (as_input[(size_t)out] ? 1 : 0);
            v.push_back(lv[q]);
            v.push_back(lv[q + 1]);
            v.push_back(out);
            v.push_back(code);
        }
        S.levels4.push_back(std::move(v));
    }
    return true;
}

int64_t balance_levels(Schedule &S, int64_t min_jobs) {
    const int nl = (int)S.levels4.size();
    if (nl < 2 || min_jobs <= 0 || S.levels.size() != S.levels4.size()) return 0;
    int64_t moved = 0;
    for (int t = nl - 1; t >= 1; t--) {
        int64_t need = min_jobs - (int64_t)(S.levels4[(size_t)t].size() / 4);
        for (int s = 0; s < t && need > 0; s++) {
            auto &src4 = S.levels4[(size_t)s];
            auto &src3 = S.levels[(size_t)s];
            const int64_t have = (int64_t)(src4.size() / 4);
            int64_t give = std::min(need, have - min_jobs);
            if (give <= 0) continue;
            // the level's last `give` summed-only jobs (code bit 0 clear), order kept
            std::vector<int32_t> keep4, keep3, mv4, mv3;
            keep4.reserve(src4.size());
            keep3.reserve(src3.size());
            for (int64_t q = have - 1; q >= 0; q--) {
                const bool leaf = (src4[(size_t)(4 * q + 3)] & 1) == 0;
                auto &d4 = (leaf && give > 0) ? mv4 : keep4;
                auto &d3 = (leaf && give > 0) ? mv3 : keep3;
                if (leaf && give > 0) give--;
                for (int c = 3; c >= 0; c--) d4.push_back(src4[(size_t)(4 * q + c)]);
                for (int c = 2; c >= 0; c--) d3.push_back(src3[(size_t)(3 * q + c)]);
            }
            std::reverse(keep4.begin(), keep4.end());
            std::reverse(keep3.begin(), keep3.end());
            std::reverse(mv4.begin(), mv4.end());
            std::reverse(mv3.begin(), mv3.end());
            const int64_t got = (int64_t)(mv4.size() / 4);
            if (got == 0) continue;
            src4 = std::move(keep4);
            src3 = std::move(keep3);
            auto &dst4 = S.levels4[(size_t)t];
            auto &dst3 = S.levels[(size_t)t];
            dst4.insert(dst4.end(), mv4.begin(), mv4.end());
            dst3.insert(dst3.end(), mv3.begin(), mv3.end());
            need -= got;
            moved += got;
        }
    }
    return moved;
}

bool replicate_schedule(Schedule &S, int32_t n, int32_t B, std::string &err) {
    const int64_t M = S.M, J = S.nslots - n - M, nl = S.nlimb;
    const int64_t total = (int64_t)B * n + M + (int64_t)B * J;
    if (total > INT32_MAX / 4) { err = "batch too large (slots overflow int32)"; return false; }
    if ((int64_t)B * nl >= (1LL << 29)) { err = "batch too large (limb slots overflow the job code)"; return false; }
    const int64_t ntasks0 = (int64_t)S.N + (int64_t)S.N * n;
    if ((int64_t)B * ntasks0 + 1 > INT32_MAX || (int64_t)B * (int64_t)S.ent_slot.size() > INT32_MAX) {
        err = "batch too large (addition jobs overflow int32)";
        return false;
    }
    auto map = [&](int32_t slot, int32_t b) -> int32_t {
        if (slot < n) return (int32_t)((int64_t)b * n + slot);
        if (slot < n + M) return (int32_t)((int64_t)B * n + (slot - n));
        return (int32_t)((int64_t)B * n + M + (int64_t)b * J + (slot - n - M));
    };
    std::vector<std::vector<int32_t>> lv4;
    for (auto &lv : S.levels4) {
        std::vector<int32_t> v;
        v.reserve(lv.size() * (size_t)B);
        for (int32_t b = 0; b < B; b++)
            for (size_t q = 0; q < lv.size(); q += 4) {
                v.push_back(map(lv[q], b));
                v.push_back(map(lv[q + 1], b));
                v.push_back(map(lv[q + 2], b));
                int32_t code = lv[q + 3];
                if (code & 2) code = (int32_t)((((int64_t)(code >> 2) + (int64_t)b * nl) << 2) | (code & 3));
                v.push_back(code);
            }
        lv4.push_back(std::move(v));
    }
    std::vector<int32_t> tp{0}, es, ew, el;
    auto copy_task = [&](int64_t t, int32_t b) {
        for (int32_t e = S.task_ptr[(size_t)t]; e < S.task_ptr[(size_t)t + 1]; e++) {
            es.push_back(map(S.ent_slot[(size_t)e], b));
            ew.push_back(S.ent_w[(size_t)e]);
            el.push_back(S.ent_lslot.empty() ? -1 : (int32_t)(S.ent_lslot[(size_t)e] + (int64_t)b * nl));
        }
        tp.push_back((int32_t)es.size());
    };
    for (int32_t b = 0; b < B; b++)
        for (int64_t t = 0; t < S.N; t++) copy_task(t, b);
    for (int32_t b = 0; b < B; b++)
        for (int64_t t = S.N; t < ntasks0; t++) copy_task(t, b);
    S.limb_slot1.assign(S.limb_slot.begin(), S.limb_slot.begin() + (size_t)(n + M));
    S.nlimb1 = nl;
    S.levels4 = std::move(lv4);
    S.task_ptr = std::move(tp);
    S.ent_slot = std::move(es);
    S.ent_w = std::move(ew);
    S.ent_lslot = std::move(el);
    S.nslots = total;
    S.nlimb = (int64_t)B * nl;
    S.products *= B;
    S.batch = B;
    return true;
}

}  // namespace mdps

namespace mdps {

namespace {

// slots by liveness: acquire() the lowest-numbered free slot... a LIFO free
// list keeps recently used (L2-warm) slots in use
struct SlotPool {
    int64_t base, next;
    std::vector<int32_t> free_;
    explicit SlotPool(int64_t b) : base(b), next(b) {}
    int32_t acquire() {
        if (!free_.empty()) {
            const int32_t s = free_.back();
            free_.pop_back();
            return s;
        }
        return (int32_t)next++;
    }
    void release(int32_t s) { free_.push_back(s); }
};

}  // namespace

bool plan_memory(Schedule &S, int32_t n, int32_t chunks, bool eft, std::string &err) {
    const int64_t B = S.batch, nx = B * n, nfix = nx + S.M;
    const int64_t ndyn = S.nslots - nfix;
    if (chunks < 1) chunks = 1;
    if (B > 1) chunks = 1;  // rows of a batch are per point: one chunk
    if (chunks > S.N) chunks = S.N;
    // ---- rows -> chunks, contiguous, balanced by product count
    std::vector<int32_t> chunk_of_row((size_t)S.N, 0);
    std::vector<int32_t> row_lo((size_t)chunks + 1, S.N);
    row_lo[0] = 0;
    if (chunks > 1) {
        if ((int64_t)S.job_row.size() != ndyn) { err = "plan_memory: no row map"; return false; }
        std::vector<int64_t> cost((size_t)S.N, 0);
        for (int32_t r : S.job_row) cost[(size_t)r]++;
        int64_t total = 0;
        for (int64_t c : cost) total += c;
        int64_t acc = 0;
        int c = 0;
        for (int32_t r = 0; r < S.N; r++) {
            // start chunk c+1 once this chunk holds its share
            if (c + 1 < chunks && acc >= total * (c + 1) / chunks && r > row_lo[(size_t)c]) row_lo[(size_t)++c] = r;
            chunk_of_row[(size_t)r] = c;
            acc += cost[(size_t)r];
        }
        chunks = c + 1;
        row_lo.resize((size_t)chunks + 1);
        row_lo[(size_t)chunks] = S.N;
    }
    // ---- launch order: chunk-major, level-minor (empty levels skipped), then
    // the chunk's addition jobs
    S.chunks.assign((size_t)chunks, Schedule::Chunk());
    const int nlev = (int)S.levels4.size();
    std::vector<std::vector<std::vector<int32_t>>> cl((size_t)chunks, std::vector<std::vector<int32_t>>((size_t)nlev));
    for (int lv = 0; lv < nlev; lv++) {
        const auto &v = S.levels4[(size_t)lv];
        for (size_t q = 0; q < v.size(); q += 4) {
            const int32_t out = v[q + 2];
            const int c = chunks > 1 ? chunk_of_row[(size_t)S.job_row[(size_t)(out - nfix)]] : 0;
            auto &d = cl[(size_t)c][(size_t)lv];
            d.insert(d.end(), v.begin() + (long)q, v.begin() + (long)q + 4);
        }
    }
    // launch index of every dynamic slot's producer, last product read, and
    // the chunk's addition launch (summed series)
    std::vector<int64_t> t_prod((size_t)ndyn, -1), t_read((size_t)ndyn, -1), t_sum((size_t)ndyn, -1);
    std::vector<int64_t> t_accum((size_t)chunks, 0);
    int64_t t = 0;
    for (int c = 0; c < chunks; c++) {
        for (int lv = 0; lv < nlev; lv++) {
            const auto &v = cl[(size_t)c][(size_t)lv];
            if (v.empty()) continue;
            for (size_t q = 0; q < v.size(); q += 4) {
                for (int k = 0; k < 2; k++)
                    if (v[q + k] >= nfix) t_read[(size_t)(v[q + k] - nfix)] = t;
                t_prod[(size_t)(v[q + 2] - nfix)] = t;
            }
            t++;
        }
        t_accum[(size_t)c] = t++;
    }
    const int64_t nlaunch = t;
    // summed series: read by the addition launch of the chunk of their row
    // (entries of task i, N + i n + j belong to row i)
    const int64_t N = S.N;
    auto task_row = [&](int64_t task) -> int64_t {
        const int64_t per = N + N * n;  // tasks per point
        const int64_t tt = task % per;
        return tt < N ? tt : (tt - N) / n;
    };
    for (int64_t task = 0; task + 1 < (int64_t)S.task_ptr.size(); task++) {
        const int c = chunks > 1 ? chunk_of_row[(size_t)task_row(task)] : 0;
        for (int32_t e = S.task_ptr[(size_t)task]; e < S.task_ptr[(size_t)task + 1]; e++) {
            const int32_t sl = S.ent_slot[(size_t)e];
            if (sl >= nfix) t_sum[(size_t)(sl - nfix)] = t_accum[(size_t)c];
        }
    }
    // ---- slot assignment in launch order; a slot whose last use is launch t
    // is released before launch t + 1
    std::vector<std::vector<int32_t>> rel_d((size_t)nlaunch + 1), rel_l((size_t)nlaunch + 1);
    std::vector<int32_t> dslot((size_t)ndyn, -1), lslot((size_t)ndyn, -1);
    // fixed limb slots: summed x / coefficient series, first
    S.fixed_limb.clear();
    int64_t nfixed_l = 0;
    if (!eft) {
        std::vector<int32_t> fl((size_t)nfix, -1);
        for (int32_t sl : S.ent_slot)
            if (sl < nfix && fl[(size_t)sl] < 0) fl[(size_t)sl] = 0;
        for (int64_t sl = 0; sl < nfix; sl++)
            if (fl[(size_t)sl] == 0) S.fixed_limb.emplace_back((int32_t)sl, (int32_t)nfixed_l++);
    }
    SlotPool pd(nfix), pl(nfixed_l);
    t = 0;
    for (int c = 0; c < chunks; c++) {
        for (int lv = 0; lv < nlev; lv++) {
            auto &v = cl[(size_t)c][(size_t)lv];
            if (v.empty()) continue;
            for (int32_t r : rel_d[(size_t)t]) pd.release(r);
            for (int32_t r : rel_l[(size_t)t]) pl.release(r);
            for (size_t q = 0; q < v.size(); q += 4) {
                const int64_t o = v[q + 2] - nfix;
                const bool input = t_read[(size_t)o] >= 0, summed = t_sum[(size_t)o] >= 0;
                if (eft) {
                    const int64_t last = std::max(t_read[(size_t)o], t_sum[(size_t)o]);
                    if (last < 0) { err = "plan_memory: a product nobody reads"; return false; }
                    dslot[(size_t)o] = pd.acquire();
                    rel_d[(size_t)last + 1].push_back(dslot[(size_t)o]);
                } else {
                    if (input) {
                        dslot[(size_t)o] = pd.acquire();
                        rel_d[(size_t)t_read[(size_t)o] + 1].push_back(dslot[(size_t)o]);
                    }
                    if (summed) {
                        lslot[(size_t)o] = pl.acquire();
                        rel_l[(size_t)t_sum[(size_t)o] + 1].push_back(lslot[(size_t)o]);
                    }
                    if (!input && !summed) { err = "plan_memory: a product nobody reads"; return false; }
                }
            }
            t++;
        }
        for (int32_t r : rel_d[(size_t)t]) pd.release(r);
        for (int32_t r : rel_l[(size_t)t]) pl.release(r);
        t++;
    }
    if (pd.next > INT32_MAX / 4 || (pl.next << 2) > INT32_MAX) { err = "plan_memory: slots overflow int32"; return false; }
    S.dig_slots = pd.next;
    S.plan_nlimb = pl.next;
    // ---- rewrite the jobs and the addition entries
    auto map_in = [&](int32_t s) -> int32_t { return s < nfix ? s : dslot[(size_t)(s - nfix)]; };
    for (int c = 0; c < chunks; c++) {
        auto &ch = S.chunks[(size_t)c];
        for (int lv = 0; lv < nlev; lv++) {
            auto &v = cl[(size_t)c][(size_t)lv];
            if (v.empty()) continue;
            std::vector<int32_t> w, o3;
            w.reserve(v.size());
            o3.reserve(v.size() / 4 * 3);
            for (size_t q = 0; q < v.size(); q += 4) {
                const int64_t o = v[q + 2] - nfix;
                o3.push_back(v[q]);
                o3.push_back(v[q + 1]);
                o3.push_back(v[q + 2]);
                w.push_back(map_in(v[q]));
                w.push_back(map_in(v[q + 1]));
                if (eft) {
                    w.push_back(dslot[(size_t)o]);
                    w.push_back(0);
                } else {
                    w.push_back(dslot[(size_t)o] >= 0 ? dslot[(size_t)o] : 0);
                    w.push_back((lslot[(size_t)o] >= 0 ? ((lslot[(size_t)o] << 2) | 2) : 0) | (dslot[(size_t)o] >= 0 ? 1 : 0));
                }
            }
            ch.levels4.push_back(std::move(w));
            ch.orig3.push_back(std::move(o3));
        }
        if (chunks > 1) {
            const int32_t r0 = row_lo[(size_t)c], r1 = row_lo[(size_t)c + 1];
            ch.task0[0] = r0;
            ch.ntask[0] = r1 - r0;
            ch.task0[1] = (int32_t)(N + (int64_t)r0 * n);
            ch.ntask[1] = (int32_t)((int64_t)(r1 - r0) * n);
        } else {
            ch.task0[0] = 0;
            ch.ntask[0] = (int32_t)(S.task_ptr.size() - 1);
        }
    }
    std::vector<int32_t> fixl((size_t)nfix, -1);
    for (auto &fl : S.fixed_limb) fixl[(size_t)fl.first] = fl.second;
    S.plan_ent.resize(S.ent_slot.size());
    for (size_t e = 0; e < S.ent_slot.size(); e++) {
        const int32_t sl = S.ent_slot[e];
        if (eft) S.plan_ent[e] = map_in(sl);
        else S.plan_ent[e] = sl < nfix ? fixl[(size_t)sl] : lslot[(size_t)(sl - nfix)];
    }
    S.planned = true;
    return check_schedule(S, n, eft, err);
}

int64_t plan_bytes(const Schedule &S, int S_digits, int L, int D, bool eft) {
    const int64_t limb = (int64_t)2 * L * D * 8;
    if (eft) return (S.planned ? S.dig_slots : S.nslots) * limb;
    const int64_t dig = (int64_t)2 * S_digits * D * 8 + (int64_t)D * 4;  // digits [S][D][2], exponents [D]
    return (S.planned ? S.dig_slots : S.nslots) * dig + (S.planned ? S.plan_nlimb : S.nlimb) * limb;
}

bool check_schedule(const Schedule &S, int32_t n, bool eft, std::string &err) {
    const int64_t nfix = (int64_t)S.batch * n + S.M;
    auto fail = [&](const std::string &m) {
        err = "schedule check: " + m;
        return false;
    };
    if (!S.planned) {
        // every dynamic slot written exactly once, at a level above its inputs'
        std::vector<int32_t> lev((size_t)S.nslots, -1);
        for (int64_t s = 0; s < nfix; s++) lev[(size_t)s] = 0;
        for (size_t lv = 0; lv < S.levels4.size(); lv++) {
            const auto &v = S.levels4[lv];
            for (size_t q = 0; q < v.size(); q += 4) {
                for (int k = 0; k < 3; k++)
                    if (v[q + k] < 0 || v[q + k] >= S.nslots) return fail("slot out of range");
                if (lev[(size_t)v[q + 2]] >= 0) return fail("a slot written twice");
                for (int k = 0; k < 2; k++)
                    if (lev[(size_t)v[q + k]] < 0 || lev[(size_t)v[q + k]] > (int)lv)
                        return fail("an input not written by an earlier level");
            }
            for (size_t q = 0; q < v.size(); q += 4) lev[(size_t)v[q + 2]] = (int32_t)lv + 1;
        }
        for (int32_t sl : S.ent_slot)
            if (sl < 0 || sl >= S.nslots || lev[(size_t)sl] < 0) return fail("a summed series never written");
        return true;
    }
    // planned: replay the launches; per pool slot the original series it holds
    const int64_t npool = S.dig_slots;
    std::vector<int32_t> holds((size_t)npool, -1), holds_l((size_t)S.plan_nlimb, -1);
    std::vector<int64_t> wrote_at((size_t)npool, -1), wrote_at_l((size_t)S.plan_nlimb, -1);
    for (int64_t s = 0; s < nfix && s < npool; s++) holds[(size_t)s] = (int32_t)s;
    for (auto &fl : S.fixed_limb) {
        if (fl.second < 0 || fl.second >= S.plan_nlimb) return fail("fixed limb slot out of range");
        holds_l[(size_t)fl.second] = fl.first;
    }
    int64_t t = 0;
    for (const auto &ch : S.chunks) {
        for (size_t lv = 0; lv < ch.levels4.size(); lv++) {
            const auto &v = ch.levels4[lv];
            const auto &o = ch.orig3[lv];
            if (o.size() / 3 != v.size() / 4) return fail("planned/original job count");
            for (size_t j = 0; j < v.size() / 4; j++)  // reads: the intended series, written by an earlier launch
                for (int k = 0; k < 2; k++) {
                    const int32_t p = v[4 * j + k];
                    if (p < 0 || p >= npool) return fail("input slot out of range");
                    if (holds[(size_t)p] != o[3 * j + k]) return fail("an input overwritten or never written");
                }
            for (size_t j = 0; j < v.size() / 4; j++) {  // writes: no slot twice per launch, none read in it
                const int32_t p = v[4 * j + 2], code = v[4 * j + 3];
                const bool wd = eft || (code & 1), wl = !eft && (code & 2);
                if (wd) {
                    if (p < nfix || p >= npool) return fail("output slot out of range");
                    if (wrote_at[(size_t)p] == t) return fail("a slot written twice in one launch");
                    holds[(size_t)p] = o[3 * j + 2];
                    wrote_at[(size_t)p] = t;
                }
                if (wl) {
                    const int32_t ls = code >> 2;
                    if (ls < 0 || ls >= S.plan_nlimb) return fail("limb slot out of range");
                    if (wrote_at_l[(size_t)ls] == t) return fail("a limb slot written twice in one launch");
                    holds_l[(size_t)ls] = o[3 * j + 2];
                    wrote_at_l[(size_t)ls] = t;
                }
            }
            for (size_t j = 0; j < v.size() / 4; j++)  // no input slot of this launch also written in it
                for (int k = 0; k < 2; k++)
                    if (wrote_at[(size_t)v[4 * j + k]] == t) return fail("a slot read and overwritten in one launch");
            t++;
        }
        // the chunk's addition jobs read the series they sum
        for (int r = 0; r < 2; r++)
            for (int32_t task = ch.task0[r]; task < ch.task0[r] + ch.ntask[r]; task++)
                for (int32_t e = S.task_ptr[(size_t)task]; e < S.task_ptr[(size_t)task + 1]; e++) {
                    const int32_t p = S.plan_ent[(size_t)e];
                    if (eft) {
                        if (p < 0 || p >= npool || holds[(size_t)p] != S.ent_slot[(size_t)e])
                            return fail("a summed series overwritten or never written");
                    } else if (p < 0 || p >= S.plan_nlimb || holds_l[(size_t)p] != S.ent_slot[(size_t)e]) {
                        return fail("a summed series overwritten or never written");
                    }
                }
        t++;
    }
    // every addition job covered by exactly one chunk range
    std::vector<uint8_t> cov(S.task_ptr.size() - 1, 0);
    for (const auto &ch : S.chunks)
        for (int r = 0; r < 2; r++)
            for (int32_t task = ch.task0[r]; task < ch.task0[r] + ch.ntask[r]; task++) {
                if (task < 0 || task >= (int32_t)cov.size() || cov[(size_t)task]) return fail("addition ranges");
                cov[(size_t)task] = 1;
            }
    for (uint8_t c : cov)
        if (!c) return fail("an addition job in no chunk");
    return true;
}

}  // namespace mdps
