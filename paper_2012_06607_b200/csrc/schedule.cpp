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
    for (int i = 0; i < n_polys; i++) {
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
