// a0: workload-aware drafting-strategy selection (§5), host C++.
//   dl(u) = prod_{v in Path(root,u)} o(v)                       (reading Z9: includes u)
//   w(u)  = F(dl(u)), F monotone piecewise linear, clamped [0,1]
//   al(n) = sum_{u in S(n)} w(u) over all samples of the batch     (Z20 shared n)
//   t_sd(n) = regression on N_seq, N_draft behind a bucket cache    (Z12)
//   layer-level search with a max priority queue, S(n) = S(n-1) U {u_max}
//   objective al/t_sd (Eq. 2), early stop after `patience` consecutive decreases (Eq. 3)
// and rs_cost_model_fit: least squares of the regression coefficients to measured times.
#include <algorithm>
#include <cmath>
#include <queue>
#include <unordered_map>
#include <vector>

#include "common.cuh"

struct rs_selector {
    rs_cost_model cost;
    std::vector<double> kx, ky;
    std::unordered_map<unsigned long long, double> cache;   // (seq bucket, draft bucket) -> t_sd
};

namespace {

double acceptance_fit(const rs_selector* s, double x) {
    const auto& kx = s->kx;
    const auto& ky = s->ky;
    double y;
    if (x <= kx.front()) {
        y = ky.front();
    } else if (x >= kx.back()) {
        y = ky.back();
    } else {
        size_t j = 0;                       // largest j with kx[j] <= x (same formula as np.interp)
        while (j + 1 < kx.size() && kx[j + 1] <= x) ++j;
        const double slope = (ky[j + 1] - ky[j]) / (kx[j + 1] - kx[j]);
        y = slope * (x - kx[j]) + ky[j];
    }
    return y < 0.0 ? 0.0 : (y > 1.0 ? 1.0 : y);
}

double regression(const rs_cost_model& c, double n_seq, double n_draft) {
    const double relu = n_draft - c.k_sat > 0.0 ? n_draft - c.k_sat : 0.0;
    return c.c_draft + c.b0 + c.b1 * n_seq + c.b2 * n_draft + c.b3 * relu * n_draft;
}

// t_sd at the lower corner of the (N_seq, N_draft) bucket; cached.
double t_sd(rs_selector* s, long long n_seq, long long n_draft, bool* hit) {
    const long long bs = n_seq / s->cost.seq_bucket, bd = n_draft / s->cost.draft_bucket;
    const unsigned long long key = ((unsigned long long)bs << 24) ^ (unsigned long long)bd;
    auto it = s->cache.find(key);
    if (it != s->cache.end()) {
        *hit = true;
        return it->second;
    }
    *hit = false;
    const double v = regression(s->cost, (double)(bs * s->cost.seq_bucket), (double)(bd * s->cost.draft_bucket));
    s->cache.emplace(key, v);
    return v;
}

struct PQItem {
    double w;
    int depth, id;
    bool operator<(const PQItem& o) const {   // max-heap on w; ties: lower depth, then lower id first
        if (w != o.w) return w < o.w;
        if (depth != o.depth) return depth > o.depth;
        return id > o.id;
    }
};

}  // namespace

extern "C" rs_status rs_selector_create(const rs_cost_model* cost, const double* knots_x, const double* knots_y,
                                        int32_t n_knots, rs_selector** out) {
    RS_REQUIRE(cost && knots_x && knots_y && out && n_knots >= 1, RS_ERR_INVALID_ARG, "rs_selector_create: bad args");
    RS_REQUIRE(cost->seq_bucket >= 1 && cost->draft_bucket >= 1, RS_ERR_INVALID_ARG,
               "rs_selector_create: bucket widths must be >= 1");
    for (int i = 1; i < n_knots; ++i)
        RS_REQUIRE(knots_x[i] > knots_x[i - 1] && knots_y[i] >= knots_y[i - 1], RS_ERR_INVALID_ARG,
                   "rs_selector_create: knots must be increasing in x and non-decreasing in y (monotone F)");
    auto* s = new rs_selector();
    s->cost = *cost;
    s->kx.assign(knots_x, knots_x + n_knots);
    s->ky.assign(knots_y, knots_y + n_knots);
    *out = s;
    return RS_OK;
}

extern "C" void rs_selector_destroy(rs_selector* sel) { delete sel; }

namespace {
// Reused per-thread buffers of the selector (no allocation per call once warm).
struct SelScratch {
    std::vector<double> w, ow;            // per candidate (flat over the batch): w; per (sample, step): popped w
    std::vector<int> dep, byd, cnt, cnt_off, ord, odep, lo, maxd, hsz;
    std::vector<PQItem> heap;             // per sample a heap slice of its candidate count
};
thread_local SelScratch tls;
}  // namespace

extern "C" rs_status rs_select_strategy(rs_selector* sel, const int32_t* cand_parent, const double* cand_o,
                                        const int32_t* cand_off, const int32_t* prefix_len, int32_t B, int32_t n_min,
                                        int32_t n_max, int32_t patience, rs_strategy* out, int32_t* selected) {
    RS_REQUIRE(sel && out && cand_off && prefix_len, RS_ERR_INVALID_ARG, "rs_select_strategy: null pointer");
    RS_REQUIRE(n_min >= 1 && n_max >= n_min && patience >= 1, RS_ERR_INVALID_ARG,
               "rs_select_strategy: need 1 <= n_min <= n_max, patience >= 1");
    RS_REQUIRE(B >= 1, RS_ERR_EMPTY_TREE, "rs_select_strategy: empty batch");
    SelScratch& S = tls;
    const int NT = cand_off[B] - cand_off[0];
    S.ord.assign((size_t)B * n_max, -1);   // per sample: the popped candidates in order (S(n) = first n)
    S.ow.resize((size_t)B * n_max);
    S.odep.resize((size_t)B * n_max);
    S.w.resize(NT > 0 ? NT : 1);
    S.dep.resize(NT > 0 ? NT : 1);
    S.byd.resize(NT > 0 ? NT : 1);
    S.heap.resize(NT > 0 ? NT : 1);
    S.cnt_off.assign(B + 1, 0);
    S.lo.assign(B, 0);
    S.maxd.assign(B, 0);
    S.hsz.assign(B, 0);
    S.cnt.clear();
    // per sample: dl, depth, w = F(dl), nodes grouped by depth (layer m is one contiguous range)
    for (int b = 0; b < B; ++b) {
        const int o0 = cand_off[b], N = cand_off[b + 1] - cand_off[b];
        RS_REQUIRE(N >= 0, RS_ERR_INVALID_ARG, "rs_select_strategy: cand_off not non-decreasing at %d", b);
        const int base = o0 - cand_off[0];
        double* dl = S.w.data() + base;   // dl first, then replaced by w in place
        int* dep = S.dep.data() + base;
        bool has_root_child = false;
        int max_dep = 0;
        for (int i = 0; i < N; ++i) {
            const int pa = cand_parent[o0 + i];
            RS_REQUIRE(pa < i, RS_ERR_MALFORMED_TREE, "rs_select_strategy: sample %d node %d parent %d", b, i, pa);
            dl[i] = cand_o[o0 + i] * (pa < 0 ? 1.0 : dl[pa]);
            dep[i] = pa < 0 ? 0 : dep[pa] + 1;
            max_dep = std::max(max_dep, dep[i]);
            has_root_child |= pa < 0;
        }
        RS_REQUIRE(N > 0 && has_root_child, RS_ERR_EMPTY_TREE, "rs_select_strategy: sample %d has no candidates", b);
        for (int i = 0; i < N; ++i) dl[i] = acceptance_fit(sel, dl[i]);
        S.maxd[b] = max_dep;
        S.cnt_off[b] = (int)S.cnt.size();
        S.cnt.resize(S.cnt.size() + max_dep + 2, 0);
        int* cnt = S.cnt.data() + S.cnt_off[b];
        for (int i = 0; i < N; ++i) ++cnt[dep[i] + 1];
        for (int d = 0; d <= max_dep; ++d) cnt[d + 1] += cnt[d];
        int* byd = S.byd.data() + base;
        for (int i = 0; i < N; ++i) byd[cnt[dep[i]]++] = i;   // cnt[d] ends at the start of d + 1
    }
    // layer-level search, step-major over the batch so the early stop of Eq. 3 also
    // stops the search: at step m every sample pushes its layer m (depth m-1) and pops its u_max;
    // al(m) adds the popped weights (Z20: one n for the batch). A sample whose heap runs dry ends
    // the feasible range (S(n) must exist for every sample).
    long long n_seq = 0;
    for (int b = 0; b < B; ++b) n_seq += prefix_len[b];
    double al = 0.0, best_obj = -INFINITY, prev = 0.0;
    int best_n = -1, dec = 0, n_stop = 0, best_hit = 0, feasible = n_max;
    double best_al = 0.0, best_t = 0.0;
    bool have_prev = false;
    for (int m = 1; m <= n_max; ++m) {
        double add = 0.0;
        bool dry = false;
        for (int b = 0; b < B && !dry; ++b) {
            const int base = cand_off[b] - cand_off[0];
            PQItem* hp = S.heap.data() + base;
            int& hs = S.hsz[b];
            if (m - 1 <= S.maxd[b]) {
                const int* cnt = S.cnt.data() + S.cnt_off[b];
                const int* byd = S.byd.data() + base;
                const int hi = cnt[m - 1];
                for (int k = S.lo[b]; k < hi; ++k) {
                    const int i = byd[k];
                    hp[hs++] = {S.w[base + i], S.dep[base + i], i};
                    std::push_heap(hp, hp + hs);
                }
                S.lo[b] = hi;
            }
            if (hs == 0) { dry = true; break; }
            std::pop_heap(hp, hp + hs);
            const PQItem top = hp[--hs];
            S.ord[(size_t)b * n_max + m - 1] = top.id;
            S.ow[(size_t)b * n_max + m - 1] = top.w;
            S.odep[(size_t)b * n_max + m - 1] = top.depth;
        }
        if (dry) { feasible = m - 1; break; }
        for (int b = 0; b < B; ++b) add += S.ow[(size_t)b * n_max + m - 1];   // (the reference's summation order)
        al += add;
        bool hit = false;
        const double t = t_sd(sel, n_seq, (long long)B * (m + 1), &hit);
        n_stop = m;
        if (m < n_min) continue;
        const double obj = al / t;
        if (obj > best_obj) {
            best_obj = obj;
            best_n = m;
            best_al = al;
            best_t = t;
            best_hit = hit ? 1 : 0;
        }
        if (have_prev && obj < prev) ++dec;
        else dec = 0;
        prev = obj;
        have_prev = true;
        if (dec >= patience) break;
    }
    RS_REQUIRE(feasible >= n_min && best_n >= 1, RS_ERR_INSUFFICIENT_NODES,
               "rs_select_strategy: only %d candidate steps (n_min %d)", feasible, n_min);
    // selection rows are defined up to n_stop (the search stopped there); -1 after
    for (int b = 0; b < B; ++b)
        for (int k = n_stop; k < n_max; ++k) S.ord[(size_t)b * n_max + k] = -1;
    int depth = 0, width = 0;
    int per_layer[RS_MAX_TREE + 2];
    for (int b = 0; b < B; ++b) {
        std::fill(per_layer, per_layer + RS_MAX_TREE + 2, 0);
        for (int k = 0; k < best_n; ++k) {
            const int d = S.odep[(size_t)b * n_max + k] + 1;   // verification-tree depth (root = 0)
            depth = std::max(depth, d);
            if (d <= RS_MAX_TREE) width = std::max(width, ++per_layer[d]);
        }
    }
    if (selected) std::copy(S.ord.begin(), S.ord.end(), selected);
    out->n = best_n;
    out->depth = depth;
    out->width = width;
    out->n_stop = n_stop;
    out->cache_hit = best_hit;
    out->cache_entries = (int32_t)sel->cache.size();
    out->al = best_al;
    out->t_sd = best_t;
    out->objective = best_obj;
    return RS_OK;
}

// dl(u) = o(u) * dl(parent(u)) (reading Z9: the product includes u), per candidate.
extern "C" rs_status rs_draft_logits(const int32_t* cand_parent, const double* cand_o, const int32_t* cand_off,
                                     int32_t B, double* dl_out) {
    RS_REQUIRE(cand_parent && cand_o && cand_off && dl_out && B >= 0, RS_ERR_INVALID_ARG, "rs_draft_logits: bad args");
    for (int b = 0; b < B; ++b) {
        const int o0 = cand_off[b], N = cand_off[b + 1] - o0;
        for (int i = 0; i < N; ++i) {
            const int pa = cand_parent[o0 + i];
            RS_REQUIRE(pa < i, RS_ERR_MALFORMED_TREE, "rs_draft_logits: sample %d node %d parent %d", b, i, pa);
            dl_out[o0 + i] = cand_o[o0 + i] * (pa < 0 ? 1.0 : dl_out[o0 + pa]);
        }
    }
    return RS_OK;
}

// F from (dl, accepted) observations (reading Z24): K equal-width
// buckets of dl over [0, 1] -> per non-empty bucket the mean dl and the mean acceptance (weight =
// count) -> weighted pool-adjacent-violators (non-decreasing least squares) -> knots.
extern "C" rs_status rs_acceptance_fit(const double* dl, const double* accepted, int64_t n, int32_t n_buckets,
                                       double* knots_x, double* knots_y, int32_t* n_knots) {
    RS_REQUIRE(dl && accepted && knots_x && knots_y && n_knots && n >= 0 && n_buckets >= 1, RS_ERR_INVALID_ARG,
               "rs_acceptance_fit: bad args");
    bool two = false;
    for (int64_t i = 1; i < n && !two; ++i) two = dl[i] != dl[0];
    RS_REQUIRE(two, RS_ERR_INVALID_ARG, "rs_acceptance_fit: InsufficientData (< 2 distinct draft logits)");
    const int K = n_buckets;
    std::vector<double> sx(K, 0.0), sy(K, 0.0);
    std::vector<long long> cnt(K, 0);
    for (int64_t i = 0; i < n; ++i) {
        const double x = dl[i] < 0.0 ? 0.0 : (dl[i] > 1.0 ? 1.0 : dl[i]);
        int k = (int)std::floor(x * K);
        if (k > K - 1) k = K - 1;
        sx[k] += x;
        sy[k] += accepted[i];
        ++cnt[k];
    }
    // blocks of the PAV pass: (sum of n*y, sum of n, first knot index)
    struct Blk { double sy, sw; int first; };
    std::vector<Blk> st;
    int m = 0;
    for (int k = 0; k < K; ++k) {
        if (!cnt[k]) continue;
        const double w = (double)cnt[k], r = sy[k] / w;
        knots_x[m] = sx[k] / w;
        st.push_back({r * w, w, m});
        ++m;
        while (st.size() > 1 && st[st.size() - 2].sy / st[st.size() - 2].sw > st.back().sy / st.back().sw) {
            const Blk a = st.back();
            st.pop_back();
            st.back().sy += a.sy;
            st.back().sw += a.sw;
        }
    }
    for (size_t j = 0; j < st.size(); ++j) {
        const int e = j + 1 < st.size() ? st[j + 1].first : m;
        for (int i = st[j].first; i < e; ++i) knots_y[i] = st[j].sy / st[j].sw;
    }
    *n_knots = m;
    return RS_OK;
}

extern "C" rs_status rs_cost_model_fit(const double* n_seq, const double* n_draft, const double* t_sec, int32_t n,
                                       rs_cost_model* io) {
    RS_REQUIRE(n_seq && n_draft && t_sec && io && n >= 4, RS_ERR_INVALID_ARG, "rs_cost_model_fit: need >= 4 samples");
    // normal equations for t - c_draft = b0 + b1*Ns + b2*Nd + b3*relu(Nd - k)*Nd
    double A[4][5] = {{0}};
    for (int i = 0; i < n; ++i) {
        const double relu = n_draft[i] - io->k_sat > 0.0 ? n_draft[i] - io->k_sat : 0.0;
        const double x[4] = {1.0, n_seq[i], n_draft[i], relu * n_draft[i]};
        const double y = t_sec[i] - io->c_draft;
        for (int r = 0; r < 4; ++r) {
            for (int c = 0; c < 4; ++c) A[r][c] += x[r] * x[c];
            A[r][4] += x[r] * y;
        }
    }
    // Gaussian elimination with partial pivoting; an all-zero column (e.g. no sample past
    // k_sat) keeps its coefficient at 0.
    int used[4] = {1, 1, 1, 1};
    for (int col = 0; col < 4; ++col) {
        int piv = col;
        for (int r = col + 1; r < 4; ++r)
            if (std::fabs(A[r][col]) > std::fabs(A[piv][col])) piv = r;
        if (std::fabs(A[piv][col]) < 1e-300) { used[col] = 0; continue; }
        if (piv != col)
            for (int c = 0; c < 5; ++c) std::swap(A[piv][c], A[col][c]);
        for (int r = 0; r < 4; ++r) {
            if (r == col) continue;
            const double f = A[r][col] / A[col][col];
            for (int c = col; c < 5; ++c) A[r][c] -= f * A[col][c];
        }
    }
    double b[4];
    for (int i = 0; i < 4; ++i) b[i] = used[i] ? A[i][4] / A[i][i] : 0.0;
    io->b0 = b[0];
    io->b1 = b[1];
    io->b2 = b[2];
    io->b3 = b[3];
    return RS_OK;
}
