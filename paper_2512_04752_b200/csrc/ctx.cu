// rs_ctx: one generation instance's registrations (KV pools of the SSM and the LLM, non-owning)
// and its drafting-strategy state (the acceptance fit F and the t_sd cost model behind a
// selector), plus rs_calibrate: the offline profiling of P:192 / P:213-215 ("we construct a
// regression model and perform offline profiling of the data for model training"; P:427 one-time
// profiling) done on THIS box with the library's own kernels — the verification attention of
// every registered LLM layer (+ the tree-mask build) timed on a grid of (B, P, T) batches, the
// non-attention per-token cost added by the caller (the dense GEMMs are outside this library),
// and rs_cost_model_fit run on the result.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"

struct rs_ctx {
    rs_ctx_desc desc{};
    struct Model {
        int32_t L = 0, num_pages = 0, Hkv = 0, d = 0;
        std::vector<void*> k, v;
    } model[2];                       // 0 = SSM, 1 = LLM
    rs_cost_model cost{};
    std::vector<double> kx, ky;
    rs_selector* sel = nullptr;
};

static rs_status rebuild_selector(rs_ctx* c) {
    if (c->kx.empty()) return RS_OK;   // no F yet
    rs_selector* s = nullptr;
    const rs_status st = rs_selector_create(&c->cost, c->kx.data(), c->ky.data(), (int32_t)c->kx.size(), &s);
    if (st != RS_OK) return st;
    if (c->sel) rs_selector_destroy(c->sel);
    c->sel = s;                        // a fresh selector: the t_sd bucket cache starts empty
    return RS_OK;
}

extern "C" rs_status rs_ctx_create(const rs_ctx_desc* desc, rs_ctx** out) {
    RS_REQUIRE(desc && out && desc->world >= 1 && desc->rank >= 0 && desc->rank < desc->world &&
                   desc->page_size > 0,
               RS_ERR_INVALID_ARG, "rs_ctx_create: bad descriptor");
    auto* c = new rs_ctx();
    c->desc = *desc;
    c->cost.seq_bucket = 256;
    c->cost.draft_bucket = 4;
    c->cost.k_sat = 1e30;
    *out = c;
    return RS_OK;
}

extern "C" rs_status rs_ctx_destroy(rs_ctx* c) {
    if (!c) return RS_OK;
    if (c->sel) rs_selector_destroy(c->sel);
    delete c;
    return RS_OK;
}

extern "C" rs_status rs_ctx_register_kv(rs_ctx* c, int32_t model, int32_t L, void* const* k_layers,
                                        void* const* v_layers, int32_t num_pages, int32_t Hkv, int32_t head_dim) {
    RS_REQUIRE(c && (model == 0 || model == 1) && L >= 0 && num_pages >= 0 && Hkv > 0 && head_dim > 0 &&
                   (L == 0 || (k_layers && v_layers)),
               RS_ERR_INVALID_ARG, "rs_ctx_register_kv: bad args");
    auto& m = c->model[model];
    m.L = L;
    m.num_pages = num_pages;
    m.Hkv = Hkv;
    m.d = head_dim;
    m.k.assign(k_layers, k_layers + L);
    m.v.assign(v_layers, v_layers + L);
    return RS_OK;
}

extern "C" rs_status rs_ctx_set_strategy(rs_ctx* c, const rs_cost_model* cost, const double* knots_x,
                                         const double* knots_y, int32_t n_knots) {
    RS_REQUIRE(c && (cost || (knots_x && knots_y && n_knots >= 1)), RS_ERR_INVALID_ARG,
               "rs_ctx_set_strategy: bad args");
    const rs_cost_model old = c->cost;
    const std::vector<double> okx = c->kx, oky = c->ky;
    if (cost) c->cost = *cost;
    if (knots_x && knots_y && n_knots >= 1) {
        c->kx.assign(knots_x, knots_x + n_knots);
        c->ky.assign(knots_y, knots_y + n_knots);
    }
    const rs_status st = rebuild_selector(c);
    if (st != RS_OK) {   // invalid input: the ctx keeps its previous state
        c->cost = old;
        c->kx = okx;
        c->ky = oky;
    }
    return st;
}

extern "C" rs_status rs_ctx_get_strategy(const rs_ctx* c, rs_cost_model* cost, double* knots_x, double* knots_y,
                                         int32_t* n_knots) {
    RS_REQUIRE(c && n_knots, RS_ERR_INVALID_ARG, "rs_ctx_get_strategy: bad args");
    if (cost) *cost = c->cost;
    const int32_t cap = *n_knots;
    *n_knots = (int32_t)c->kx.size();
    if (knots_x && knots_y) {
        RS_REQUIRE(cap >= (int32_t)c->kx.size(), RS_ERR_INVALID_ARG, "rs_ctx_get_strategy: knot capacity %d < %zu",
                   cap, c->kx.size());
        std::copy(c->kx.begin(), c->kx.end(), knots_x);
        std::copy(c->ky.begin(), c->ky.end(), knots_y);
    }
    return RS_OK;
}

extern "C" rs_selector* rs_ctx_selector(rs_ctx* c) { return c ? c->sel : nullptr; }

extern "C" rs_status rs_ctx_fit_acceptance(rs_ctx* c, const double* dl, const double* accepted, int64_t n,
                                           int32_t n_buckets) {
    RS_REQUIRE(c && n_buckets >= 1, RS_ERR_INVALID_ARG, "rs_ctx_fit_acceptance: bad args");
    std::vector<double> kx(n_buckets), ky(n_buckets);
    int32_t m = 0;
    const rs_status st = rs_acceptance_fit(dl, accepted, n, n_buckets, kx.data(), ky.data(), &m);
    if (st != RS_OK) return st;
    return rs_ctx_set_strategy(c, nullptr, kx.data(), ky.data(), m);
}

// ------------------------------------------------------------------ rs_calibrate
namespace {
constexpr size_t kAlign = 256;
inline size_t up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct PointLayout {   // device metadata of one grid point inside the workspace
    size_t prefix, tree_off, parent, bt, mask, depth, flags, plan, total;
};
PointLayout layout(int B, int T, int max_pages, size_t plan_bytes) {
    PointLayout l{};
    size_t o = 0;
    l.prefix = o;   o += up(sizeof(int32_t) * B);
    l.tree_off = o; o += up(sizeof(int32_t) * (B + 1));
    l.parent = o;   o += up(sizeof(int32_t) * (size_t)B * T);
    l.bt = o;       o += up(sizeof(int32_t) * (size_t)B * max_pages);
    l.mask = o;     o += up(sizeof(uint64_t) * (size_t)B * T);
    l.depth = o;    o += up(sizeof(int32_t) * (size_t)B * T);
    l.flags = o;    o += up(sizeof(int32_t) * B);
    l.plan = o;     o += up(plan_bytes);
    l.total = o;
    return l;
}
}  // namespace

static rs_status calib_check(const rs_ctx* c, const rs_calib_desc* d) {
    RS_REQUIRE(c && d && d->n_points >= 4 && d->B && d->P && d->T && d->reps >= 1 && d->Hq > 0, RS_ERR_INVALID_ARG,
               "rs_calibrate: need a descriptor with >= 4 grid points and reps >= 1");
    const auto& m = c->model[1];
    RS_REQUIRE(m.L >= 1, RS_ERR_INVALID_ARG, "rs_calibrate: no LLM KV registered (rs_ctx_register_kv model 1)");
    RS_REQUIRE(d->Hq % m.Hkv == 0, RS_ERR_INVALID_ARG, "rs_calibrate: Hq %% Hkv != 0");
    const int ps = c->desc.page_size;
    for (int i = 0; i < d->n_points; ++i) {
        const int B = d->B[i], P = d->P[i], T = d->T[i];
        RS_REQUIRE(B >= 1 && P >= 0 && T >= 1 && T <= RS_MAX_TREE, RS_ERR_INVALID_ARG, "rs_calibrate: point %d", i);
        const int64_t pages = (int64_t)B * ((P + T + ps - 1) / ps);
        RS_REQUIRE(pages <= m.num_pages, RS_ERR_INVALID_ARG,
                   "rs_calibrate: point %d needs %lld pages > %d registered", i, (long long)pages, m.num_pages);
        RS_REQUIRE((size_t)B * T * d->Hq * m.d <= d->qo_elems, RS_ERR_WORKSPACE,
                   "rs_calibrate: Q/O scratch too small for point %d", i);
    }
    return RS_OK;
}

extern "C" size_t rs_calibrate_workspace_bytes(const rs_ctx* c, const rs_calib_desc* d) {
    if (calib_check(c, d) != RS_OK) return 0;
    const auto& m = c->model[1];
    const int ps = c->desc.page_size;
    size_t need = 0;
    for (int i = 0; i < d->n_points; ++i) {
        const int B = d->B[i], P = d->P[i], T = d->T[i];
        std::vector<int32_t> pl(B, P), to(B + 1);
        for (int b = 0; b <= B; ++b) to[b] = b * T;
        rs_attn_plan* plan = nullptr;
        if (rs_attn_plan_create(pl.data(), to.data(), B, d->Hq, m.Hkv, m.d, ps, 0, &plan) != RS_OK) return 0;
        const size_t pb = rs_attn_plan_workspace_bytes(plan);
        rs_attn_plan_destroy(plan);
        need = std::max(need, layout(B, T, (P + T + ps - 1) / ps, pb).total);
    }
    return need;
}

extern "C" rs_status rs_calibrate(rs_ctx* c, const rs_calib_desc* d, double* t_attn_out) {
    rs_status st = calib_check(c, d);
    if (st != RS_OK) return st;
    RS_REQUIRE(!c->kx.empty(), RS_ERR_INVALID_ARG, "rs_calibrate: set F first (rs_ctx_set_strategy / fit)");
    const auto& m = c->model[1];
    const int ps = c->desc.page_size, L = m.L;
    cudaStream_t s = rs::as_stream(d->stream);
    cudaEvent_t e0, e1;
    RS_CUDA_CHECK(cudaEventCreate(&e0));
    RS_CUDA_CHECK(cudaEventCreate(&e1));
    std::vector<const void*> qa(L, d->q), ka(m.k.begin(), m.k.end()), va(m.v.begin(), m.v.end());
    std::vector<void*> oa(L, d->out);
    std::vector<double> ns(d->n_points), nd(d->n_points), tt(d->n_points);
    const float scale = 1.0f / sqrtf((float)m.d);
    for (int i = 0; i < d->n_points && st == RS_OK; ++i) {
        const int B = d->B[i], P = d->P[i], T = d->T[i];
        const int npg = (P + T + ps - 1) / ps;
        // synthetic batch: every sample prefix P, a chain tree of T nodes, pages b*npg .. b*npg+npg-1
        std::vector<int32_t> pl(B, P), to(B + 1), par((size_t)B * T), bt((size_t)B * npg);
        for (int b = 0; b <= B; ++b) to[b] = b * T;
        for (int b = 0; b < B; ++b)
            for (int t = 0; t < T; ++t) par[(size_t)b * T + t] = t - 1;
        for (size_t k = 0; k < bt.size(); ++k) bt[k] = (int32_t)k;
        rs_attn_plan* plan = nullptr;
        st = rs_attn_plan_create(pl.data(), to.data(), B, d->Hq, m.Hkv, m.d, ps, 0, &plan);
        if (st != RS_OK) break;
        const PointLayout lay = layout(B, T, npg, rs_attn_plan_workspace_bytes(plan));
        if (lay.total > d->ws_bytes) {
            rs_attn_plan_destroy(plan);
            rs::set_error("rs_calibrate: workspace %zu < %zu (rs_calibrate_workspace_bytes)", d->ws_bytes, lay.total);
            st = RS_ERR_WORKSPACE;
            break;
        }
        auto* w = static_cast<uint8_t*>(d->ws);
        auto at = [&](size_t off) { return w + off; };
        cudaMemcpyAsync(at(lay.prefix), pl.data(), sizeof(int32_t) * B, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(at(lay.tree_off), to.data(), sizeof(int32_t) * (B + 1), cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(at(lay.parent), par.data(), sizeof(int32_t) * par.size(), cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(at(lay.bt), bt.data(), sizeof(int32_t) * bt.size(), cudaMemcpyHostToDevice, s);
        st = rs_attn_plan_upload(plan, at(lay.plan), lay.total - lay.plan, d->stream);
        std::vector<float> ms;
        for (int r = 0; r <= d->reps && st == RS_OK; ++r) {   // r = 0: warm-up
            cudaEventRecord(e0, s);
            st = rs_tree_build_mask(reinterpret_cast<int32_t*>(at(lay.parent)), reinterpret_cast<int32_t*>(at(lay.tree_off)),
                                    B, reinterpret_cast<uint64_t*>(at(lay.mask)), reinterpret_cast<int32_t*>(at(lay.depth)),
                                    reinterpret_cast<int32_t*>(at(lay.flags)), d->stream);
            if (st != RS_OK) break;
            st = rs_tree_verify_attention_layers(
                plan, L, qa.data(), ka.data(), va.data(), m.num_pages, reinterpret_cast<int32_t*>(at(lay.bt)), npg,
                reinterpret_cast<int32_t*>(at(lay.prefix)), reinterpret_cast<int32_t*>(at(lay.tree_off)),
                reinterpret_cast<uint64_t*>(at(lay.mask)), B, d->Hq, m.Hkv, m.d, ps, scale, oa.data(), nullptr,
                at(lay.plan), lay.total - lay.plan, d->stream);
            cudaEventRecord(e1, s);
            if (st != RS_OK) break;
            if (cudaEventSynchronize(e1) != cudaSuccess) {
                rs::set_error("rs_calibrate: %s", cudaGetErrorString(cudaGetLastError()));
                st = RS_ERR_CUDA;
                break;
            }
            float x = 0.f;
            cudaEventElapsedTime(&x, e0, e1);
            if (r > 0) ms.push_back(x);
        }
        rs_attn_plan_destroy(plan);
        if (st != RS_OK) break;
        std::sort(ms.begin(), ms.end());
        const double t_attn = 1e-3 * ms[ms.size() / 2];   // median
        if (t_attn_out) t_attn_out[i] = t_attn;
        ns[i] = (double)B * P;
        nd[i] = (double)B * T;
        tt[i] = c->cost.c_draft + t_attn + d->dense_s_per_token * nd[i];
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (st != RS_OK) return st;
    rs_cost_model fit = c->cost;
    st = rs_cost_model_fit(ns.data(), nd.data(), tt.data(), d->n_points, &fit);
    if (st != RS_OK) return st;
    return rs_ctx_set_strategy(c, &fit, nullptr, nullptr, 0);
}
