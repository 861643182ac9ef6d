// a2: tree-verification attention on sm_100a (P:76-80 single-pass tree verification; P:213
// "attention primarily incurs cost due to KVCache loading"). Readings Z1-Z4.
//
// Work unit = (sample b, kv head, M tile of 128 query rows). Query rows of a unit are the
// T_b*g (node, head-in-group) pairs, node-major, padded to 128 (UMMA M = 128). Keys are the
// sample's logical slots 0..P_b+T_b-1 in 64-key blocks = one KV page each.
//
// Persistent kernel, one CTA per SM (grid = plan.n_ctas), warp-specialised (attention_kernel.cuh
// has the roles): TMA producers for Q/K and V, an S = Q K^T issuer and an O += P V issuer
// (tcgen05.mma, accumulators in TMEM), two softmax warpgroups taking alternate key blocks, and
// for plans whose tiles all have T*g <= 64 an epilogue warpgroup with items alternating between
// the two 16-lane halves of TMEM so one item's epilogue overlaps the next item's blocks.
// The schedule is built on the host by rs_attn_plan_create from the step's lengths and reused by
// all layers: unit groups (sample, kv head) with M query tiles run as gangs of M CTAs over the
// same key blocks (L2 reuse), balanced contiguous fill with split-KV cuts, merged in-kernel by the
// last CTA of a unit. Consecutive layers are chained with programmatic dependent launch.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "sm100_ptx.cuh"

#include "attention_kernel.cuh"

using namespace attn;

#ifndef RS_ATTN_R16_MAX
#define RS_ATTN_R16_MAX 64   // units with T*g above this use 32-row tiles (else 16-row, several per unit as a gang)
#endif

// Profiling hook state (rs_attn_set_trace).
static unsigned long long* g_trace_buf = nullptr;
static size_t g_trace_bytes = 0;
static constexpr int kOvhBlocksDefault = 2;   // per-item fixed cost in block units (planning)
// Ablation / tuning switches are compile-time only (tools/build_variant.sh -D...): the product
// library has no runtime switch that changes its schedule or results.
#ifndef RS_ATTN_OVH
#define RS_ATTN_OVH -1      // per-item overhead in key blocks; -1: by kernel mode
#endif
#ifndef RS_ATTN_DUAL
#define RS_ATTN_DUAL 1      // dual items (RM = 4) when every unit allows them
#endif
#ifndef RS_ATTN_DYNFRAC
#define RS_ATTN_DYNFRAC 0   // percent of the work left to a dynamic tail queue (measured slower at 6-20: off)
#endif
#ifndef RS_ATTN_DYNPART
#define RS_ATTN_DYNPART 8   // key blocks per dynamic tail part (at least; cap/16 for long lists)
#endif
#ifndef RS_ATTN_L2PROMO
#define RS_ATTN_L2PROMO 3   // CUtensorMapL2promotion of the K/V page loads
#endif
#ifndef RS_ATTN_DBG
#define RS_ATTN_DBG 0       // profiling ablations (results wrong if != 0)
#endif
#ifndef RS_ATTN_PDL
#define RS_ATTN_PDL 1       // programmatic dependent launch between consecutive launches
#endif
static constexpr int kMinPart = 4;      // smallest split-KV part, in blocks

namespace {

// ---------------------------------------------------------------- host: tensor maps
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(ptr);
    }
    return fn;
}

}  // namespace

// ---------------------------------------------------------------- plan
struct rs_attn_plan {
    int B, Hq, Hkv, D, ps, g, n_ctas, NT;
    int rmodes;                 // bit 0: some unit has R = 16, bit 1: some unit has R = 32
    std::vector<int32_t> cta_off;
    std::vector<WorkItem> items;
    std::vector<SplitUnit> units;
    int n_parts;
    size_t off_cta, off_items, off_units, off_counter, off_qorder, off_qctr, off_part_o, off_part_lse, ws_bytes;
    int dyn;                    // dynamic item queue (RM = 1 plans)
    int early_prefix = 0;       // rs_attn_plan_set_early_prefix
    std::vector<int32_t> qorder;
    std::vector<uint8_t> blob;  // [0, off_part_o): header tables, uploaded verbatim
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

extern "C" rs_status rs_attn_plan_create(const int32_t* prefix_len_host, const int32_t* tree_off_host,
                                         int32_t B, int32_t Hq, int32_t Hkv, int32_t head_dim,
                                         int32_t page_size, int32_t num_ctas,
                                         rs_attn_plan** plan_out) {
    RS_REQUIRE(plan_out && (B == 0 || (prefix_len_host && tree_off_host)), RS_ERR_INVALID_ARG,
               "rs_attn_plan_create: null pointer");
    RS_REQUIRE(B >= 0 && Hq > 0 && Hkv > 0 && Hq % Hkv == 0, RS_ERR_INVALID_ARG,
               "rs_attn_plan_create: bad heads Hq=%d Hkv=%d", Hq, Hkv);
    RS_REQUIRE(head_dim == 64 || head_dim == 128, RS_ERR_UNSUPPORTED,
               "rs_attn_plan_create: head_dim %d (supported: 64, 128)", head_dim);
    RS_REQUIRE(page_size == kBlockN, RS_ERR_UNSUPPORTED, "rs_attn_plan_create: page_size %d != 64",
               page_size);
    const int g = Hq / Hkv;
    // per-item overhead (epilogue, Q load) in KV-block units; RS_ATTN_OVH >= 0 overrides (tuning builds)
    const bool ovh_env = RS_ATTN_OVH >= 0;
    int kOvhBlocks = ovh_env ? RS_ATTN_OVH : kOvhBlocksDefault;
    RS_REQUIRE(g <= 16 && (16 % g) == 0, RS_ERR_UNSUPPORTED, "rs_attn_plan_create: group size %d (need g | 16)", g);
    if (num_ctas <= 0) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
        cudaGetLastError();
        num_ctas = sms;
    }
    auto* pl = new rs_attn_plan();
    pl->rmodes = 0;
    pl->B = B; pl->Hq = Hq; pl->Hkv = Hkv; pl->D = head_dim; pl->ps = page_size; pl->g = g;
    pl->NT = B ? tree_off_host[B] : 0;
    // Unit groups: all M query tiles of one (sample, kv head) read the same K/V blocks.
    struct GU { int b, kvh, M, nblk, R, P, node0, T; };
    std::vector<GU> gus;
    int n_tiles = 0;
    for (int b = 0; b < B; ++b) {
        const int T = tree_off_host[b + 1] - tree_off_host[b];
        const int P = prefix_len_host[b];
        if (T < 1 || T > RS_MAX_TREE || P < 0 || T * g > 4 * kM) {
            delete pl;
            rs::set_error("rs_attn_plan_create: sample %d has T=%d P=%d (need 1<=T<=64, T*g<=512)", b, T, P);
            return (T < 1 || T > RS_MAX_TREE) ? RS_ERR_MALFORMED_TREE : RS_ERR_UNSUPPORTED;
        }
        const int nblk = (P + T + kBlockN - 1) / kBlockN;
        const int R = (T * g <= RS_ATTN_R16_MAX) ? 16 : 32;   // rows per TMEM sub-partition
        const int M = (T * g + 4 * R - 1) / (4 * R);   // query tiles per (sample, kv head)
        for (int kvh = 0; kvh < Hkv; ++kvh) gus.push_back({b, kvh, M, nblk, R, P, tree_off_host[b], T});
        pl->rmodes |= (R == 16) ? 1 : 2;
        n_tiles += Hkv * M;
    }
    // Dual items (kernel RM = 4): when every unit group has R = 32 and an even number of query
    // tiles, an item covers tiles (2s, 2s + 1) and each softmax warpgroup owns one, so each K/V
    // tile in shared memory feeds twice the MMA work (config 5: L2 -> SM traffic halved). The
    // gang machinery below then runs on "super tiles" (M / 2 per group). -DRS_ATTN_DUAL=0: off.
    bool dual = pl->rmodes == 2 && RS_ATTN_DUAL != 0;
    for (const GU& u : gus) dual = dual && (u.M % 2 == 0);
    if (dual) {
        for (GU& u : gus) u.M /= 2;
        n_tiles /= 2;
        pl->rmodes = 4;
    }
    const int tile_mul = dual ? 2 : 1;   // item.mtile = tile_mul * (super) tile index
    // per-item overhead by kernel mode (measured sweeps): the 16-warp kernel hides its
    // epilogue behind the next item (2 blocks); the 12-warp kernels run it inline (~5k cycles,
    // ~4-6 blocks); a dual item's block carries two tiles of work, so its overhead is ~1 block
    if (!ovh_env) kOvhBlocks = dual ? 1 : (pl->rmodes == 1 ? kOvhBlocksDefault : 6);
    const int n_ctas = std::max(1, std::min<int>(num_ctas, std::max(n_tiles, 1)));
    // Gangs: the M tiles of a unit group run on M different CTAs ("a gang") that process the
    // same key-block ranges in the same order at the same time, so the K/V blocks the first CTA
    // brings into L2 serve the other M-1 (HBM reads each block ~once instead of M times). CTAs
    // are shared among the tile-count classes in proportion to their work.
    long long Wc[5] = {0, 0, 0, 0, 0};
    for (const GU& u : gus) Wc[u.M] += (long long)(u.nblk + kOvhBlocks) * u.M;
    const long long Wt = Wc[1] + Wc[2] + Wc[3] + Wc[4];
    int gangs[5] = {0, 0, 0, 0, 0};
    int used = 0;
    for (int M = 1; M <= 4; ++M)
        if (Wc[M] > 0) {
            gangs[M] = std::max(1, (int)((double)n_ctas * Wc[M] / std::max(Wt, 1ll) / M));
            used += gangs[M] * M;
        }
    while (used > n_ctas) {   // (rounding up to one gang per class can overshoot)
        int worst = 0;
        for (int M = 1; M <= 4; ++M)
            if (gangs[M] > 1 && (worst == 0 || gangs[M] * M > gangs[worst] * worst)) worst = M;
        if (worst == 0) break;
        --gangs[worst];
        used -= worst;
    }
    if (used > n_ctas) {
        // too few CTAs for one gang per class: multi-tile groups run tile by tile on single
        // CTAs (class 1, no L2 sharing)
        for (int M = 2; M <= 4; ++M) {
            Wc[1] += Wc[M];
            used -= gangs[M] * M;
            gangs[M] = 0;
            Wc[M] = 0;
        }
        if (gangs[1] == 0) { gangs[1] = 1; used += 1; }
        while (used > n_ctas) { --gangs[1]; --used; }
    }
    for (;;) {   // spend leftover CTAs on the class with the most work per CTA that still fits
        int best = 0;
        double load = -1.0;
        for (int M = 1; M <= 4; ++M)
            if (gangs[M] > 0 && used + M <= n_ctas) {
                const double l = (double)Wc[M] / (gangs[M] * M);
                if (l > load) { load = l; best = M; }
            }
        if (best == 0) break;
        ++gangs[best];
        used += best;
    }
    // Balanced contiguous fill with split-KV cuts over the gangs of one class: unit groups are
    // poured, in order, into gangs of a common capacity (the smallest that fits, below); parts
    // are never smaller than kMinPart blocks.
    struct Seg { int gu, tile, start, end; };   // tile -1: every tile of the gang
    std::vector<std::vector<WorkItem>> per_cta(n_ctas);
    std::vector<Seg> dyn_segs;          // hybrid tail parts of the current class
    std::vector<WorkItem> dyn_items;    // ... as work items (after every static list)
    int n_parts = 0;
    int cta_base = 0;
    for (int M = 1; M <= 4; ++M) {
        const int G = gangs[M];
        if (G == 0) continue;
        std::vector<std::vector<Seg>> per_g(G);
        // work entries of this class: (unit group, tile); tile -1 = the whole gang
        std::vector<std::pair<int, int>> entries;
        for (int gi = 0; gi < (int)gus.size(); ++gi) {
            if (gus[gi].M == M) entries.push_back({gi, M == 1 ? 0 : -1});
            else if (M == 1 && gangs[gus[gi].M] == 0)
                for (int m = 0; m < gus[gi].M; ++m) entries.push_back({gi, m});
        }
        // Balanced fill: the smallest per-gang capacity (blocks + kOvhBlocks per item, so every
        // extra split part pays its overhead) for which pouring the entries in order into the G
        // gangs fits, found by bisection; then the fill at that capacity. (A running-average
        // target drifted: the last gangs absorbed every split overhead, 76 vs 63 blocks of cost
        // on config 2.)
        std::vector<std::vector<std::pair<int, int>>> where_of(entries.size());
        long long W = 0;
        int max_nblk = 0;
        for (auto& e : entries) {
            W += gus[e.first].nblk + kOvhBlocks;
            max_nblk = std::max(max_nblk, gus[e.first].nblk);
        }
        // hybrid (single-tile class, no dual items): the static lists take a (1 - DYNFRAC) share
        // of that capacity and what does not fit becomes small split parts in a global queue
        // that CTAs pull from once their own list is done (atomic counter): the launch then ends
        // when the average CTA does, not the slowest (SMs do not all stream HBM at the same rate;
        // config 2 CTA end times spread 48-62 us with balanced static lists).
        const bool hybrid = M == 1 && !dual && RS_ATTN_DYNFRAC > 0;
        int dyn_part = RS_ATTN_DYNPART;
        auto fill = [&](long long cap, bool commit, bool to_dyn) -> bool {
            int v = 0;
            long long load = 0;
            for (int ei = 0; ei < (int)entries.size(); ++ei) {
                const int gi = entries[ei].first;
                int rem = gus[gi].nblk, start = 0;
                while (rem > 0) {
                    if (v >= G) {
                        if (!to_dyn) return false;
                        // the rest of this entry and every later one: tail parts
                        const int take = rem < dyn_part + kMinPart ? rem : dyn_part;
                        if (commit) {
                            where_of[ei].push_back({-1, (int)dyn_segs.size()});
                            dyn_segs.push_back({gi, entries[ei].second, start, start + take});
                        }
                        start += take;
                        rem -= take;
                        continue;
                    }
                    const long long room = cap - load - kOvhBlocks;
                    int take;
                    if (room >= rem) {
                        take = rem;
                    } else {
                        take = (int)std::min<long long>(room, rem - kMinPart);   // leave >= kMinPart
                        if (take < kMinPart) {
                            if (load == 0) take = rem;   // an empty gang takes the whole entry
                            else { ++v; load = 0; continue; }
                        }
                    }
                    if (commit) {
                        where_of[ei].push_back({v, (int)per_g[v].size()});
                        per_g[v].push_back({gi, entries[ei].second, start, start + take});
                    }
                    load += take + kOvhBlocks;
                    start += take;
                    rem -= take;
                }
            }
            return true;
        };
        long long lo = std::max<long long>((W + G - 1) / G, 1), hi = lo + max_nblk + 2 * kOvhBlocks + kMinPart;
        while (!fill(hi, false, false)) hi *= 2;
        while (lo < hi) {
            const long long mid = (lo + hi) / 2;
            if (fill(mid, false, false)) hi = mid;
            else lo = mid + 1;
        }
        dyn_part = std::max<int>(RS_ATTN_DYNPART, (int)(lo / 16));
        if (hybrid) fill(std::max<long long>(lo * (100 - RS_ATTN_DYNFRAC) / 100, kMinPart + kOvhBlocks), true, true);
        else fill(lo, true, false);
        for (const Seg& sg : dyn_segs) {   // (hybrid: M == 1)
            const GU& u = gus[sg.gu];
            dyn_items.push_back({u.b, u.kvh, tile_mul * sg.tile, sg.start, sg.end, -1, u.R, -1, u.P, u.node0, u.T, 0});
        }
        dyn_segs.clear();
        // expand: gang v -> CTAs cta_base + v*M + m (tile m); split units per tile
        for (int vv = 0; vv < G; ++vv)
            for (int m = 0; m < M; ++m)
                for (const Seg& sg : per_g[vv]) {
                    const GU& u = gus[sg.gu];
                    per_cta[cta_base + vv * M + m].push_back(
                        {u.b, u.kvh, tile_mul * (sg.tile >= 0 ? sg.tile : m), sg.start, sg.end, -1, u.R, -1, u.P,
                         u.node0, u.T, 0});
                }
        for (int ei = 0; ei < (int)entries.size(); ++ei) {
            if (where_of[ei].size() <= 1) continue;
            const GU& u = gus[entries[ei].first];
            for (int m = 0; m < M; ++m) {
                const int uid = (int)pl->units.size();
                const int tile = tile_mul * (entries[ei].second >= 0 ? entries[ei].second : m);
                const int k = (int)where_of[ei].size();
                pl->units.push_back({u.b, u.kvh, tile, k, n_parts, u.R});
                // dual: a second unit for tile + 1 whose k parts follow (item.pad = k)
                if (dual) pl->units.push_back({u.b, u.kvh, tile + 1, k, n_parts + k, u.R});
                for (int i = 0; i < k; ++i) {
                    const auto& wc = where_of[ei][i];
                    WorkItem& it = wc.first >= 0 ? per_cta[cta_base + wc.first * M + m][wc.second]
                                                 : dyn_items[wc.second];
                    it.part = n_parts + i;
                    it.unit = uid;
                    it.pad = dual ? k : 0;
                }
                n_parts += tile_mul * k;
            }
        }
        cta_base += G * M;
    }
    pl->cta_off.assign(n_ctas + 1, 0);
    for (int c = 0; c < n_ctas; ++c) {
        pl->cta_off[c] = (int)pl->items.size();
        pl->items.insert(pl->items.end(), per_cta[c].begin(), per_cta[c].end());
    }
    pl->cta_off[n_ctas] = (int)pl->items.size();
    pl->n_ctas = n_ctas;
    // Dynamic tail: item indices after the static lists, longest first, pulled by CTAs that
    // finished their own list (p.dyn); none -> pure static schedule.
    pl->qorder.clear();
    for (size_t i = 0; i < dyn_items.size(); ++i) pl->qorder.push_back((int)(pl->items.size() + i));
    pl->items.insert(pl->items.end(), dyn_items.begin(), dyn_items.end());
    std::stable_sort(pl->qorder.begin(), pl->qorder.end(), [&](int x, int y) {
        return pl->items[x].blk_end - pl->items[x].blk_begin > pl->items[y].blk_end - pl->items[y].blk_begin;
    });
    pl->dyn = pl->qorder.empty() ? 0 : 1;
    pl->n_parts = n_parts;
    pl->off_cta = 0;
    pl->off_items = align_up(sizeof(int32_t) * (n_ctas + 1), 256);
    pl->off_units = align_up(pl->off_items + sizeof(WorkItem) * pl->items.size(), 256);
    pl->off_counter = align_up(pl->off_units + sizeof(SplitUnit) * pl->units.size(), 256);
    pl->off_qorder = align_up(pl->off_counter + sizeof(int32_t) * pl->units.size(), 256);
    pl->off_qctr = align_up(pl->off_qorder + sizeof(int32_t) * pl->qorder.size(), 256);
    pl->off_part_o = align_up(pl->off_qctr + sizeof(int32_t) * 2, 256);
    pl->off_part_lse = align_up(pl->off_part_o + sizeof(float) * (size_t)n_parts * kM * head_dim, 256);
    pl->ws_bytes = align_up(pl->off_part_lse + sizeof(float) * (size_t)n_parts * kM, 256);
    pl->blob.assign(pl->off_part_o, 0);   // includes the zeroed split-unit counters
    memcpy(pl->blob.data() + pl->off_cta, pl->cta_off.data(), sizeof(int32_t) * (n_ctas + 1));
    if (!pl->items.empty())
        memcpy(pl->blob.data() + pl->off_items, pl->items.data(), sizeof(WorkItem) * pl->items.size());
    if (!pl->units.empty())
        memcpy(pl->blob.data() + pl->off_units, pl->units.data(), sizeof(SplitUnit) * pl->units.size());
    if (!pl->qorder.empty())
        memcpy(pl->blob.data() + pl->off_qorder, pl->qorder.data(), sizeof(int32_t) * pl->qorder.size());
    *plan_out = pl;
    return RS_OK;
}

extern "C" size_t rs_attn_plan_workspace_bytes(const rs_attn_plan* plan) {
    return plan ? plan->ws_bytes : 0;
}

extern "C" rs_status rs_attn_plan_upload(const rs_attn_plan* plan, void* ws, size_t ws_bytes, void* stream) {
    rs::bind_device(ws);
    RS_REQUIRE(plan && ws, RS_ERR_INVALID_ARG, "rs_attn_plan_upload: null pointer");
    RS_REQUIRE(ws_bytes >= plan->ws_bytes, RS_ERR_WORKSPACE, "rs_attn_plan_upload: workspace %zu < %zu",
               ws_bytes, plan->ws_bytes);
    RS_REQUIRE((reinterpret_cast<uintptr_t>(ws) & 255) == 0, RS_ERR_INVALID_ARG,
               "rs_attn_plan_upload: workspace not 256-byte aligned");
    RS_CUDA_CHECK(cudaMemcpyAsync(ws, plan->blob.data(), plan->blob.size(), cudaMemcpyHostToDevice,
                                  rs::as_stream(stream)));
    return RS_OK;
}

extern "C" rs_status rs_attn_plan_info(const rs_attn_plan* plan, int32_t* num_ctas, int32_t* num_items,
                                       int32_t* num_split_units) {
    RS_REQUIRE(plan, RS_ERR_INVALID_ARG, "rs_attn_plan_info: null plan");
    if (num_ctas) *num_ctas = plan->n_ctas;
    if (num_items) *num_items = (int32_t)plan->items.size();
    if (num_split_units) *num_split_units = (int32_t)plan->units.size();
    return RS_OK;
}

extern "C" rs_status rs_attn_plan_items(const rs_attn_plan* plan, int32_t* cta_off, int32_t* items) {
    RS_REQUIRE(plan, RS_ERR_INVALID_ARG, "rs_attn_plan_items: null plan");
    if (cta_off) memcpy(cta_off, plan->cta_off.data(), sizeof(int32_t) * plan->cta_off.size());
    if (items && !plan->items.empty()) memcpy(items, plan->items.data(), sizeof(WorkItem) * plan->items.size());
    return RS_OK;
}

extern "C" void rs_attn_plan_destroy(rs_attn_plan* plan) { delete plan; }

extern "C" rs_status rs_attn_plan_set_early_prefix(rs_attn_plan* plan, int32_t enable) {
    RS_REQUIRE(plan, RS_ERR_INVALID_ARG, "rs_attn_plan_set_early_prefix: null plan");
    plan->early_prefix = enable ? 1 : 0;
    return RS_OK;
}

extern "C" rs_status rs_attn_set_trace(void* buf, size_t bytes) {
    g_trace_buf = static_cast<unsigned long long*>(buf);
    g_trace_bytes = buf ? bytes : 0;
    return RS_OK;
}

template <int D>
static rs_status launch_attn(const rs_attn_plan* pl, const void* q, const void* k_pages, const void* v_pages,
                             int64_t num_pages, const int32_t* block_table, int32_t max_pages,
                             const int32_t* prefix_len, const int32_t* tree_off, const uint64_t* tree_mask,
                             float sm_scale, void* out, float* lse, void* ws, cudaStream_t st) {
    using C = Cfg<D>;
    PFN_encodeTiled enc = get_encode();
    RS_REQUIRE(enc, RS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap tmQ, tmK, tmV, tmO;
    // Q (load) and O (store) share the geometry [NT][Hq][D]; box = 16 rows (16/g nodes x g heads) x 64 d
    const void* qo[2] = {q, out};
    CUtensorMap* tqo[2] = {&tmQ, &tmO};
    for (int i = 0; i < 2; ++i) {
        cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)pl->Hq, (cuuint64_t)std::max(pl->NT, 1)};
        cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)pl->Hq * D * 2};
        cuuint32_t box[3] = {64, (cuuint32_t)pl->g, (cuuint32_t)(16 / pl->g)};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = enc(tqo[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(qo[i]), dims, strides, box,
                         es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        RS_REQUIRE(r == CUDA_SUCCESS, RS_ERR_CUDA, "tensor map Q/O failed (%d)", (int)r);
    }
    // L2 sector promotion of the K/V page loads (-DRS_ATTN_L2PROMO = 0..3 for measurements)
    const CUtensorMapL2promotion kv_promo = (CUtensorMapL2promotion)(RS_ATTN_L2PROMO & 3);
    const void* kv[2] = {k_pages, v_pages};
    CUtensorMap* tm[2] = {&tmK, &tmV};
    for (int i = 0; i < 2; ++i) {
        cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)num_pages * pl->Hkv * kBlockN};
        cuuint64_t strides[1] = {(cuuint64_t)D * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)kBlockN};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(tm[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(kv[i]), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         kv_promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        RS_REQUIRE(r == CUDA_SUCCESS, RS_ERR_CUDA, "tensor map KV failed (%d)", (int)r);
    }
    Params prm;
    uint8_t* w = static_cast<uint8_t*>(ws);
    prm.cta_off = reinterpret_cast<const int32_t*>(w + pl->off_cta);
    prm.items = reinterpret_cast<const WorkItem*>(w + pl->off_items);
    prm.part_o = reinterpret_cast<float*>(w + pl->off_part_o);
    prm.part_lse = reinterpret_cast<float*>(w + pl->off_part_lse);
    prm.units = reinterpret_cast<const SplitUnit*>(w + pl->off_units);
    prm.unit_counter = reinterpret_cast<int*>(w + pl->off_counter);
    prm.qorder = reinterpret_cast<const int32_t*>(w + pl->off_qorder);
    prm.qctr = reinterpret_cast<int*>(w + pl->off_qctr);
    prm.n_items = (int)pl->qorder.size();   // dynamic tail items
    prm.dyn = pl->dyn;
    prm.prefix_len = prefix_len;
    prm.tree_off = tree_off;
    prm.tree_mask = tree_mask;
    prm.block_table = block_table;
    prm.max_pages = max_pages;
    prm.Hq = pl->Hq;
    prm.Hkv = pl->Hkv;
    prm.g = pl->g;
    prm.scale_log2 = sm_scale * 1.4426950408889634f;
    prm.out = static_cast<__nv_bfloat16*>(out);
    prm.lse = lse;
    prm.dbg = RS_ATTN_DBG;   // profiling ablations only (variant builds)
    prm.early_prefix = pl->early_prefix;
    prm.trace = (g_trace_bytes >= (size_t)pl->n_ctas * kTraceJ * 16 * sizeof(unsigned long long)) ? g_trace_buf
                                                                                               : nullptr;
    // row mode: kernels specialised for plans whose tiles all use R = 16 (half-split rows) or all
    // R = 32, so each carries only the registers of its own softmax path; mixed plans take both.
    const int rm = pl->rmodes == 1 ? 1 : (pl->rmodes == 2 ? 2 : (pl->rmodes == 4 ? 4 : 3));
    auto kern = rm == 1 ? tree_attn_kernel<D, 1>
                        : (rm == 2 ? tree_attn_kernel<D, 2> : (rm == 4 ? tree_attn_kernel<D, 4> : tree_attn_kernel<D, 3>));
    const int smem_bytes = rm == 1 ? Cfg<D, 1>::kSmemBytes : (rm == 4 ? Cfg<D, 4>::kSmemBytes : Cfg<D, 2>::kSmemBytes);
    static bool attr_set[2][5] = {};
    if (!attr_set[D == 128][rm]) {
        RS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
        attr_set[D == 128][rm] = true;
    }
    const int threads = rm == 1 ? KT<1>::kThreads : (rm == 4 ? KT<4>::kThreads : KT<2>::kThreads);
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)pl->n_ctas);
    lc.blockDim = dim3((unsigned)threads);
    lc.dynamicSmemBytes = (size_t)smem_bytes;
    lc.stream = st;
    cudaLaunchAttribute la[1];
    constexpr bool pdl = RS_ATTN_PDL != 0;
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = la;
    lc.numAttrs = pdl ? 1 : 0;
    RS_CUDA_CHECK(cudaLaunchKernelEx(&lc, kern, tmQ, tmK, tmV, tmO, prm));
    RS_LAUNCH_CHECK();
    return RS_OK;
}

extern "C" rs_status rs_tree_verify_attention(const rs_attn_plan* plan, const void* q, const void* k_pages,
                                              const void* v_pages, int64_t num_pages,
                                              const int32_t* block_table, int32_t max_pages,
                                              const int32_t* prefix_len, const int32_t* tree_off,
                                              const uint64_t* tree_mask, int32_t B, int32_t Hq,
                                              int32_t Hkv, int32_t head_dim, int32_t page_size,
                                              float sm_scale, void* out, float* lse, void* ws,
                                              size_t ws_bytes, void* stream) {
    rs::bind_device(q);
    RS_REQUIRE(plan, RS_ERR_INVALID_ARG, "rs_tree_verify_attention: null plan");
    RS_REQUIRE(plan->B == B && plan->Hq == Hq && plan->Hkv == Hkv && plan->D == head_dim &&
                   plan->ps == page_size,
               RS_ERR_INVALID_ARG, "rs_tree_verify_attention: arguments differ from the plan");
    RS_REQUIRE(ws && ws_bytes >= plan->ws_bytes, RS_ERR_WORKSPACE,
               "rs_tree_verify_attention: workspace %zu < %zu", ws_bytes, plan->ws_bytes);
    if (B == 0 || plan->items.empty()) return RS_OK;
    RS_REQUIRE(q && k_pages && v_pages && block_table && prefix_len && tree_off && tree_mask && out,
               RS_ERR_INVALID_ARG, "rs_tree_verify_attention: null pointer");
    RS_REQUIRE(num_pages > 0 && num_pages * Hkv * kBlockN < (1ll << 31), RS_ERR_UNSUPPORTED,
               "rs_tree_verify_attention: num_pages out of range");
    RS_REQUIRE(((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k_pages) |
                 reinterpret_cast<uintptr_t>(v_pages) | reinterpret_cast<uintptr_t>(out)) & 15) == 0,
               RS_ERR_INVALID_ARG, "rs_tree_verify_attention: pointers must be 16-byte aligned");
    cudaStream_t st = rs::as_stream(stream);
    if (head_dim == 128)
        return launch_attn<128>(plan, q, k_pages, v_pages, num_pages, block_table, max_pages, prefix_len,
                                tree_off, tree_mask, sm_scale, out, lse, ws, st);
    return launch_attn<64>(plan, q, k_pages, v_pages, num_pages, block_table, max_pages, prefix_len, tree_off,
                           tree_mask, sm_scale, out, lse, ws, st);
}

extern "C" rs_status rs_tree_verify_attention_layers(
    const rs_attn_plan* plan, int32_t L, const void* const* q_layers, const void* const* k_layers,
    const void* const* v_layers, int64_t num_pages, const int32_t* block_table, int32_t max_pages,
    const int32_t* prefix_len, const int32_t* tree_off, const uint64_t* tree_mask, int32_t B, int32_t Hq,
    int32_t Hkv, int32_t head_dim, int32_t page_size, float sm_scale, void* const* out_layers,
    float* const* lse_layers, void* ws, size_t ws_bytes, void* stream) {
    rs::bind_device(block_table);
    RS_REQUIRE(L >= 0 && q_layers && k_layers && v_layers && out_layers, RS_ERR_INVALID_ARG,
               "rs_tree_verify_attention_layers: null layer arrays");
    for (int32_t l = 0; l < L; ++l) {
        rs_status st = rs_tree_verify_attention(plan, q_layers[l], k_layers[l], v_layers[l], num_pages, block_table,
                                                max_pages, prefix_len, tree_off, tree_mask, B, Hq, Hkv, head_dim,
                                                page_size, sm_scale, out_layers[l], lse_layers ? lse_layers[l] : nullptr,
                                                ws, ws_bytes, stream);
        if (st != RS_OK) return st;
    }
    return RS_OK;
}
