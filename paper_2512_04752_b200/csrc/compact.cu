// a4: KV commit of the accepted path (Markov property; Z2).
//   for k = 1..a_b: K/V[b, P_b+k] <- K/V[b, P_b+path[k]]   (all layers, all kv heads)
// The per-sample commit (sequential ascending-k semantics, lane-owned 128-bit gathers and
// scatters, ballot-scanned move list) is rs::compact_sample in compact_tail.cuh, which the fused
// acceptance kernels (rs_tree_accept_compact) run in their tail; this kernel runs it standalone.
#include "common.cuh"
#include "compact_tail.cuh"

namespace {

constexpr int kLayersPerCta = 2;
constexpr int kThreads = 256;

// One CTA per (sample, group of kLayersPerCta layers): rs::compact_sample over that group's lanes.
__global__ void __launch_bounds__(kThreads)
kv_compact_kernel(const __grid_constant__ rs::CompactArgs A, const int32_t* __restrict__ accepted_len,
                  const int32_t* __restrict__ path) {
    __shared__ rs::CompactSmem cm;
    const int b = blockIdx.x;
    const int32_t* pth = path + (int64_t)b * RS_MAX_TREE;
    rs::compact_sample(A, b, accepted_len[b], [&](int k) { return pth[k]; }, blockIdx.y, gridDim.y, blockIdx.y == 0,
                       cm);
}

}  // namespace

extern "C" rs_status rs_kv_compact(void* const* k_layers_host, void* const* v_layers_host, int32_t L,
                                   int64_t num_pages, int32_t Hkv, int32_t head_dim,
                                   int32_t page_size, const int32_t* block_table, int32_t max_pages,
                                   const int32_t* prefix_len, const int32_t* accepted_len,
                                   const int32_t* path, int32_t B, int32_t* new_len,
                                   int32_t* moves, void* stream) {
    rs::bind_device(block_table);
    (void)num_pages;
    RS_REQUIRE(B >= 0 && L >= 0 && Hkv > 0 && page_size > 0, RS_ERR_INVALID_ARG, "rs_kv_compact: bad sizes");
    RS_REQUIRE(head_dim % 8 == 0, RS_ERR_UNSUPPORTED, "rs_kv_compact: head_dim %% 8 != 0");
    if (B == 0) return RS_OK;
    RS_REQUIRE(k_layers_host && v_layers_host && block_table && prefix_len && accepted_len && path && new_len,
               RS_ERR_INVALID_ARG, "rs_kv_compact: null pointer");
    for (int l0 = 0; l0 < (L == 0 ? 1 : L); l0 += rs::kCompactMaxLayers) {
        const int nl = L == 0 ? 0 : (L - l0 < rs::kCompactMaxLayers ? L - l0 : rs::kCompactMaxLayers);
        rs::CompactArgs A;
        for (int i = 0; i < nl; ++i) {
            RS_REQUIRE(k_layers_host[l0 + i] && v_layers_host[l0 + i], RS_ERR_INVALID_ARG,
                       "rs_kv_compact: null layer pointer");
            A.k[i] = k_layers_host[l0 + i];
            A.v[i] = v_layers_host[l0 + i];
        }
        A.nl = nl;
        A.Hkv = Hkv;
        A.d = head_dim;
        A.ps = page_size;
        A.max_pages = max_pages;
        A.block_table = block_table;
        A.prefix_len = prefix_len;
        A.new_len = new_len;
        A.moves = l0 == 0 ? moves : nullptr;
        const int groups = nl > 0 ? (nl + kLayersPerCta - 1) / kLayersPerCta : 1;
        dim3 grid(B, groups);
        kv_compact_kernel<<<grid, kThreads, 0, rs::as_stream(stream)>>>(A, accepted_len, path);
        RS_LAUNCH_CHECK();
    }
    return RS_OK;
}
