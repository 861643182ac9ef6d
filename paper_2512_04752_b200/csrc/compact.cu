// a4: KV commit of the accepted path (Markov property; Z2).
//   for k = 1..a_b: K/V[b, P_b+k] <- K/V[b, P_b+path[k]]   (all layers, all kv heads)
// Sequential ascending-k semantics. Since path[k] >= k (node indices are topological and the
// node at depth k has index >= k), copy k never reads a slot written by an earlier copy; only a
// LATER copy can overwrite a slot an earlier one reads. So the rows are processed in chunks of
// ascending k, each chunk gathered into registers (all loads in flight) before it is scattered.
// One CTA per (sample, group of layers): the flattened row index runs k-major over
// (layer, K|V, head, 16-byte column), so one CTA moves every layer of its group at once with
// coalesced 128-bit loads/stores. Identity moves (path[k] == k) are skipped.
#include "common.cuh"

namespace {

constexpr int kMaxLayers = 256;
constexpr int kLayersPerCta = 8;
constexpr int kThreads = 256;
constexpr int kPerThread = 16;   // 16-byte registers per thread per chunk

struct LayerPtrs {
    void* k[kMaxLayers];
    void* v[kMaxLayers];
};

__global__ void __launch_bounds__(kThreads)
kv_compact_kernel(LayerPtrs layers, int nl, int Hkv, int d, int ps, const int32_t* __restrict__ block_table,
                  int max_pages, const int32_t* __restrict__ prefix_len, const int32_t* __restrict__ accepted_len,
                  const int32_t* __restrict__ path, int32_t* __restrict__ new_len, int32_t* __restrict__ moves) {
    const int b = blockIdx.x;
    const int l0 = blockIdx.y * kLayersPerCta;
    const int a = accepted_len[b];
    const int P = prefix_len[b];
    const int32_t* pth = path + (int64_t)b * RS_MAX_TREE;
    if (blockIdx.y == 0) {
        if (threadIdx.x == 0) new_len[b] = P + 1 + a;
        if (moves) {
            for (int k = threadIdx.x; k < RS_MAX_TREE; k += blockDim.x) {
                const int2 m = (k < a) ? make_int2(P + pth[k + 1], P + k + 1) : make_int2(-1, -1);
                reinterpret_cast<int2*>(moves)[(int64_t)b * RS_MAX_TREE + k] = m;
            }
        }
    }
    const int nlay = min(kLayersPerCta, nl - l0);
    if (a <= 0 || nlay <= 0) return;
    const int vec_per_row = d / 8;                        // 16-byte vectors per (token, head) row
    const int per_layer_kv = Hkv * vec_per_row;           // one token, one layer, one of K/V
    const int per_k = nlay * 2 * per_layer_kv;            // one accepted token, all layers of the group
    const int32_t* bt = block_table + (int64_t)b * max_pages;
    const int total = a * per_k;
    for (int e0 = 0; e0 < total; e0 += kThreads * kPerThread) {
        uint4 buf[kPerThread];
        uint4* dst[kPerThread];
#pragma unroll
        for (int r = 0; r < kPerThread; ++r) {
            const int e = e0 + threadIdx.x + r * kThreads;
            dst[r] = nullptr;
            if (e < total) {
                const int k = 1 + e / per_k;
                int rem = e % per_k;
                const int lay = rem / (2 * per_layer_kv);
                rem %= 2 * per_layer_kv;
                const int kv = rem / per_layer_kv;
                rem %= per_layer_kv;
                const int h = rem / vec_per_row, c = rem % vec_per_row;
                const int src = P + pth[k], dsts = P + k;
                if (src != dsts) {
                    uint4* cache = reinterpret_cast<uint4*>(kv ? layers.v[l0 + lay] : layers.k[l0 + lay]);
                    const int64_t so = (((int64_t)bt[src / ps] * Hkv + h) * ps + (src % ps)) * vec_per_row + c;
                    const int64_t dof = (((int64_t)bt[dsts / ps] * Hkv + h) * ps + (dsts % ps)) * vec_per_row + c;
                    buf[r] = cache[so];
                    dst[r] = cache + dof;
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kPerThread; ++r)
            if (dst[r]) *dst[r] = buf[r];
        __syncthreads();
    }
}

}  // namespace

extern "C" rs_status rs_kv_compact(void* const* k_layers_host, void* const* v_layers_host, int32_t L,
                                   int64_t num_pages, int32_t Hkv, int32_t head_dim,
                                   int32_t page_size, const int32_t* block_table, int32_t max_pages,
                                   const int32_t* prefix_len, const int32_t* accepted_len,
                                   const int32_t* path, int32_t B, int32_t* new_len,
                                   int32_t* moves, void* stream) {
    (void)num_pages;
    RS_REQUIRE(B >= 0 && L >= 0 && Hkv > 0 && page_size > 0, RS_ERR_INVALID_ARG, "rs_kv_compact: bad sizes");
    RS_REQUIRE(head_dim % 8 == 0, RS_ERR_UNSUPPORTED, "rs_kv_compact: head_dim %% 8 != 0");
    if (B == 0) return RS_OK;
    RS_REQUIRE(k_layers_host && v_layers_host && block_table && prefix_len && accepted_len && path && new_len,
               RS_ERR_INVALID_ARG, "rs_kv_compact: null pointer");
    for (int l0 = 0; l0 < (L == 0 ? 1 : L); l0 += kMaxLayers) {
        const int nl = L == 0 ? 0 : (L - l0 < kMaxLayers ? L - l0 : kMaxLayers);
        LayerPtrs lp;
        for (int i = 0; i < nl; ++i) {
            RS_REQUIRE(k_layers_host[l0 + i] && v_layers_host[l0 + i], RS_ERR_INVALID_ARG,
                       "rs_kv_compact: null layer pointer");
            lp.k[i] = k_layers_host[l0 + i];
            lp.v[i] = v_layers_host[l0 + i];
        }
        const int groups = nl > 0 ? (nl + kLayersPerCta - 1) / kLayersPerCta : 1;
        dim3 grid(B, groups);
        kv_compact_kernel<<<grid, kThreads, 0, rs::as_stream(stream)>>>(
            lp, nl, Hkv, head_dim, page_size, block_table, max_pages, prefix_len, accepted_len, path, new_len,
            l0 == 0 ? moves : nullptr);
        RS_LAUNCH_CHECK();
    }
    return RS_OK;
}
