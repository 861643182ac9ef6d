// a4: KV commit of the accepted path (Markov property; Z2).
//   for k = 1..a_b: K/V[b, P_b+k] <- K/V[b, P_b+path[k]]   (all layers, all kv heads)
// Sequential ascending-k semantics. Since path[k] >= k (node indices are topological and the
// node at depth k has index >= k), copy k never reads a slot written by an earlier copy;
// only a LATER copy can overwrite a slot an earlier one reads. So each CTA gathers a chunk
// of consecutive k into registers, syncs, then scatters; chunks run in ascending k.
// One CTA per (sample, layer, K|V); 128-bit coalesced loads/stores over the head_dim rows.
#include "common.cuh"

namespace {

constexpr int kMaxLayers = 256;
constexpr int kThreads = 256;
constexpr int kPerThread = 4;   // uint4 registers per thread per chunk

struct LayerPtrs {
    void* k[kMaxLayers];
    void* v[kMaxLayers];
};

__global__ void __launch_bounds__(kThreads)
kv_compact_kernel(LayerPtrs layers, int nl, int Hkv, int d, int ps, const int32_t* __restrict__ block_table,
                  int max_pages, const int32_t* __restrict__ prefix_len,
                  const int32_t* __restrict__ accepted_len, const int32_t* __restrict__ path,
                  int32_t* __restrict__ new_len, int32_t* __restrict__ moves) {
    const int b = blockIdx.x;
    const int layer = blockIdx.y;
    const int kv = blockIdx.z;
    const int a = accepted_len[b];
    const int P = prefix_len[b];
    const int32_t* pth = path + (int64_t)b * RS_MAX_TREE;
    if (layer == 0 && kv == 0) {
        if (threadIdx.x == 0) new_len[b] = P + 1 + a;
        if (moves) {
            for (int k = threadIdx.x; k < RS_MAX_TREE; k += blockDim.x) {
                int2 m = (k < a) ? make_int2(P + pth[k + 1], P + k + 1) : make_int2(-1, -1);
                reinterpret_cast<int2*>(moves)[(int64_t)b * RS_MAX_TREE + k] = m;
            }
        }
    }
    if (a <= 0 || nl == 0) return;
    uint4* cache = reinterpret_cast<uint4*>(kv ? layers.v[layer] : layers.k[layer]);
    const int vec_per_row = d / 8;                     // uint4 per (token, head) row
    const int vec_per_tok = Hkv * vec_per_row;         // all heads of one token
    const int32_t* bt = block_table + (int64_t)b * max_pages;
    const int chunk_rows = max(1, (kThreads * kPerThread) / vec_per_tok);
    for (int k0 = 1; k0 <= a; k0 += chunk_rows) {
        const int k1 = min(a, k0 + chunk_rows - 1);
        const int nvec = (k1 - k0 + 1) * vec_per_tok;
        uint4 buf[kPerThread];
        int64_t dst_off[kPerThread];
#pragma unroll
        for (int r = 0; r < kPerThread; ++r) {
            int e = threadIdx.x + r * kThreads;
            dst_off[r] = -1;
            if (e < nvec) {
                int k = k0 + e / vec_per_tok;
                int rem = e % vec_per_tok;
                int h = rem / vec_per_row, c = rem % vec_per_row;
                int src = P + pth[k], dst = P + k;
                if (src != dst) {
                    int64_t so = (((int64_t)bt[src / ps] * Hkv + h) * ps + (src % ps)) * vec_per_row + c;
                    dst_off[r] = (((int64_t)bt[dst / ps] * Hkv + h) * ps + (dst % ps)) * vec_per_row + c;
                    buf[r] = cache[so];
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < kPerThread; ++r)
            if (dst_off[r] >= 0) cache[dst_off[r]] = buf[r];
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
    RS_REQUIRE(B >= 0 && L >= 0 && Hkv > 0 && page_size > 0, RS_ERR_INVALID_ARG,
               "rs_kv_compact: bad sizes");
    RS_REQUIRE(head_dim % 8 == 0, RS_ERR_UNSUPPORTED, "rs_kv_compact: head_dim %% 8 != 0");
    RS_REQUIRE(Hkv * head_dim / 8 <= kThreads * kPerThread, RS_ERR_UNSUPPORTED,
               "rs_kv_compact: Hkv*head_dim too large");
    if (B == 0) return RS_OK;
    RS_REQUIRE(k_layers_host && v_layers_host && block_table && prefix_len && accepted_len && path &&
                   new_len,
               RS_ERR_INVALID_ARG, "rs_kv_compact: null pointer");
    for (int l0 = 0; l0 < (L == 0 ? 1 : L); l0 += kMaxLayers) {
        int nl = L == 0 ? 0 : (L - l0 < kMaxLayers ? L - l0 : kMaxLayers);
        LayerPtrs lp;
        for (int i = 0; i < nl; ++i) {
            RS_REQUIRE(k_layers_host[l0 + i] && v_layers_host[l0 + i], RS_ERR_INVALID_ARG,
                       "rs_kv_compact: null layer pointer");
            lp.k[i] = k_layers_host[l0 + i];
            lp.v[i] = v_layers_host[l0 + i];
        }
        dim3 grid(B, nl > 0 ? nl : 1, nl > 0 ? 2 : 1);
        kv_compact_kernel<<<grid, kThreads, 0, rs::as_stream(stream)>>>(
            lp, nl, Hkv, head_dim, page_size, block_table, max_pages, prefix_len, accepted_len,
            path, new_len, l0 == 0 ? moves : nullptr);
        RS_LAUNCH_CHECK();
    }
    return RS_OK;
}
