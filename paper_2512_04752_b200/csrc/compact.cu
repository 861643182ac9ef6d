// a4: KV commit of the accepted path (Markov property; Z2).
//   for k = 1..a_b: K/V[b, P_b+k] <- K/V[b, P_b+path[k]]   (all layers, all kv heads)
// Sequential ascending-k semantics. Since path[k] >= k (node indices are topological and the
// node at depth k has index >= k), copy k never reads a slot written by an earlier copy; only a
// LATER copy can overwrite a slot an earlier one reads. So the rows are processed in chunks of
// ascending k, each chunk gathered into registers (all loads in flight) before it is scattered.
// The move list is built by two warps in parallel (ballot scan). One CTA per (sample, pair of layers); consecutive threads own consecutive 16-byte columns,
// so every gather/scatter is a coalesced 128-bit access. Identity moves (path[k] == k) are skipped.
#include "common.cuh"

namespace {

constexpr int kMaxLayers = 256;
constexpr int kLayersPerCta = 2;
constexpr int kThreads = 256;
constexpr int kLanesPerThread = 2;   // (layer, K|V, head, 16-byte column) lanes owned by a thread
constexpr int kChunk = 4;            // accepted tokens gathered per round

struct LayerPtrs {
    void* k[kMaxLayers];
    void* v[kMaxLayers];
};

// A "lane" = one 16-byte column of one (layer, K|V, kv head) row. Every copy of a lane is done
// by the thread that owns it, in ascending-k chunks, each chunk gathered into registers before it
// is scattered: that reproduces the sequential semantics without any block barrier (copies of
// different lanes never touch the same bytes).
__global__ void __launch_bounds__(kThreads)
kv_compact_kernel(LayerPtrs layers, int nl, int Hkv, int d, int ps, const int32_t* __restrict__ block_table,
                  int max_pages, const int32_t* __restrict__ prefix_len, const int32_t* __restrict__ accepted_len,
                  const int32_t* __restrict__ path, int32_t* __restrict__ new_len, int32_t* __restrict__ moves) {
    __shared__ int64_t s_src[RS_MAX_TREE], s_dst[RS_MAX_TREE];   // token row offsets (16-byte units, head 0)
    __shared__ int s_n;
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
    const int vpr = d / 8;                                  // 16-byte vectors per (token, head) row
    const int32_t* bt = block_table + (int64_t)b * max_pages;
    // move list in parallel: thread t < 64 takes k = t + 1; the non-identity moves are packed
    // in ascending k by a two-warp ballot scan (the order the sequential semantics need)
    {
        const int t = threadIdx.x;
        bool mv = false;
        int64_t so = 0, dso = 0;
        if (t < RS_MAX_TREE && t + 1 <= a) {
            const int src = P + pth[t + 1], dst = P + t + 1;
            mv = src != dst;                                // identity moves are skipped
            if (mv) {
                so = ((int64_t)bt[src / ps] * Hkv * ps + (src % ps)) * vpr;
                dso = ((int64_t)bt[dst / ps] * Hkv * ps + (dst % ps)) * vpr;
            }
        }
        __shared__ int s_cnt[2];
        const unsigned bal = __ballot_sync(0xffffffffu, mv);
        const int lane = t & 31;
        if (t == 0 || t == 32) s_cnt[t >> 5] = __popc(bal);
        __syncthreads();
        if (mv) {
            const int pos = __popc(bal & ((1u << lane) - 1u)) + (t >= 32 ? s_cnt[0] : 0);
            s_src[pos] = so;
            s_dst[pos] = dso;
        }
        if (t == 0) s_n = s_cnt[0] + s_cnt[1];
    }
    __syncthreads();
    const int n = s_n;
    if (n == 0) return;
    const int lanes_per_layer = 2 * Hkv * vpr;
    const int lanes = nlay * lanes_per_layer;
    for (int lb = 0; lb < lanes; lb += kThreads * kLanesPerThread) {
        uint4* base[kLanesPerThread];
        int64_t loff[kLanesPerThread];
#pragma unroll
        for (int i = 0; i < kLanesPerThread; ++i) {
            const int q = lb + threadIdx.x + i * kThreads;
            base[i] = nullptr;
            loff[i] = 0;
            if (q < lanes) {
                const int lay = q / lanes_per_layer;
                int rem = q - lay * lanes_per_layer;
                const int kv = rem / (Hkv * vpr);
                rem -= kv * (Hkv * vpr);
                const int h = rem / vpr, c = rem - h * vpr;
                base[i] = reinterpret_cast<uint4*>(kv ? layers.v[l0 + lay] : layers.k[l0 + lay]);
                loff[i] = (int64_t)h * ps * vpr + c;
            }
        }
        for (int k0 = 0; k0 < n; k0 += kChunk) {
            uint4 buf[kLanesPerThread][kChunk];
#pragma unroll
            for (int i = 0; i < kLanesPerThread; ++i)
#pragma unroll
                for (int j = 0; j < kChunk; ++j)
                    if (base[i] && k0 + j < n) buf[i][j] = base[i][s_src[k0 + j] + loff[i]];
#pragma unroll
            for (int i = 0; i < kLanesPerThread; ++i)
#pragma unroll
                for (int j = 0; j < kChunk; ++j)
                    if (base[i] && k0 + j < n) base[i][s_dst[k0 + j] + loff[i]] = buf[i][j];
        }
    }
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
