// a4 device side: the KV commit of ONE sample's accepted path (Markov property;
// DESIGN.md Z2), shared by kv_compact_kernel (a CTA per (sample, group of layers)) and by the
// fused acceptance kernels (the CTAs of the sample's cluster, right after its walk).
//   for k = 1..a_b: K/V[b, P_b+k] <- K/V[b, P_b+path[k]]   (all layers, all kv heads)
// Sequential ascending-k semantics. Since path[k] >= k (node indices are topological and the
// node at depth k has index >= k), copy k never reads a slot written by an earlier copy; only a
// LATER copy can overwrite a slot an earlier one reads. So the rows are processed in chunks of
// ascending k, each chunk gathered into registers (all loads in flight) before it is scattered.
// A "lane" = one 16-byte column of one (layer, K|V, kv head) row; every copy of a lane is done by
// the thread that owns it, so no barrier is needed between chunks (copies of different lanes
// never touch the same bytes). The move list (non-identity moves in ascending k) is built by two
// warps with a ballot scan.
#pragma once

#include "common.cuh"

namespace rs {

constexpr int kCompactMaxLayers = 256;

struct CompactArgs {                    // kernel parameter (by value)
    static constexpr bool kOn = true;
    void* k[kCompactMaxLayers];
    void* v[kCompactMaxLayers];
    int nl, Hkv, d, ps, max_pages;
    const int32_t* block_table;         // [B, max_pages]
    const int32_t* prefix_len;          // [B]
    int32_t* new_len;                   // [B] out
    int32_t* moves;                     // [B, RS_MAX_TREE, 2] out or nullptr
};
struct NoCompact {                      // acceptance without the fused commit
    static constexpr bool kOn = false;
};

struct CompactSmem {
    int64_t src[RS_MAX_TREE], dst[RS_MAX_TREE];   // token row offsets (16-byte units, head 0)
    int cnt[2];
    int n;
};

// Commit sample b's path (path_of(k) = path[k], k = 1..a) for the lanes of part `part` of
// `nparts` (contiguous equal shares of the nl x 2 x Hkv x d/8 lanes). write_meta: this CTA also
// writes new_len[b] and the moves row. Every thread of the CTA calls it (it holds CTA barriers;
// all its early returns are uniform). blockDim.x >= 64.
template <int kLanesPerThread = 2, int kChunk = 4, typename PathFn>
__device__ __forceinline__ void compact_sample(const CompactArgs& A, int b, int a, PathFn path_of, int part,
                                               int nparts, bool write_meta, CompactSmem& cm) {
    const int P = A.prefix_len[b];
    if (write_meta) {
        if (threadIdx.x == 0) A.new_len[b] = P + 1 + a;
        if (A.moves) {
            for (int k = threadIdx.x; k < RS_MAX_TREE; k += blockDim.x) {
                const int2 m = (k < a) ? make_int2(P + path_of(k + 1), P + k + 1) : make_int2(-1, -1);
                reinterpret_cast<int2*>(A.moves)[(int64_t)b * RS_MAX_TREE + k] = m;
            }
        }
    }
    const int vpr = A.d / 8;                                  // 16-byte vectors per (token, head) row
    const int lanes_per_layer = 2 * A.Hkv * vpr;
    const int total = A.nl * lanes_per_layer;
    const int share = (total + nparts - 1) / nparts;
    const int lo = min(total, part * share), hi = min(total, lo + share);
    if (a <= 0 || lo >= hi) return;
    const int32_t* bt = A.block_table + (int64_t)b * A.max_pages;
    {
        const int t = threadIdx.x;
        bool mv = false;
        int64_t so = 0, dso = 0;
        if (t < RS_MAX_TREE && t + 1 <= a) {
            const int src = P + path_of(t + 1), dst = P + t + 1;
            mv = src != dst;                                // identity moves are skipped
            if (mv) {
                so = ((int64_t)bt[src / A.ps] * A.Hkv * A.ps + (src % A.ps)) * vpr;
                dso = ((int64_t)bt[dst / A.ps] * A.Hkv * A.ps + (dst % A.ps)) * vpr;
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, mv);
        const int lane = t & 31;
        if (t == 0 || t == 32) cm.cnt[t >> 5] = __popc(bal);
        __syncthreads();
        if (mv) {
            const int pos = __popc(bal & ((1u << lane) - 1u)) + (t >= 32 ? cm.cnt[0] : 0);
            cm.src[pos] = so;
            cm.dst[pos] = dso;
        }
        if (t == 0) cm.n = cm.cnt[0] + cm.cnt[1];
    }
    __syncthreads();
    const int n = cm.n;
    if (n > 0) {
        for (int lb = lo; lb < hi; lb += (int)blockDim.x * kLanesPerThread) {
            uint4* base[kLanesPerThread];
            int64_t loff[kLanesPerThread];
#pragma unroll
            for (int i = 0; i < kLanesPerThread; ++i) {
                const int q = lb + (int)threadIdx.x + i * (int)blockDim.x;
                base[i] = nullptr;
                loff[i] = 0;
                if (q < hi) {
                    const int lay = q / lanes_per_layer;
                    int rem = q - lay * lanes_per_layer;
                    const int kv = rem / (A.Hkv * vpr);
                    rem -= kv * (A.Hkv * vpr);
                    const int h = rem / vpr, c = rem - h * vpr;
                    base[i] = reinterpret_cast<uint4*>(kv ? A.v[lay] : A.k[lay]);
                    loff[i] = (int64_t)h * A.ps * vpr + c;
                }
            }
            for (int k0 = 0; k0 < n; k0 += kChunk) {
                uint4 buf[kLanesPerThread][kChunk];
#pragma unroll
                for (int i = 0; i < kLanesPerThread; ++i)
#pragma unroll
                    for (int j = 0; j < kChunk; ++j)
                        if (base[i] && k0 + j < n) buf[i][j] = base[i][cm.src[k0 + j] + loff[i]];
#pragma unroll
                for (int i = 0; i < kLanesPerThread; ++i)
#pragma unroll
                    for (int j = 0; j < kChunk; ++j)
                        if (base[i] && k0 + j < n) base[i][cm.dst[k0 + j] + loff[i]] = buf[i][j];
            }
        }
    }
    __syncthreads();   // cm is reusable after this
}

}  // namespace rs
