// a1: ancestor-or-self bitmask + depth per tree node (reading Z1/Z3).
// One warp per sample: the lanes stage the <= 64 parent indices in shared memory (coalesced),
// lane 0 walks them in topological order (mask[i] = mask[parent[i]] | 1 << i,
// depth[i] = depth[parent[i]] + 1) on shared memory, and the lanes write the results back.
#include "common.cuh"

namespace {

constexpr int kWarpsPerBlock = 4;

__global__ void __launch_bounds__(32 * kWarpsPerBlock)
tree_mask_kernel(const int32_t* __restrict__ parent, const int32_t* __restrict__ tree_off, int B,
                 uint64_t* __restrict__ mask, int32_t* __restrict__ depth, int32_t* __restrict__ flags) {
    __shared__ int par[kWarpsPerBlock][RS_MAX_TREE];
    __shared__ uint64_t msk[kWarpsPerBlock][RS_MAX_TREE];
    __shared__ int dep[kWarpsPerBlock][RS_MAX_TREE];
    __shared__ int okf[kWarpsPerBlock];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * kWarpsPerBlock + w;
    if (b >= B) return;
    const int off = tree_off[b];
    const int T = tree_off[b + 1] - off;
    const bool size_ok = T >= 1 && T <= RS_MAX_TREE;
    if (size_ok) {
        if (lane < T) par[w][lane] = parent[off + lane];
        if (lane + 32 < T) par[w][lane + 32] = parent[off + lane + 32];
    }
    __syncwarp();
    if (lane == 0) {
        bool ok = size_ok && par[w][0] == -1;
        if (ok) {
            msk[w][0] = 1ull;
            dep[w][0] = 0;
            for (int i = 1; i < T; ++i) {
                const int p = par[w][i];
                if (p < 0 || p >= i) { ok = false; break; }
                msk[w][i] = msk[w][p] | (1ull << i);
                dep[w][i] = dep[w][p] + 1;
            }
        }
        okf[w] = ok;
    }
    __syncwarp();
    const bool ok = okf[w] != 0;
    if (T > 0) {
        for (int i = lane; i < T; i += 32) {
            mask[off + i] = ok ? msk[w][i] : 0ull;
            depth[off + i] = ok ? dep[w][i] : 0;
        }
    }
    if (lane == 0 && flags) flags[b] = ok ? 0 : RS_FLAG_MALFORMED;
}

}  // namespace

extern "C" rs_status rs_tree_build_mask(const int32_t* parent, const int32_t* tree_off, int32_t B,
                                        uint64_t* tree_mask, int32_t* depth, int32_t* status_flags,
                                        void* stream) {
    rs::bind_device(parent);
    RS_REQUIRE(B >= 0, RS_ERR_INVALID_ARG, "rs_tree_build_mask: B < 0");
    if (B == 0) return RS_OK;
    RS_REQUIRE(parent && tree_off && tree_mask && depth, RS_ERR_INVALID_ARG,
               "rs_tree_build_mask: null pointer");
    tree_mask_kernel<<<(B + kWarpsPerBlock - 1) / kWarpsPerBlock, 32 * kWarpsPerBlock, 0, rs::as_stream(stream)>>>(
        parent, tree_off, B, tree_mask, depth, status_flags);
    RS_LAUNCH_CHECK();
    return RS_OK;
}
