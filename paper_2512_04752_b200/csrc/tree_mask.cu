// a1: ancestor-or-self bitmask + depth per tree node (reading Z1/Z3).
// One thread per sample walks its <= 64 nodes in topological order:
//   mask[i] = mask[parent[i]] | (1 << i),  depth[i] = depth[parent[i]] + 1.
#include "common.cuh"

namespace {

__global__ void tree_mask_kernel(const int32_t* __restrict__ parent,
                                 const int32_t* __restrict__ tree_off, int B,
                                 uint64_t* __restrict__ mask, int32_t* __restrict__ depth,
                                 int32_t* __restrict__ flags) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    int off = tree_off[b];
    int T = tree_off[b + 1] - off;
    bool ok = (T >= 1 && T <= RS_MAX_TREE && parent[off] == -1);
    uint64_t m[RS_MAX_TREE];
    int dep[RS_MAX_TREE];
    if (ok) {
        m[0] = 1ull;
        dep[0] = 0;
        for (int i = 1; i < T; ++i) {
            int p = parent[off + i];
            if (p < 0 || p >= i) { ok = false; break; }
            m[i] = m[p] | (1ull << i);
            dep[i] = dep[p] + 1;
        }
    }
    int n = (T > 0) ? T : 0;
    for (int i = 0; i < n; ++i) {
        mask[off + i] = ok ? m[i] : 0ull;
        depth[off + i] = ok ? dep[i] : 0;
    }
    if (flags) flags[b] = ok ? 0 : RS_FLAG_MALFORMED;
}

}  // namespace

extern "C" rs_status rs_tree_build_mask(const int32_t* parent, const int32_t* tree_off, int32_t B,
                                        uint64_t* tree_mask, int32_t* depth,
                                        int32_t* status_flags, void* stream) {
    RS_REQUIRE(B >= 0, RS_ERR_INVALID_ARG, "rs_tree_build_mask: B < 0");
    if (B == 0) return RS_OK;
    RS_REQUIRE(parent && tree_off && tree_mask && depth, RS_ERR_INVALID_ARG,
               "rs_tree_build_mask: null pointer");
    int threads = 128;
    tree_mask_kernel<<<(B + threads - 1) / threads, threads, 0, rs::as_stream(stream)>>>(
        parent, tree_off, B, tree_mask, depth, status_flags);
    RS_LAUNCH_CHECK();
    return RS_OK;
}
