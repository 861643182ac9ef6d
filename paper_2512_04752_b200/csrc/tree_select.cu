// f3: verification trees built on the GPU from the draft's candidate trees, for
// the n that select_strategy chose (readings Z1, Z6, Z9, Z11):
//   dl(u) = o(u) * dl(parent(u))               (Z9: the product includes u; -1 = virtual root)
//   w(u)  = F(dl(u))                           (F piecewise linear as np.interp, clamped [0, 1])
//   S(n)  = the first n pops of the layer-level search: at step m the nodes of depth m-1 enter
//           a max queue keyed (w desc, depth asc, id asc) and the max leaves it
//   tree  = root (the last committed token) + S(n) in ascending candidate index, parents
//           re-indexed (a root-level candidate hangs under node 0), ancestor masks and depths.
// One warp per sample; candidates staged in shared memory. dl is computed level by level in the
// same multiplication order as the definition (so the doubles are bit-identical to the host's);
// every double operation is an explicit round-to-nearest intrinsic (no contraction). The queue
// is a per-lane bitmask of available candidates (lane l holds candidates l, l+32, ...); a pop is a
// warp arg-max over (w, depth, id).
#include <cfloat>

#include "common.cuh"

namespace {

constexpr int kMaxCand = 256;
constexpr int kPerLane = kMaxCand / 32;
constexpr int kWarps = 4;
constexpr int kMaxKnots = 16;

struct WarpSmem {
    double dl[kMaxCand];
    double w[kMaxCand];
    int par[kMaxCand];
    int dep[kMaxCand];
    int pos[kMaxCand];             // position in the verification tree (0 = not selected)
    int vpar[RS_MAX_TREE];
    uint64_t vmask[RS_MAX_TREE];
};

__device__ __forceinline__ double acceptance_fit(double x, const double* kx, const double* ky, int nk) {
    double y;
    if (x <= kx[0]) {
        y = ky[0];
    } else if (x >= kx[nk - 1]) {
        y = ky[nk - 1];
    } else {
        int j = 0;                                          // largest j with kx[j] <= x
        while (j + 1 < nk && kx[j + 1] <= x) ++j;
        const double slope = __ddiv_rn(__dsub_rn(ky[j + 1], ky[j]), __dsub_rn(kx[j + 1], kx[j]));
        y = __dadd_rn(__dmul_rn(slope, __dsub_rn(x, kx[j])), ky[j]);
    }
    return y < 0.0 ? 0.0 : (y > 1.0 ? 1.0 : y);
}

// a better than b in the queue order (w desc, depth asc, id asc); id < 0 = empty
__device__ __forceinline__ bool better(double wa, int da, int ia, double wb, int db, int ib) {
    if (ib < 0) return ia >= 0;
    if (ia < 0) return false;
    if (wa != wb) return wa > wb;
    if (da != db) return da < db;
    return ia < ib;
}

__global__ void __launch_bounds__(32 * kWarps)
tree_select_kernel(const int32_t* __restrict__ cand_parent, const double* __restrict__ cand_o,
                   const int32_t* __restrict__ cand_token, const int32_t* __restrict__ cand_off,
                   const int32_t* __restrict__ root_token, int B, int n, const double* __restrict__ knots_x,
                   const double* __restrict__ knots_y, int nk, int32_t* __restrict__ parent_out,
                   int32_t* __restrict__ token_out, uint64_t* __restrict__ mask_out,
                   int32_t* __restrict__ depth_out, int32_t* __restrict__ flags_out) {
    __shared__ WarpSmem sms[kWarps];
    __shared__ double kx[kMaxKnots], ky[kMaxKnots];
    if (threadIdx.x < nk) { kx[threadIdx.x] = knots_x[threadIdx.x]; ky[threadIdx.x] = knots_y[threadIdx.x]; }
    __syncthreads();
    // F must be a monotone piecewise-linear fit: knots_x strictly increasing, knots_y
    // non-decreasing, all finite. Then w = F(dl) is non-increasing along every path (o <= 1), so
    // S(n) is closed under parents. Invalid knots flag every sample MALFORMED.
    bool knots_ok = true;
    for (int j = 0; j < nk; ++j) knots_ok = knots_ok && isfinite(kx[j]) && isfinite(ky[j]);
    for (int j = 0; j + 1 < nk; ++j) knots_ok = knots_ok && kx[j] < kx[j + 1] && ky[j] <= ky[j + 1];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * kWarps + wid;
    if (b >= B) return;
    WarpSmem& sm = sms[wid];
    const int off = cand_off[b];
    const int N = cand_off[b + 1] - off;
    const int T = n + 1;
    const int64_t ob = (int64_t)b * T;
    int flags = 0;
    bool ok = knots_ok && N >= 1 && N <= kMaxCand;
    // stage the candidates; check the tree (parent[i] in [-1, i)) and o(u) in [0, 1]
    bool bad = false;
    if (ok) {
        for (int i = lane; i < N; i += 32) {
            const int p = cand_parent[off + i];
            const double o = cand_o[off + i];
            sm.par[i] = p;
            sm.dl[i] = o;
            sm.pos[i] = 0;
            bad |= !(p >= -1 && p < i) || !(o >= 0.0 && o <= 1.0);
        }
    }
    ok = ok && !__any_sync(0xffffffffu, bad);
    __syncwarp();
    int maxdep = 0;
    if (ok && lane == 0) {
        for (int i = 0; i < N; ++i) {
            const int p = sm.par[i];
            const int d = p < 0 ? 0 : sm.dep[p] + 1;
            sm.dep[i] = d;
            maxdep = d > maxdep ? d : maxdep;
        }
    }
    maxdep = __shfl_sync(0xffffffffu, maxdep, 0);
    __syncwarp();
    int taken = 0;
    if (ok) {
        // dl level by level: o(u) * dl(parent) with the parent's dl final (one level up)
        for (int k = 1; k <= maxdep; ++k) {
            for (int i = lane; i < N; i += 32)
                if (sm.dep[i] == k) sm.dl[i] = __dmul_rn(sm.dl[i], sm.dl[sm.par[i]]);
            __syncwarp();
        }
        for (int i = lane; i < N; i += 32) sm.w[i] = acceptance_fit(sm.dl[i], kx, ky, nk);
        __syncwarp();
        // layer-level search
        uint32_t avail = 0;
        for (int m = 1; m <= n; ++m) {
#pragma unroll
            for (int j = 0; j < kPerLane; ++j) {
                const int i = lane + 32 * j;
                if (i < N && sm.dep[i] == m - 1) avail |= 1u << j;
            }
            double bw = -DBL_MAX;
            int bd = 0, bi = -1;
#pragma unroll
            for (int j = 0; j < kPerLane; ++j) {
                const int i = lane + 32 * j;
                if ((avail >> j) & 1u) {
                    const double wi = sm.w[i];
                    const int di = sm.dep[i];
                    if (better(wi, di, i, bw, bd, bi)) { bw = wi; bd = di; bi = i; }
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double w2 = __shfl_xor_sync(0xffffffffu, bw, o);
                const int d2 = __shfl_xor_sync(0xffffffffu, bd, o);
                const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
                if (better(w2, d2, i2, bw, bd, bi)) { bw = w2; bd = d2; bi = i2; }
            }
            if (bi < 0) break;                              // queue empty: fewer than n nodes
            if ((bi & 31) == lane) { avail &= ~(1u << (bi >> 5)); sm.pos[bi] = 1; }
            ++taken;
        }
        __syncwarp();
        if (taken < n) flags |= RS_FLAG_INSUFFICIENT;
        // positions: 1 + number of selected candidates with a lower index
        int base = 0;
        for (int c0 = 0; c0 < N; c0 += 32) {
            const int i = c0 + lane;
            const bool s = i < N && sm.pos[i] != 0;
            const uint32_t bal = __ballot_sync(0xffffffffu, s);
            if (s) sm.pos[i] = 1 + base + __popc(bal & ((1u << lane) - 1u));
            base += __popc(bal);
        }
        __syncwarp();
        bool orphan = false;   // a selected node whose parent was not selected (S(n) not closed)
        for (int i = lane; i < N; i += 32) {
            const int p = sm.pos[i];
            if (p) {
                const int cp = sm.par[i];
                const bool lost = cp >= 0 && sm.pos[cp] == 0;
                orphan |= lost;
                sm.vpar[p] = cp < 0 ? 0 : sm.pos[cp];
                parent_out[ob + p] = sm.vpar[p];
                token_out[ob + p] = lost ? -1 : cand_token[off + i];   // -1: rs_tree_accept flags it
                depth_out[ob + p] = sm.dep[i] + 1;
            }
        }
        if (__any_sync(0xffffffffu, orphan)) flags |= RS_FLAG_MALFORMED;
    } else {
        flags |= RS_FLAG_MALFORMED;
    }
    // padding nodes (flagged samples only): children of the root with token -1
    for (int p = taken + 1 + lane; p < T; p += 32) {
        sm.vpar[p] = 0;
        parent_out[ob + p] = 0;
        token_out[ob + p] = -1;
        depth_out[ob + p] = 1;
    }
    if (lane == 0) {
        sm.vpar[0] = -1;
        parent_out[ob] = -1;
        token_out[ob] = root_token[b];
        depth_out[ob] = 0;
        flags_out[b] = flags;
    }
    __syncwarp();
    if (lane == 0) {                                        // masks in topological order
        sm.vmask[0] = 1ull;
        for (int p = 1; p < T; ++p) sm.vmask[p] = sm.vmask[sm.vpar[p]] | (1ull << p);
    }
    __syncwarp();
    for (int p = lane; p < T; p += 32) mask_out[ob + p] = sm.vmask[p];
}

}  // namespace

extern "C" rs_status rs_tree_select(const int32_t* cand_parent, const double* cand_o, const int32_t* cand_token,
                                    const int32_t* cand_off, const int32_t* root_token, int32_t B, int32_t n,
                                    const double* knots_x, const double* knots_y, int32_t n_knots,
                                    int32_t* parent_out, int32_t* token_out, uint64_t* tree_mask_out,
                                    int32_t* depth_out, int32_t* status_flags, void* stream) {
    rs::bind_device(cand_parent);
    RS_REQUIRE(B >= 0, RS_ERR_INVALID_ARG, "rs_tree_select: B < 0");
    RS_REQUIRE(n >= 1 && n + 1 <= RS_MAX_TREE, RS_ERR_UNSUPPORTED, "rs_tree_select: n=%d outside [1, 63]", n);
    RS_REQUIRE(n_knots >= 2 && n_knots <= kMaxKnots, RS_ERR_INVALID_ARG, "rs_tree_select: %d knots", n_knots);
    if (B == 0) return RS_OK;
    RS_REQUIRE(cand_parent && cand_o && cand_token && cand_off && root_token && knots_x && knots_y && parent_out &&
                   token_out && tree_mask_out && depth_out && status_flags,
               RS_ERR_INVALID_ARG, "rs_tree_select: null pointer");
    tree_select_kernel<<<(B + kWarps - 1) / kWarps, 32 * kWarps, 0, rs::as_stream(stream)>>>(
        cand_parent, cand_o, cand_token, cand_off, root_token, B, n, knots_x, knots_y, n_knots, parent_out, token_out,
        tree_mask_out, depth_out, status_flags);
    RS_LAUNCH_CHECK();
    return RS_OK;
}
