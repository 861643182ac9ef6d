// a3: tree acceptance (readings Z5-Z8, Z15, "Bit-exact sampling").
//
// One CTA per sample walks its tree from the root. Only the rows of the nodes on the walk
// are read (the algorithmic bytes are the visited rows): at node c the CTA
// streams row c of the target logits (and, for MSS, the draft row) with 128-bit loads,
// reduces with warp shuffles + shared memory, decides the child in one thread and moves on.
//   GREEDY: block argmax (ties -> lowest id); accept the lowest-index child whose token
//           equals it; bonus = argmax at the last node.
//   DELTA / MSS: integer weights w_v (exp_spec), Philox uniforms, 128-bit exact tests; the
//           residual after a rejection is kept implicitly (DELTA: excluded-token list; MSS:
//           the chain of (Z, shift) scalars, re-applied per element when the row is re-read).
#include "common.cuh"
#include "sampling.cuh"

namespace {

using rs::u128;
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxTiles = 512;          // inverse-CDF tiles of kThreads*8 elements (V <= 2M)
constexpr int kMaxChain = RS_MAX_TREE;  // residual steps per node (<= children)

struct RowView {
    const void* base;
    int64_t row;
    int V;
    int dtype;      // RS_DTYPE_BF16 | RS_DTYPE_F32
    bool vec_ok;    // 16-byte aligned rows with V a multiple of the vector width
};

// Elements 8*i .. 8*i+7 of the row; n = number valid (elements past V are not touched).
__device__ __forceinline__ int load8(const RowView& rv, int i, float (&x)[8]) {
    int v0 = i * 8;
    int n = min(8, rv.V - v0);
    if (rv.dtype == RS_DTYPE_BF16) {
        const uint16_t* p = reinterpret_cast<const uint16_t*>(rv.base) + rv.row * (int64_t)rv.V + v0;
        if (rv.vec_ok && n == 8) {
            uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
            uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                x[2 * j] = __uint_as_float(w[j] << 16);
                x[2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = (j < n) ? rs::bf16_bits_to_f32(__ldg(p + j)) : 0.0f;
        }
    } else {
        const float* p = reinterpret_cast<const float*>(rv.base) + rv.row * (int64_t)rv.V + v0;
        if (rv.vec_ok && n == 8) {
            float4 a = __ldg(reinterpret_cast<const float4*>(p));
            float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
            x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
            x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = (j < n) ? __ldg(p + j) : 0.0f;
        }
    }
    return n;
}

struct Smem {
    float f[kWarps];
    int idx[kWarps];
    unsigned long long u[kWarps];
    unsigned long long uhi[kWarps];
    int flag;
    unsigned long long tile_sum[kMaxTiles];
    unsigned long long scan[kWarps];
    // per-sample state
    int parent[RS_MAX_TREE];
    int token[RS_MAX_TREE];
    int excluded[RS_MAX_TREE];
    int n_excluded;
    unsigned long long chainZ[kMaxChain];
    int chainS[kMaxChain];
    int n_chain;
    int bcast_i;
    unsigned long long bcast_u;
    int bonus_v;
};

__device__ __forceinline__ float block_max_f(float v, bool bad, Smem& sm, bool* any_bad) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    unsigned b = __ballot_sync(0xffffffffu, bad);
    __syncthreads();
    if (lane == 0) { sm.f[w] = v; sm.idx[w] = b ? 1 : 0; }
    __syncthreads();
    float r = sm.f[0];
    int anyb = sm.idx[0];
    for (int i = 1; i < kWarps; ++i) { r = fmaxf(r, sm.f[i]); anyb |= sm.idx[i]; }
    *any_bad = anyb != 0;
    return r;
}

// (value, index) argmax with lowest index on ties.
__device__ __forceinline__ void argmax_merge(float& v, int& i, float v2, int i2) {
    if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

__device__ __forceinline__ int block_argmax(float v, int i, bool bad, Smem& sm, bool* any_bad) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        float v2 = __shfl_xor_sync(0xffffffffu, v, o);
        int i2 = __shfl_xor_sync(0xffffffffu, i, o);
        argmax_merge(v, i, v2, i2);
    }
    unsigned b = __ballot_sync(0xffffffffu, bad);
    __syncthreads();
    if (lane == 0) { sm.f[w] = v; sm.idx[w] = i; sm.u[w] = b ? 1ull : 0ull; }
    __syncthreads();
    float rv = sm.f[0];
    int ri = sm.idx[0];
    unsigned long long anyb = sm.u[0];
    for (int k = 1; k < kWarps; ++k) { argmax_merge(rv, ri, sm.f[k], sm.idx[k]); anyb |= sm.u[k]; }
    *any_bad = anyb != 0;
    return ri;
}

__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v, Smem& sm) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) sm.u[w] = v;
    __syncthreads();
    unsigned long long r = 0;
    for (int k = 0; k < kWarps; ++k) r += sm.u[k];
    return r;
}

__device__ __forceinline__ u128 block_max_u128(u128 v, Smem& sm) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        unsigned long long hi = __shfl_xor_sync(0xffffffffu, (unsigned long long)(v >> 64), o);
        unsigned long long lo = __shfl_xor_sync(0xffffffffu, (unsigned long long)v, o);
        u128 v2 = ((u128)hi << 64) | lo;
        if (v2 > v) v = v2;
    }
    __syncthreads();
    if (lane == 0) { sm.uhi[w] = (unsigned long long)(v >> 64); sm.u[w] = (unsigned long long)v; }
    __syncthreads();
    u128 r = 0;
    for (int k = 0; k < kWarps; ++k) {
        u128 x = ((u128)sm.uhi[k] << 64) | sm.u[k];
        if (x > r) r = x;
    }
    return r;
}

// Current residual weight of a token from its base weight: DELTA zeroes excluded tokens;
// MSS re-applies the recorded residual steps w <- max(w*Zq - qw*Z_j, 0) >> s_j.
__device__ __forceinline__ uint64_t residual_weight(int mode, uint64_t w, uint64_t qw, int tok,
                                                    uint64_t Zq, const Smem& sm) {
    if (mode == RS_ACCEPT_SAMPLE_DELTA) {
        for (int e = 0; e < sm.n_excluded; ++e)
            if (sm.excluded[e] == tok) return 0;
        return w;
    }
    for (int j = 0; j < sm.n_chain; ++j) {
        u128 lhs = (u128)w * Zq, rhs = (u128)qw * sm.chainZ[j];
        u128 r = lhs > rhs ? lhs - rhs : 0;
        w = (uint64_t)(r >> sm.chainS[j]);
    }
    return w;
}

__global__ void __launch_bounds__(kThreads)
tree_accept_kernel(int mode, const void* __restrict__ logits, int dtype,
                   const float* __restrict__ draft, const int32_t* __restrict__ parent,
                   const int32_t* __restrict__ token, const int32_t* __restrict__ tree_off,
                   const int64_t* __restrict__ gid, int V, float inv_tau, uint64_t seed,
                   uint64_t step, int32_t* __restrict__ acc_out, int32_t* __restrict__ path_out,
                   int32_t* __restrict__ bonus_out, int32_t* __restrict__ flags_out,
                   bool logits_vec_ok, bool draft_vec_ok) {
    __shared__ Smem sm;
    const int b = blockIdx.x;
    const int tid = threadIdx.x;
    const int off = tree_off[b];
    const int T = tree_off[b + 1] - off;
    int32_t* pth = path_out + (int64_t)b * RS_MAX_TREE;
    if (tid < RS_MAX_TREE) pth[tid] = -1;
    if (tid == 0) {
        bool ok = (T >= 1 && T <= RS_MAX_TREE);
        if (ok) ok = parent[off] == -1;
        for (int i = 1; ok && i < T; ++i) {
            int p = parent[off + i];
            ok = (p >= 0 && p < i);
        }
        sm.flag = ok ? 0 : RS_FLAG_MALFORMED;
    }
    __syncthreads();
    if (sm.flag) {
        if (tid == 0) { acc_out[b] = 0; bonus_out[b] = -1; flags_out[b] = RS_FLAG_MALFORMED; }
        return;
    }
    if (tid < T) { sm.parent[tid] = parent[off + tid]; sm.token[tid] = token[off + tid]; }
    const int64_t g = gid[b];
    const int nvec = (V + 7) / 8;
    int c = 0, a = 0, bonus = -1, flags = 0;
    if (tid == 0) pth[0] = 0;
    __syncthreads();

    for (;;) {
        RowView lv{logits, (int64_t)(off + c), V, dtype, logits_vec_ok};
        int next = -1;
        bool stop = false;
        if (mode == RS_ACCEPT_GREEDY) {
            float best = -INFINITY;
            int bi = 0x7fffffff;
            bool bad = false;
            for (int i = tid; i < nvec; i += kThreads) {
                float x[8];
                int n = load8(lv, i, x);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (j < n) {
                        bad |= !isfinite(x[j]);
                        argmax_merge(best, bi, x[j], i * 8 + j);
                    }
                }
            }
            bool any_bad;
            int am = block_argmax(best, bi, bad, sm, &any_bad);
            if (any_bad) { flags |= RS_FLAG_NONFINITE; break; }
            for (int x = c + 1; x < T; ++x)
                if (sm.parent[x] == c && sm.token[x] == am) { next = x; break; }
            if (next < 0) { bonus = am; stop = true; }
        } else {
            // pass 1: row max (+ non-finite check)
            float mx = -INFINITY;
            bool bad = false;
            for (int i = tid; i < nvec; i += kThreads) {
                float x[8];
                int n = load8(lv, i, x);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < n) { bad |= !isfinite(x[j]); mx = fmaxf(mx, x[j]); }
            }
            bool any_bad;
            const float m = block_max_f(mx, bad, sm, &any_bad);
            if (any_bad) { flags |= RS_FLAG_NONFINITE; break; }
            // pass 2: Z = sum w, Zq = sum qw
            RowView qv{draft, (int64_t)(off + c), V, RS_DTYPE_F32, draft_vec_ok};
            unsigned long long zs = 0, zq = 0;
            for (int i = tid; i < nvec; i += kThreads) {
                float x[8];
                int n = load8(lv, i, x);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (j < n) zs += rs::target_weight(x[j], m, inv_tau);
                if (mode == RS_ACCEPT_SAMPLE_MSS) {
                    float q[8];
                    load8(qv, i, q);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (j < n) zq += rs::draft_weight(q[j]);
                }
            }
            uint64_t Z = block_sum_u64(zs, sm);
            const uint64_t Zq = (mode == RS_ACCEPT_SAMPLE_MSS) ? block_sum_u64(zq, sm) : 0ull;
            if (tid == 0) { sm.n_excluded = 0; sm.n_chain = 0; }
            __syncthreads();
            int rank = 0;
            for (int x = c + 1; x < T && next < 0; ++x) {
                if (sm.parent[x] != c) continue;
                const int tk = sm.token[x];
                if (tid == 0) {
                    const int64_t ro = (int64_t)(off + c) * V + tk;
                    float l = (dtype == RS_DTYPE_BF16)
                                  ? rs::bf16_bits_to_f32(reinterpret_cast<const uint16_t*>(logits)[ro])
                                  : reinterpret_cast<const float*>(logits)[ro];
                    uint64_t qw = (mode == RS_ACCEPT_SAMPLE_MSS) ? rs::draft_weight(draft[ro]) : 0ull;
                    uint64_t wt = residual_weight(mode, rs::target_weight(l, m, inv_tau), qw, tk, Zq, sm);
                    uint32_t U = rs::uniform_word(seed, step, g, (uint32_t)rank, (uint32_t)c);
                    bool acc;
                    if (mode == RS_ACCEPT_SAMPLE_DELTA)
                        acc = ((u128)U * Z) < ((u128)wt << 32);
                    else if (qw == 0)
                        acc = wt > 0;
                    else
                        acc = ((u128)U * ((u128)qw * Z)) < (((u128)wt * Zq) << 32);
                    sm.bcast_i = acc ? 1 : 0;
                    sm.bcast_u = wt;
                }
                __syncthreads();
                const bool accepted = sm.bcast_i != 0;
                const uint64_t wt = sm.bcast_u;
                __syncthreads();
                if (accepted) { next = x; break; }
                ++rank;
                if (mode == RS_ACCEPT_SAMPLE_DELTA) {
                    Z -= wt;
                    if (tid == 0) sm.excluded[sm.n_excluded++] = tk;
                    __syncthreads();
                } else {
                    // residual r_v = max(w_v*Zq - qw_v*Z, 0): max, then shifted sum
                    u128 rmax = 0;
                    for (int i = tid; i < nvec; i += kThreads) {
                        float x8[8], q8[8];
                        int n = load8(lv, i, x8);
                        load8(qv, i, q8);
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            if (j < n) {
                                uint64_t qw = rs::draft_weight(q8[j]);
                                uint64_t w = residual_weight(mode, rs::target_weight(x8[j], m, inv_tau),
                                                             qw, 0, Zq, sm);
                                u128 lhs = (u128)w * Zq, rhs = (u128)qw * Z;
                                u128 r = lhs > rhs ? lhs - rhs : 0;
                                if (r > rmax) rmax = r;
                            }
                        }
                    }
                    u128 mxr = block_max_u128(rmax, sm);
                    int s = rs::bitlen128(mxr) - 32;
                    if (s < 0) s = 0;
                    unsigned long long zn = 0;
                    for (int i = tid; i < nvec; i += kThreads) {
                        float x8[8], q8[8];
                        int n = load8(lv, i, x8);
                        load8(qv, i, q8);
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            if (j < n) {
                                uint64_t qw = rs::draft_weight(q8[j]);
                                uint64_t w = residual_weight(mode, rs::target_weight(x8[j], m, inv_tau),
                                                             qw, 0, Zq, sm);
                                u128 lhs = (u128)w * Zq, rhs = (u128)qw * Z;
                                u128 r = lhs > rhs ? lhs - rhs : 0;
                                zn += (unsigned long long)(r >> s);
                            }
                        }
                    }
                    uint64_t Znew = block_sum_u64(zn, sm);
                    __syncthreads();
                    if (Znew != 0) {      // an all-zero residual keeps the pre-rejection weights
                        if (tid == 0) {
                            sm.chainZ[sm.n_chain] = Z;
                            sm.chainS[sm.n_chain] = s;
                            sm.n_chain++;
                        }
                        Z = Znew;
                    }
                    __syncthreads();
                }
            }
            if (next < 0) {
                // bonus ~ current residual: t = (U' * Z) >> 32, smallest v with cumsum > t
                uint32_t U2 = rs::uniform_word(seed, step, g, 0xFFFFFFFFu, (uint32_t)c);
                const uint64_t t = (uint64_t)(((u128)U2 * Z) >> 32);
                const int tile_elems = kThreads * 8;
                const int ntiles = (V + tile_elems - 1) / tile_elems;
                for (int k = tid; k < ntiles; k += kThreads) sm.tile_sum[k] = 0ull;
                __syncthreads();
                // thread tid owns elements tile*tile_elems + tid*8 .. +7 (contiguous within a tile)
                for (int tile = 0; tile < ntiles; ++tile) {
                    int i = tile * kThreads + tid;
                    unsigned long long s8 = 0;
                    if (i < nvec) {
                        float x8[8], q8[8];
                        int n = load8(lv, i, x8);
                        if (mode == RS_ACCEPT_SAMPLE_MSS) load8(qv, i, q8);
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            if (j < n) {
                                uint64_t qw = (mode == RS_ACCEPT_SAMPLE_MSS) ? rs::draft_weight(q8[j]) : 0ull;
                                s8 += residual_weight(mode, rs::target_weight(x8[j], m, inv_tau), qw,
                                                      i * 8 + j, Zq, sm);
                            }
                        }
                    }
#pragma unroll
                    for (int o = 16; o; o >>= 1) s8 += __shfl_xor_sync(0xffffffffu, s8, o);
                    if ((tid & 31) == 0 && s8) atomicAdd(&sm.tile_sum[tile], s8);
                }
                __syncthreads();
                if (tid == 0) {
                    unsigned long long run = 0;
                    int tile = ntiles - 1;
                    for (int k = 0; k < ntiles; ++k) {
                        if (run + sm.tile_sum[k] > t) { tile = k; break; }
                        run += sm.tile_sum[k];
                    }
                    sm.bcast_i = tile;
                    sm.bcast_u = run;
                }
                __syncthreads();
                const int tile = sm.bcast_i;
                const unsigned long long base = sm.bcast_u;
                // exclusive scan of per-thread 8-element sums inside the tile
                int i = tile * kThreads + tid;
                uint64_t w8[8];
                unsigned long long s8 = 0;
                int n = 0;
                if (i < nvec) {
                    float x8[8], q8[8];
                    n = load8(lv, i, x8);
                    if (mode == RS_ACCEPT_SAMPLE_MSS) load8(qv, i, q8);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        w8[j] = 0;
                        if (j < n) {
                            uint64_t qw = (mode == RS_ACCEPT_SAMPLE_MSS) ? rs::draft_weight(q8[j]) : 0ull;
                            w8[j] = residual_weight(mode, rs::target_weight(x8[j], m, inv_tau), qw,
                                                    i * 8 + j, Zq, sm);
                            s8 += w8[j];
                        }
                    }
                }
                unsigned long long incl = s8;
                const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                if (lane == 31) sm.scan[wid] = incl;
                if (tid == 0) sm.bonus_v = V - 1;
                __syncthreads();
                unsigned long long wbase = base;
                for (int k = 0; k < wid; ++k) wbase += sm.scan[k];
                unsigned long long excl = wbase + incl - s8;
                if (s8 && excl <= t && t < excl + s8) {
                    unsigned long long accum = excl;
                    for (int j = 0; j < 8; ++j) {
                        accum += w8[j];
                        if (accum > t) { sm.bonus_v = i * 8 + j; break; }
                    }
                }
                __syncthreads();
                bonus = sm.bonus_v;
                stop = true;
            }
        }
        if (stop) break;
        c = next;
        ++a;
        if (tid == 0) pth[a] = c;
        __syncthreads();
    }
    if (tid == 0) {
        acc_out[b] = a;
        bonus_out[b] = (flags & RS_FLAG_NONFINITE) ? -1 : bonus;
        flags_out[b] = flags;
    }
}

__global__ void philox_kernel(const uint4* ctr, int64_t n, uint2 key, uint4* out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = rs::philox4x32_10(ctr[i], key);
}

__global__ void exp_spec_kernel(const float* x, int64_t n, float* y) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) y[i] = rs::exp_spec(x[i]);
}

}  // namespace

extern "C" rs_status rs_tree_accept(int32_t mode, const void* logits, int32_t logits_dtype,
                                    const float* draft_probs, const int32_t* parent,
                                    const int32_t* token, const int32_t* tree_off,
                                    const int64_t* gid, int32_t B, int32_t V, float temperature,
                                    uint64_t seed, uint64_t step, int32_t* accepted_len,
                                    int32_t* path, int32_t* bonus_token, int32_t* status_flags,
                                    void* ws, size_t ws_bytes, void* stream) {
    (void)ws;
    (void)ws_bytes;
    RS_REQUIRE(mode == RS_ACCEPT_GREEDY || mode == RS_ACCEPT_SAMPLE_DELTA ||
                   mode == RS_ACCEPT_SAMPLE_MSS,
               RS_ERR_INVALID_ARG, "rs_tree_accept: bad mode %d", mode);
    RS_REQUIRE(logits_dtype == RS_DTYPE_BF16 || logits_dtype == RS_DTYPE_F32, RS_ERR_INVALID_ARG,
               "rs_tree_accept: bad logits dtype %d", logits_dtype);
    RS_REQUIRE(B >= 0 && V >= 1, RS_ERR_INVALID_ARG, "rs_tree_accept: B=%d V=%d", B, V);
    RS_REQUIRE((mode == RS_ACCEPT_SAMPLE_MSS) == (draft_probs != nullptr), RS_ERR_INVALID_ARG,
               "rs_tree_accept: draft_probs must be given for MSS only");
    RS_REQUIRE(mode == RS_ACCEPT_GREEDY || temperature > 0.0f, RS_ERR_INVALID_ARG,
               "rs_tree_accept: temperature must be > 0");
    RS_REQUIRE((V + kThreads * 8 - 1) / (kThreads * 8) <= kMaxTiles, RS_ERR_UNSUPPORTED,
               "rs_tree_accept: V=%d too large", V);
    if (B == 0) return RS_OK;
    RS_REQUIRE(logits && parent && token && tree_off && gid && accepted_len && path && bonus_token &&
                   status_flags,
               RS_ERR_INVALID_ARG, "rs_tree_accept: null pointer");
    const float inv_tau = (mode == RS_ACCEPT_GREEDY) ? 1.0f : 1.0f / temperature;
    const int esz = logits_dtype == RS_DTYPE_BF16 ? 2 : 4;
    bool lvec = ((reinterpret_cast<uintptr_t>(logits) & 15) == 0) && ((int64_t)V * esz % 16 == 0);
    bool dvec = draft_probs && ((reinterpret_cast<uintptr_t>(draft_probs) & 15) == 0) && (V % 4 == 0);
    tree_accept_kernel<<<B, kThreads, 0, rs::as_stream(stream)>>>(
        mode, logits, logits_dtype, draft_probs, parent, token, tree_off, gid, V, inv_tau, seed,
        step, accepted_len, path, bonus_token, status_flags, lvec, dvec);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

extern "C" rs_status rs_philox4x32_10(const uint32_t* ctr, int64_t n, const uint32_t* key_host,
                                      uint32_t* out, void* stream) {
    RS_REQUIRE(n >= 0 && key_host, RS_ERR_INVALID_ARG, "rs_philox4x32_10: bad args");
    if (n == 0) return RS_OK;
    philox_kernel<<<(unsigned)((n + 255) / 256), 256, 0, rs::as_stream(stream)>>>(
        reinterpret_cast<const uint4*>(ctr), n, make_uint2(key_host[0], key_host[1]),
        reinterpret_cast<uint4*>(out));
    RS_LAUNCH_CHECK();
    return RS_OK;
}

extern "C" rs_status rs_exp_spec(const float* x, int64_t n, float* y, void* stream) {
    RS_REQUIRE(n >= 0, RS_ERR_INVALID_ARG, "rs_exp_spec: n < 0");
    if (n == 0) return RS_OK;
    exp_spec_kernel<<<(unsigned)((n + 255) / 256), 256, 0, rs::as_stream(stream)>>>(x, n, y);
    RS_LAUNCH_CHECK();
    return RS_OK;
}
