// a3: tree acceptance (readings Z5-Z8, Z15, "Bit-exact sampling").
//
// One thread-block CLUSTER per sample walks its tree from the root. The vocabulary is split
// into contiguous slices, one per CTA of the cluster; only the rows of the nodes on the walk
// are read (the algorithmic bytes are the visited rows), with 128-bit loads
// (greedy: four 16-byte loads in flight per thread, two rounds per 32 KB slice: measured 2 us faster per walk than the whole slice at once). Every reduction (argmax, max, integer sums, 128-bit max) is done
// per CTA with warp shuffles + shared memory and then all-reduced across the cluster through
// distributed shared memory, so every CTA takes the same decision; the walk itself (child
// tests, residual bookkeeping) is replicated.
//   GREEDY: argmax (ties -> lowest id); accept the lowest-index child whose token equals it;
//           bonus = argmax at the last node.
//   DELTA / MSS: integer weights w_v (exp_spec), Philox uniforms, 128-bit exact tests; the
//           residual after a rejection is kept implicitly for DELTA (excluded-token list) and
//           materialised for MSS after the first rejection (u32 per token in the workspace,
//           updated in place; before it the weights are recomputed from the logits); every
//           pass that defines the current weights leaves per-tile sums in shared memory, so
//           the bonus (inverse CDF: cluster prefix over slice totals, the tile, then a block
//           scan inside the owning CTA) needs no extra pass.
#include <cuda_bf16.h>

#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "compact_tail.cuh"
#include "sampling.cuh"
#include "sm100_ptx.cuh"

namespace {

using rs::u128;
using namespace rs::ptx;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTileVecs = kThreads;        // 8-element vectors per inverse-CDF tile
constexpr int kMaxTiles = 256;             // tiles per CTA slice
constexpr int kMaxCluster = 8;
#ifndef RS_ACC_RES_UNROLL
#define RS_ACC_RES_UNROLL 1
#endif
constexpr int kResUnroll = RS_ACC_RES_UNROLL;
#ifndef RS_ACC_P2_UNROLL
#define RS_ACC_P2_UNROLL 2
#endif
constexpr int kP2Unroll = RS_ACC_P2_UNROLL;   // vectors in flight per thread in the MSS weight-sum pass
//   // vectors in flight per thread in the MSS residual passes
#ifndef RS_ACC_INFLIGHT
#define RS_ACC_INFLIGHT 4
#endif
constexpr int kGreedyInflight = RS_ACC_INFLIGHT;   // 16-byte loads in flight per thread (greedy, bf16)
// measurement switches: compile-time only (tools/build_variant.sh), no runtime getenv
#ifndef RS_ACC_CS
#define RS_ACC_CS 0         // force the cluster size (1/2/4/8); 0: by V and B
#endif
#ifndef RS_ACC_PF
#define RS_ACC_PF 0         // greedy: L2 prefetch of the children's rows
#endif

#ifdef RS_ACC_TRACE
// profiling variant only (-DRS_ACC_TRACE): globaltimer stamps of the greedy walk per sample
// [0] kernel start, [1..5] start of rows 1..5, [6] walk end, [7] commit end
__device__ unsigned long long g_acc_trace[4096][8];
__device__ __forceinline__ unsigned long long acc_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define ACC_TRACE(b, k) do { if (cluster_rank() == 0 && threadIdx.x == 0 && (b) < 4096) g_acc_trace[b][k] = acc_gtime(); } while (0)
#else
#define ACC_TRACE(b, k) do { } while (0)
#endif

struct RowView {
    const void* base;
    int64_t row;
    int V;
    int dtype;      // RS_DTYPE_BF16 | RS_DTYPE_F32
    bool vec_ok;    // 16-byte aligned rows with V a multiple of the vector width
};

struct Raw8 {       // one 8-element vector as loaded (bf16: 4 words; fp32: 8 words)
    uint4 a, b;
};

__device__ __forceinline__ Raw8 load_raw(const RowView& rv, int i) {
    Raw8 r;
    const int v0 = i * 8;
    if (rv.dtype == RS_DTYPE_BF16) {
        const uint16_t* p = reinterpret_cast<const uint16_t*>(rv.base) + rv.row * (int64_t)rv.V + v0;
        if (rv.vec_ok && v0 + 8 <= rv.V) {
            r.a = __ldg(reinterpret_cast<const uint4*>(p));
        } else {
            uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (v0 + j < rv.V) w[j >> 1] |= (uint32_t)__ldg(p + j) << (16 * (j & 1));
            r.a = make_uint4(w[0], w[1], w[2], w[3]);
        }
        r.b = make_uint4(0, 0, 0, 0);
    } else {
        const float* p = reinterpret_cast<const float*>(rv.base) + rv.row * (int64_t)rv.V + v0;
        if (rv.vec_ok && v0 + 8 <= rv.V) {
            r.a = __ldg(reinterpret_cast<const uint4*>(p));
            r.b = __ldg(reinterpret_cast<const uint4*>(p) + 1);
        } else {
            uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (v0 + j < rv.V) w[j] = __float_as_uint(__ldg(p + j));
            r.a = make_uint4(w[0], w[1], w[2], w[3]);
            r.b = make_uint4(w[4], w[5], w[6], w[7]);
        }
    }
    return r;
}

__device__ __forceinline__ float raw_elem(const Raw8& r, int dtype, int j) {
    if (dtype == RS_DTYPE_BF16) {
        const uint32_t w = j < 2 ? r.a.x : j < 4 ? r.a.y : j < 6 ? r.a.z : r.a.w;
        return __uint_as_float((j & 1) ? (w & 0xFFFF0000u) : (w << 16));
    }
    const uint32_t w = j == 0 ? r.a.x : j == 1 ? r.a.y : j == 2 ? r.a.z : j == 3 ? r.a.w
                     : j == 4 ? r.b.x : j == 5 ? r.b.y : j == 6 ? r.b.z : r.b.w;
    return __uint_as_float(w);
}

// Visit every element of this CTA's slice [vbeg, vend) (in 8-vectors) of row lv (and, if
// with_q, the same elements of row qv): fn(v, x, q). kUnroll loads in flight per thread.
template <int kUnroll = 4, typename F>
__device__ __forceinline__ void for_slice(const RowView& lv, const RowView& qv, bool with_q, int vbeg, int vend,
                                          F fn) {
    for (int i0 = vbeg + (int)threadIdx.x; i0 < vend; i0 += kUnroll * kThreads) {
        Raw8 x[kUnroll], q[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int i = i0 + u * kThreads;
            if (i < vend) {
                x[u] = load_raw(lv, i);
                if (with_q) q[u] = load_raw(qv, i);
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int i = i0 + u * kThreads;
            if (i < vend) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int v = i * 8 + j;
                    if (v < lv.V) fn(v, raw_elem(x[u], lv.dtype, j), with_q ? raw_elem(q[u], RS_DTYPE_F32, j) : 0.0f);
                }
            }
        }
    }
}

struct Smem {
    unsigned long long red[kWarps][2];
    unsigned long long redn[kWarps][3];   // allreduce_n's per-warp partials
    unsigned long long xch[2][kMaxCluster > 2 ? 4 : 4];   // cluster exchange slots (double-buffered)
    // push exchange (allreduce_n, draw_bonus): CTA r stores its partials into slot [phase][r] of
    // EVERY CTA before the cluster barrier, so after it all reads are local (no DSMEM round trip,
    // and no CTA touches another's shared memory after its last barrier)
    unsigned long long xp[2][16][3];
    unsigned long long tile_sum[kMaxTiles];
    unsigned long long scan[kWarps];
    int parent[RS_MAX_TREE];
    int token[RS_MAX_TREE];
    int excluded[RS_MAX_TREE];
    int n_excluded;
    int flag;
    int bcast_i;
    unsigned long long bcast_u;
    int bonus_v;
    int path_s[RS_MAX_TREE];   // the accepted path (every CTA; the fused KV commit reads it)
    unsigned long long kids;   // MSS: bit i = node i has children (its draft row is read, Z29)
    int qrow[RS_MAX_TREE];     // MSS: row of node i's draft distribution (draft_row, or off + i)
};

// Orderable 32-bit key of a float (larger float -> larger key).
__device__ __forceinline__ uint32_t fkey(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

enum Op { OP_MAX = 0, OP_SUM = 1, OP_OR = 2 };

__device__ __forceinline__ unsigned long long op_apply(int op, unsigned long long a, unsigned long long b) {
    return op == OP_MAX ? (a > b ? a : b) : op == OP_SUM ? a + b : (a | b);
}

// Block + cluster all-reduce of N u64 values (ops op[k]); identical result in every thread of
// every CTA of the cluster. Warps reduce by shuffles, lane 0 parks the warp's values; every warp
// then reduces the kWarps partials (lane w reads warp w's) by shuffles; with a cluster, warp 0's
// lane c pushes the CTA's values into CTA c's slot [phase][my rank], one cluster barrier, and every
// warp reduces the cs slots of its own shared memory. `phase` alternates the slots: CTA A writes
// B's slot [p] again only after the next barrier, which B passes only after reading [p].
template <int N>
__device__ __forceinline__ void allreduce_n(unsigned long long (&v)[N], const int (&op)[N], Smem& sm, int& phase) {
    static_assert(N >= 1 && N <= 3, "allreduce_n: 1..3 values");
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1)
#pragma unroll
        for (int k = 0; k < N; ++k) v[k] = op_apply(op[k], v[k], __shfl_xor_sync(0xffffffffu, v[k], o));
    __syncwarp();
    __syncthreads();   // every read of sm.red by the previous reduction is done
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < N; ++k) sm.redn[w][k] = v[k];
    }
    __syncwarp();
    __syncthreads();
    unsigned long long a[N];
#pragma unroll
    for (int k = 0; k < N; ++k) a[k] = lane < kWarps ? sm.redn[lane][k] : 0ull;   // 0: identity of MAX/SUM/OR
#pragma unroll
    for (int o = 16; o; o >>= 1)
#pragma unroll
        for (int k = 0; k < N; ++k) a[k] = op_apply(op[k], a[k], __shfl_xor_sync(0xffffffffu, a[k], o));
    const uint32_t cs = cluster_size();
    if (cs > 1) {
        if (w == 0 && (uint32_t)lane < cs) {
            const uint32_t me = cluster_rank();
#pragma unroll
            for (int k = 0; k < N; ++k) st_dsmem_u64(&sm.xp[phase][me][k], (uint32_t)lane, a[k]);
        }
        __syncwarp();
        cluster_sync_all();
#pragma unroll
        for (int k = 0; k < N; ++k) a[k] = (uint32_t)lane < cs ? sm.xp[phase][lane][k] : 0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1)
#pragma unroll
            for (int k = 0; k < N; ++k) a[k] = op_apply(op[k], a[k], __shfl_xor_sync(0xffffffffu, a[k], o));
        phase ^= 1;
    }
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] = a[k];
}

__device__ __forceinline__ void allreduce2(unsigned long long& v0, int op0, unsigned long long& v1, int op1, Smem& sm,
                                           int& phase) {
    unsigned long long v[2] = {v0, v1};
    const int op[2] = {op0, op1};
    allreduce_n<2>(v, op, sm, phase);
    v0 = v[0];
    v1 = v[1];
}

// 128-bit max all-reduce (hi/lo lexicographic).
__device__ __forceinline__ u128 allreduce_max128(u128 v, Smem& sm, int& phase) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        unsigned long long hi = __shfl_xor_sync(0xffffffffu, (unsigned long long)(v >> 64), o);
        unsigned long long lo = __shfl_xor_sync(0xffffffffu, (unsigned long long)v, o);
        u128 v2 = ((u128)hi << 64) | lo;
        if (v2 > v) v = v2;
    }
    __syncwarp();
    __syncthreads();
    if (lane == 0) { sm.red[w][0] = (unsigned long long)(v >> 64); sm.red[w][1] = (unsigned long long)v; }
    __syncwarp();
    __syncthreads();
    u128 r = 0;
    for (int k = 0; k < kWarps; ++k) {
        u128 x = ((u128)sm.red[k][0] << 64) | sm.red[k][1];
        if (x > r) r = x;
    }
    const uint32_t cs = cluster_size();
    if (cs > 1) {
        if (threadIdx.x == 0) { sm.xch[phase][0] = (unsigned long long)(r >> 64); sm.xch[phase][1] = (unsigned long long)r; }
        cluster_sync_all();
        const uint32_t me = cluster_rank();
        for (uint32_t c = 0; c < cs; ++c) {
            if (c == me) continue;
            u128 x = ((u128)ld_dsmem_u64(&sm.xch[phase][0], c) << 64) | ld_dsmem_u64(&sm.xch[phase][1], c);
            if (x > r) r = x;
        }
        phase ^= 1;
    }
    return r;
}

// DELTA residual: rejected tokens are excluded (weight 0); other weights are unchanged.
__device__ __forceinline__ uint64_t delta_weight(uint64_t w, int tok, const Smem& sm) {
    for (int e = 0; e < sm.n_excluded; ++e)
        if (sm.excluded[e] == tok) return 0;
    return w;
}

// Warp-reduce a per-vector weight sum and add it to the CTA's inverse-CDF tile sum (the 32
// lanes of a warp always hold vectors of the same tile: tiles are kThreads vectors).
__device__ __forceinline__ void tile_add(Smem& sm, int tile, unsigned long long s8) {
#pragma unroll
    for (int o = 16; o; o >>= 1) s8 += __shfl_xor_sync(0xffffffffu, s8, o);
    if ((threadIdx.x & 31) == 0 && s8) atomicAdd(&sm.tile_sum[tile], s8);
}

__device__ __forceinline__ void clear_tiles(Smem& sm) {
    for (int k = threadIdx.x; k < kMaxTiles; k += kThreads) sm.tile_sum[k] = 0ull;
    __syncwarp();
    __syncthreads();
}

// MSS residual weights of 8 tokens, stored u32 (a residual is shifted so its max has <= 32
// bits); rows are padded to a multiple of 8 tokens.
struct W8 {
    uint4 a, b;
};
__device__ __forceinline__ W8 load_w8(const uint32_t* wrow, int i) {
    const uint4* p = reinterpret_cast<const uint4*>(wrow) + 2 * (int64_t)i;
    return W8{__ldcg(p), __ldcg(p + 1)};
}
__device__ __forceinline__ uint32_t w8_elem(const W8& w, int j) {
    return j == 0 ? w.a.x : j == 1 ? w.a.y : j == 2 ? w.a.z : j == 3 ? w.a.w
         : j == 4 ? w.b.x : j == 5 ? w.b.y : j == 6 ? w.b.z : w.b.w;
}

// Bonus draw by inverse CDF over the current weights of the node (DESIGN.md "Bit-exact
// sampling"): the smallest token v with sum_{j<=v} w_j > t. The per-tile sums of this CTA's
// slice are current in sm.tile_sum; a cluster prefix of slice totals finds the owning CTA,
// its tile sums the tile, and a block scan over weights8(i, w8) (the 8 weights of vector i)
// the token. Sets `owner` (the CTA whose result is the bonus) and returns its token.
template <typename F>
__device__ __forceinline__ int draw_bonus(Smem& sm, int& phase, uint64_t t, int vbeg, int vend, int V, bool& owner,
                                          F weights8) {
    const int tid = threadIdx.x;
    const uint32_t cs = cluster_size(), crank = cluster_rank();
    const int ntiles = (vend - vbeg + kTileVecs - 1) / kTileVecs;
    __syncwarp();
    __syncthreads();
    unsigned long long slice_total = 0;
    for (int k = 0; k < ntiles; ++k) slice_total += sm.tile_sum[k];
    unsigned long long before = 0;
    if (cs > 1) {   // push exchange (see allreduce_n): every CTA learns every slice total locally
        if (tid < (int)cs) st_dsmem_u64(&sm.xp[phase][crank][0], (uint32_t)tid, slice_total);
        __syncwarp();
        cluster_sync_all();
        for (uint32_t r = 0; r < crank; ++r) before += sm.xp[phase][r][0];
        phase ^= 1;
    }
    owner = slice_total > 0 && before <= t && t < before + slice_total;
    if (!owner) return -1;
    if (tid == 0) {
        unsigned long long run = before;
        int tile = ntiles - 1;
        for (int k = 0; k < ntiles; ++k) {
            if (run + sm.tile_sum[k] > t) { tile = k; break; }
            run += sm.tile_sum[k];
        }
        sm.bcast_i = tile;
        sm.bcast_u = run;
        sm.bonus_v = V - 1;
    }
    __syncwarp();
    __syncthreads();
    const int i = vbeg + sm.bcast_i * kTileVecs + tid;
    const unsigned long long tbase = sm.bcast_u;
    uint64_t w8[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) w8[j] = 0;
    if (i < vend) weights8(i, w8);
    unsigned long long s8 = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s8 += w8[j];
    unsigned long long incl = s8;
    const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) sm.scan[wid] = incl;
    __syncwarp();
    __syncthreads();
    unsigned long long wbase = tbase;
    for (int k = 0; k < wid; ++k) wbase += sm.scan[k];
    const unsigned long long excl = wbase + incl - s8;
    if (s8 && excl <= t && t < excl + s8) {
        unsigned long long accum = excl;
        for (int j = 0; j < 8; ++j) {
            accum += w8[j];
            if (accum > t) { sm.bonus_v = i * 8 + j; break; }
        }
    }
    __syncwarp();
    __syncthreads();
    return sm.bonus_v;
}

// The fused KV commit (rs_tree_accept_compact): once the walk is over, the CTAs of the sample's
// cluster split its compaction lanes (rs::compact_sample; the leader writes new_len and moves).
// The inverse-CDF tile sums are dead by then: their storage holds the move list.
template <typename CA>
__device__ __forceinline__ void fused_commit(const CA& ca, int b, int a, Smem& sm) {
    static_assert(sizeof(rs::CompactSmem) <= sizeof(sm.tile_sum), "move list must fit the tile sums");
    __syncwarp();
    __syncthreads();   // sm.path_s complete; every read of the tile sums done
    rs::compact_sample(ca, b, a, [&](int k) { return sm.path_s[k]; }, (int)cluster_rank(), (int)cluster_size(),
                       cluster_rank() == 0, *reinterpret_cast<rs::CompactSmem*>(sm.tile_sum));
}

// MODE is a template parameter so the greedy walk compiles without the 128-bit sampling
// machinery (register budget: 4 CTAs/SM greedy, 2 CTAs/SM sampling); DT (the logits dtype)
// too, so a bf16 vector occupies 4 registers, not 8.
template <int MODE, int DT, typename CA>
__global__ void __launch_bounds__(kThreads, MODE == RS_ACCEPT_GREEDY ? 4 : 2)
tree_accept_kernel(int mode_rt, const void* __restrict__ logits, int dtype_rt, const float* __restrict__ draft,
                   const int32_t* __restrict__ parent, const int32_t* __restrict__ token,
                   const int32_t* __restrict__ tree_off, const int64_t* __restrict__ gid, int V, float inv_tau,
                   uint64_t seed, uint64_t step, int32_t* __restrict__ acc_out, int32_t* __restrict__ path_out,
                   int32_t* __restrict__ bonus_out, int32_t* __restrict__ flags_out, bool logits_vec_ok,
                   bool draft_vec_ok, uint32_t* __restrict__ wbuf, int prefetch_children,
                   const __grid_constant__ CA ca) {
    (void)mode_rt;
    (void)dtype_rt;
    constexpr int dtype = DT;
    constexpr int mode = MODE;
    __shared__ Smem sm;
    const uint32_t cs = cluster_size();
    const uint32_t crank = cluster_rank();
    const int b = blockIdx.x / cs;
    const int tid = threadIdx.x;
    const bool leader = crank == 0;
    const int off = tree_off[b];
    const int T = tree_off[b + 1] - off;
    int32_t* pth = path_out + (int64_t)b * RS_MAX_TREE;
    int phase = 0;
    ACC_TRACE(b, 0);
    if (leader && tid < RS_MAX_TREE) pth[tid] = -1;
    // tree check in parallel: node i needs parent[i] in [0, i) (root: -1) and, for a draft
    // node (i >= 1), a vocabulary token 0 <= token[i] < V (sampling modes index rows by it)
    bool bad_node = !(T >= 1 && T <= RS_MAX_TREE);
    if (!bad_node && tid < T) {
        const int pp = parent[off + tid];
        const int tk = token[off + tid];
        sm.parent[tid] = pp;
        sm.token[tid] = tk;
        bad_node = tid == 0 ? pp != -1 : !(pp >= 0 && pp < tid && tk >= 0 && tk < V);
    }
    if (__syncthreads_or(bad_node)) {
        if (leader && tid == 0) { acc_out[b] = 0; bonus_out[b] = -1; flags_out[b] = RS_FLAG_MALFORMED; }
        if constexpr (CA::kOn) fused_commit(ca, b, 0, sm);   // accepted_len 0: new_len only
        return;   // uniform across the cluster: no cluster barrier is reached
    }
    const int64_t g = gid[b];
    const int nvec = (V + 7) / 8;
    const int per = (nvec + (int)cs - 1) / (int)cs;
    const int vbeg = min(nvec, (int)crank * per), vend = min(nvec, vbeg + per);
    int c = 0, a = 0, bonus = -1, flags = 0;
    bool bonus_mine = leader;   // which CTA writes the bonus
    if (leader && tid == 0) pth[0] = 0;
    if (tid == 0) sm.path_s[0] = 0;
    __syncwarp();
    __syncthreads();

    for (;;) {
        if (a >= 1 && a <= 5) ACC_TRACE(b, a);
        const RowView lv{logits, (int64_t)(off + c), V, dtype, logits_vec_ok};
        const RowView qv{draft, (int64_t)(off + c), V, RS_DTYPE_F32, draft_vec_ok};
        int next = -1;
        bool stop = false;
        if (mode == RS_ACCEPT_GREEDY) {
            // key = (orderable value << 32) | ~index: max key = max value, lowest index on ties
            unsigned long long best = 0, bad = 0;
            auto upd = [&](int v, float x) {
                bad |= isfinite(x) ? 0ull : 1ull;
                const unsigned long long k = ((unsigned long long)fkey(x) << 32) | (uint32_t)(~(uint32_t)v);
                best = best > k ? best : k;
            };
            if (dtype == RS_DTYPE_BF16 && logits_vec_ok) {
                // bf16 rows: kGreedyInflight x 16-byte loads in flight per thread. Per thread:
                // packed bf16x2 max (__hmax2) and a packed |bits| max for the non-finite check,
                // then the lowest index holding that max (float equality, so -0 == +0 as in the
                // oracle's strict '>' scan); the 64-bit key is built once per thread.
                const uint4* row = reinterpret_cast<const uint4*>(
                    reinterpret_cast<const uint16_t*>(logits) + (int64_t)(off + c) * V);
                // warm L2 with this CTA's slice of every child's row while row c streams: the
                // next row of the walk is one of them (speculative reads of the siblings)
                if (prefetch_children && tid > c && tid < T && sm.parent[tid] == c && vend > vbeg)
                    bulk_prefetch_l2(row + (int64_t)(tid - c) * (V / 8) + vbeg, (uint32_t)(vend - vbeg) * 16u);
                __nv_bfloat162 vmax = __halves2bfloat162(__ushort_as_bfloat16((unsigned short)0xFF80u),
                                                        __ushort_as_bfloat16((unsigned short)0xFF80u));   // -inf
                uint32_t amag = 0;
                int first = -1;
                float fmax_t = -INFINITY;
                for (int i0 = vbeg + tid; i0 < vend; i0 += kGreedyInflight * kThreads) {
                    uint4 x[kGreedyInflight];
#pragma unroll
                    for (int u = 0; u < kGreedyInflight; ++u) {
                        const int i = i0 + u * kThreads;
                        x[u] = (i < vend) ? __ldg(row + i) : make_uint4(0xFF7FFF7Fu, 0xFF7FFF7Fu, 0xFF7FFF7Fu, 0xFF7FFF7Fu);   // lowest finite bf16
                    }
                    __nv_bfloat162 cm = vmax;
#pragma unroll
                    for (int u = 0; u < kGreedyInflight; ++u) {
                        const uint32_t w[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            cm = __hmax2(cm, *reinterpret_cast<const __nv_bfloat162*>(&w[q]));
                            amag = __vmaxu2(amag, w[q] & 0x7FFF7FFFu);
                        }
                    }
                    const float chunk_max = fmaxf(__bfloat162float(cm.x), __bfloat162float(cm.y));
                    if (chunk_max > fmax_t) {   // the new max is in this chunk: lowest index of it
                        fmax_t = chunk_max;
                        first = -1;
#pragma unroll
                        for (int u = 0; u < kGreedyInflight; ++u) {
                            const uint32_t w[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const float h = __uint_as_float((j & 1) ? (w[j >> 1] & 0xFFFF0000u) : (w[j >> 1] << 16));
                                if (first < 0 && h == chunk_max) first = (i0 + u * kThreads) * 8 + j;
                            }
                        }
                    }
                    vmax = cm;
                }
                // bf16 magnitude bits >= 0x7F80 <=> inf or NaN (padding loads are the lowest finite value)
                bad = ((amag & 0xFFFFu) >= 0x7F80u || (amag >> 16) >= 0x7F80u) ? 1ull : 0ull;
                if (first >= 0) {
                    const float mcan = fmax_t == 0.0f ? 0.0f : fmax_t;   // -0 -> +0: ties by index
                    best = ((unsigned long long)fkey(mcan) << 32) | (uint32_t)(~(uint32_t)first);
                }
            } else {
                for_slice<2>(lv, qv, false, vbeg, vend, [&](int v, float x, float) { upd(v, x); });
            }
            allreduce2(best, OP_MAX, bad, OP_OR, sm, phase);
            if (bad) { flags |= RS_FLAG_NONFINITE; break; }
            const int am = (int)(~(uint32_t)best);
            for (int x = c + 1; x < T; ++x)
                if (sm.parent[x] == c && sm.token[x] == am) { next = x; break; }
            if (next < 0) { bonus = am; stop = true; }
        } else if (mode == RS_ACCEPT_SAMPLE_MSS) {
            // pass 1: row max (+ non-finite check)
            unsigned long long mk = 0, bad = 0;
            for_slice(lv, qv, false, vbeg, vend, [&](int, float x, float) {
                bad |= isfinite(x) ? 0ull : 1ull;
                const unsigned long long k = fkey(x);
                mk = mk > k ? mk : k;
            });
            allreduce2(mk, OP_MAX, bad, OP_OR, sm, phase);
            if (bad) { flags |= RS_FLAG_NONFINITE; break; }
            const float m = fkey_inv((uint32_t)mk);
            // The weights of node c are implicit (w_v recomputed from the logits) until a
            // rejection changes them; from then on the residual lives in wrow (u32 per token).
            // Every pass that defines the current weights also leaves their per-tile sums in
            // shared memory, so the bonus draw needs no extra pass.
            const int Vp = (V + 7) & ~7;
            uint32_t* wrow = wbuf + (int64_t)b * Vp;
            bool resid = false;
            // pass 2: Z = sum w, Zq = sum qw (+ tile sums of w)
            unsigned long long zs = 0, zq = 0;
            clear_tiles(sm);
            for (int base = vbeg; base < vend; base += kP2Unroll * kThreads) {
                Raw8 x[kP2Unroll], q[kP2Unroll];
#pragma unroll
                for (int u = 0; u < kP2Unroll; ++u) {
                    const int i = base + u * kThreads + tid;
                    if (i < vend) { x[u] = load_raw(lv, i); q[u] = load_raw(qv, i); }
                }
#pragma unroll
                for (int u = 0; u < kP2Unroll; ++u) {
                    const int i = base + u * kThreads + tid;
                    unsigned long long s8 = 0;
                    if (i < vend) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            if (i * 8 + j < V) {
                                s8 += rs::target_weight(raw_elem(x[u], dtype, j), m, inv_tau);
                                zq += rs::draft_weight(raw_elem(q[u], RS_DTYPE_F32, j));
                            }
                        }
                    }
                    zs += s8;
                    tile_add(sm, (base - vbeg) / kThreads + u, s8);
                }
            }
            allreduce2(zs, OP_SUM, zq, OP_SUM, sm, phase);
            uint64_t Z = zs;
            const uint64_t Zq = zq;
            // r_v = max(prev_v * Zq - qw_v * Z, 0) for token j of vector i
            auto residual1 = [&](int i, int j, const Raw8& x, const W8& w, const Raw8& q) -> u128 {
                if (i * 8 + j >= V) return 0;
                const uint64_t prev = resid ? (uint64_t)w8_elem(w, j)
                                            : rs::target_weight(raw_elem(x, dtype, j), m, inv_tau);
                const u128 lhs = (u128)prev * Zq;
                const u128 rhs = (u128)rs::draft_weight(raw_elem(q, RS_DTYPE_F32, j)) * Z;
                return lhs > rhs ? lhs - rhs : 0;
            };
            int rank = 0;
            for (int x = c + 1; x < T && next < 0; ++x) {
                if (sm.parent[x] != c) continue;
                const int tk = sm.token[x];
                if (tid == 0) {
                    const int64_t ro = (int64_t)(off + c) * V + tk;
                    const float l = (dtype == RS_DTYPE_BF16)
                                        ? rs::bf16_bits_to_f32(reinterpret_cast<const uint16_t*>(logits)[ro])
                                        : reinterpret_cast<const float*>(logits)[ro];
                    const uint64_t qw = rs::draft_weight(draft[ro]);
                    const uint64_t wt = resid ? (uint64_t)__ldcg(wrow + tk) : rs::target_weight(l, m, inv_tau);
                    const uint32_t U = rs::uniform_word(seed, step, g, (uint32_t)rank, (uint32_t)c);
                    const bool acc = qw == 0 ? wt > 0 : ((u128)U * ((u128)qw * Z)) < (((u128)wt * Zq) << 32);
                    sm.bcast_i = acc ? 1 : 0;
                }
                __syncwarp();   // (reconverge the warp before the aligned CTA barrier)
        __syncwarp();
    __syncthreads();
                const bool accepted = sm.bcast_i != 0;
                __syncwarp();   // (reconverge the warp before the aligned CTA barrier)
        __syncwarp();
    __syncthreads();
                if (accepted) { next = x; break; }
                ++rank;
                // residual: pass A = its max (the shift), pass B = shifted values written back
                // (u32) with their sums. An all-zero residual (max 0, quantisation only) keeps
                // the pre-rejection weights.
                u128 rmax = 0;
                for (int base = vbeg; base < vend; base += kResUnroll * kThreads) {
                    Raw8 xs[kResUnroll], qs[kResUnroll];
                    W8 ws[kResUnroll];
#pragma unroll
                    for (int u = 0; u < kResUnroll; ++u) {
                        const int i = base + u * kThreads + tid;
                        if (i < vend) {
                            if (resid) ws[u] = load_w8(wrow, i); else xs[u] = load_raw(lv, i);
                            qs[u] = load_raw(qv, i);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kResUnroll; ++u) {
                        const int i = base + u * kThreads + tid;
                        if (i < vend) {
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const u128 r = residual1(i, j, xs[u], ws[u], qs[u]);
                                rmax = r > rmax ? r : rmax;
                            }
                        }
                    }
                }
                const u128 mxr = allreduce_max128(rmax, sm, phase);
                if (mxr != 0) {
                    int sh = rs::bitlen128(mxr) - 32;
                    if (sh < 0) sh = 0;
                    unsigned long long zn = 0, dummy = 0;
                    clear_tiles(sm);
                    for (int base = vbeg; base < vend; base += kResUnroll * kThreads) {
                        Raw8 xs[kResUnroll], qs[kResUnroll];
                        W8 ws[kResUnroll];
#pragma unroll
                        for (int u = 0; u < kResUnroll; ++u) {
                            const int i = base + u * kThreads + tid;
                            if (i < vend) {
                                if (resid) ws[u] = load_w8(wrow, i); else xs[u] = load_raw(lv, i);
                                qs[u] = load_raw(qv, i);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < kResUnroll; ++u) {
                            const int i = base + u * kThreads + tid;
                            unsigned long long s8 = 0;
                            if (i < vend) {
                                uint32_t wn[8];
#pragma unroll
                                for (int j = 0; j < 8; ++j) {
                                    wn[j] = (uint32_t)(residual1(i, j, xs[u], ws[u], qs[u]) >> sh);
                                    s8 += wn[j];
                                }
                                uint4* p = reinterpret_cast<uint4*>(wrow) + 2 * (int64_t)i;
                                __stcg(p, make_uint4(wn[0], wn[1], wn[2], wn[3]));
                                __stcg(p + 1, make_uint4(wn[4], wn[5], wn[6], wn[7]));
                            }
                            zn += s8;
                            tile_add(sm, (base - vbeg) / kThreads + u, s8);
                        }
                    }
                    resid = true;
                    allreduce2(zn, OP_SUM, dummy, OP_OR, sm, phase);   // (cluster barrier: the
                    Z = zn;                                             //  new weights are visible)
                }
                __syncwarp();   // (reconverge the warp before the aligned CTA barrier)
        __syncwarp();
    __syncthreads();
            }
            if (next < 0) {
                const uint32_t U2 = rs::uniform_word(seed, step, g, 0xFFFFFFFFu, (uint32_t)c);
                const uint64_t t = (uint64_t)(((u128)U2 * Z) >> 32);
                bonus = draw_bonus(sm, phase, t, vbeg, vend, V, bonus_mine, [&](int i, uint64_t w8[8]) {
                    if (resid) {
                        const W8 w = load_w8(wrow, i);
#pragma unroll
                        for (int j = 0; j < 8; ++j) w8[j] = (i * 8 + j < V) ? w8_elem(w, j) : 0u;
                    } else {
                        const Raw8 xr = load_raw(lv, i);
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            w8[j] = (i * 8 + j < V) ? rs::target_weight(raw_elem(xr, dtype, j), m, inv_tau) : 0ull;
                    }
                });
                stop = true;
            }
        } else {
            // DELTA: the residual after rejecting child x is the current weights with w_x = 0
            // (an excluded-token list), so no pass is needed per rejection.
            unsigned long long mk = 0, bad = 0;
            for_slice(lv, qv, false, vbeg, vend, [&](int, float x, float) {
                bad |= isfinite(x) ? 0ull : 1ull;
                const unsigned long long k = fkey(x);
                mk = mk > k ? mk : k;
            });
            allreduce2(mk, OP_MAX, bad, OP_OR, sm, phase);
            if (bad) { flags |= RS_FLAG_NONFINITE; break; }
            const float m = fkey_inv((uint32_t)mk);
            // pass 2: Z = sum w (+ tile sums of w)
            unsigned long long zs = 0, dummy = 0;
            clear_tiles(sm);
            for (int base = vbeg; base < vend; base += 4 * kThreads) {
                Raw8 x[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = base + u * kThreads + tid;
                    if (i < vend) x[u] = load_raw(lv, i);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = base + u * kThreads + tid;
                    unsigned long long s8 = 0;
                    if (i < vend) {
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            if (i * 8 + j < V) s8 += rs::target_weight(raw_elem(x[u], dtype, j), m, inv_tau);
                    }
                    zs += s8;
                    tile_add(sm, (base - vbeg) / kThreads + u, s8);
                }
            }
            allreduce2(zs, OP_SUM, dummy, OP_OR, sm, phase);
            uint64_t Z = zs;
            if (tid == 0) sm.n_excluded = 0;
            __syncwarp();   // (reconverge the warp before the aligned CTA barrier)
        __syncwarp();
    __syncthreads();
            int rank = 0;
            for (int x = c + 1; x < T && next < 0; ++x) {
                if (sm.parent[x] != c) continue;
                const int tk = sm.token[x];
                if (tid == 0) {
                    const int64_t ro = (int64_t)(off + c) * V + tk;
                    const float l = (dtype == RS_DTYPE_BF16)
                                        ? rs::bf16_bits_to_f32(reinterpret_cast<const uint16_t*>(logits)[ro])
                                        : reinterpret_cast<const float*>(logits)[ro];
                    const uint64_t wt = delta_weight(rs::target_weight(l, m, inv_tau), tk, sm);
                    const uint32_t U = rs::uniform_word(seed, step, g, (uint32_t)rank, (uint32_t)c);
                    const bool acc = ((u128)U * Z) < ((u128)wt << 32);
                    sm.bcast_i = acc ? 1 : 0;
                    sm.bcast_u = wt;
                    if (!acc) {
                        // the rejected token leaves the residual: its weight leaves its tile
                        const int ti = tk / 8;
                        if (wt && ti >= vbeg && ti < vend) sm.tile_sum[(ti - vbeg) / kTileVecs] -= wt;
                        sm.excluded[sm.n_excluded++] = tk;
                    }
                }
                __syncwarp();   // (reconverge the warp before the aligned CTA barrier)
        __syncwarp();
    __syncthreads();
                const bool accepted = sm.bcast_i != 0;
                const uint64_t wt = sm.bcast_u;
                __syncwarp();   // (reconverge the warp before the aligned CTA barrier)
        __syncwarp();
    __syncthreads();
                if (accepted) { next = x; break; }
                ++rank;
                Z -= wt;
            }
            if (next < 0) {
                const uint32_t U2 = rs::uniform_word(seed, step, g, 0xFFFFFFFFu, (uint32_t)c);
                const uint64_t t = (uint64_t)(((u128)U2 * Z) >> 32);
                bonus = draw_bonus(sm, phase, t, vbeg, vend, V, bonus_mine, [&](int i, uint64_t w8[8]) {
                    const Raw8 xr = load_raw(lv, i);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        w8[j] = (i * 8 + j < V) ? delta_weight(rs::target_weight(raw_elem(xr, dtype, j), m, inv_tau),
                                                               i * 8 + j, sm)
                                                : 0ull;
                });
                stop = true;
            }
        }
        if (stop) break;
        c = next;
        ++a;
        if (leader && tid == 0) pth[a] = c;
        if (tid == 0) sm.path_s[a] = c;
        __syncwarp();   // (reconverge the warp before the aligned CTA barrier)
        __syncwarp();
    __syncthreads();
    }
    if (tid == 0) {
        if (leader) {
            acc_out[b] = a;
            flags_out[b] = flags;
        }
        if (flags & RS_FLAG_NONFINITE) {
            if (leader) bonus_out[b] = -1;
        } else if (bonus_mine && mode != RS_ACCEPT_GREEDY) {
            bonus_out[b] = bonus;
        } else if (leader && mode == RS_ACCEPT_GREEDY) {
            bonus_out[b] = bonus;
        }
    }
    ACC_TRACE(b, 6);
    if constexpr (CA::kOn) fused_commit(ca, b, a, sm);
    ACC_TRACE(b, 7);
    // keep every CTA's shared memory alive until all remote reads of the cluster are done (DELTA's
    // 128-bit reductions and child tests read peers after their barriers; the greedy walk only
    // uses push exchanges, whose last barrier already orders every access)
    if (MODE != RS_ACCEPT_GREEDY && cs > 1) cluster_sync_all();
}

// ============================================================================ MSS, row in smem
// SAMPLE_MSS with the visited row kept ON CHIP. One cluster of CS CTAs (16 where the device
// allows the non-portable size, else 8) per sample; CTA r owns the vocabulary slice
// [r*per, (r+1)*per) (in 8-token vectors) and keeps per token two u32 words in shared memory:
//   wsl: the target weight w_v (<= 2^32), stored as w_v, or 0xFFFFFFFF for w_v = 2^32 (only a
//        row maximum has e = 1; every other w_v <= 2^32 - 2^8, so the code is unambiguous);
//        after the node's first rejection the shifted residual (a plain u32, "resid" state);
//   qsl: the draft weight qw_v = trunc(q_v * 2^32), encoded the same way (q_v in [0, 1]).
// A visited node costs ONE pass over HBM (logits + q: the algorithmic bytes): pass L loads the
// row (raw logits parked in wsl) with its max, a validity flag and Zq; pass E turns wsl into
// weights with Z and the inverse-CDF tile sums. A rejection runs over shared memory only:
// pass A computes every r_v = max(w_v Zq - qw_v Z, 0) once in 128 bits and stores it per
// 8-token vector as r_v >> t (t = max(0, bitlen(vector max) - 32), a byte per vector; an
// all-zero vector keeps its old words and is marked 0xFF); pass B applies the global shift
// s = max(0, bitlen(max r) - 32) >= t as (r >> t) >> (s - t) = r >> s (exact), with the sums.
// If every r_v is 0 (quantisation only) nothing was overwritten: the weights are kept.
// Children's current (w, qw) are published by the owner CTA of their token into small arrays
// before the cluster barrier that ends pass E / pass B; child tests read them through DSMEM, so
// no barrier is needed between a node's tests and the next row's loads. The bonus is the
// inverse CDF of the current weights (draw_bonus).
constexpr int kMssThreads = kThreads;   // == kTileVecs: one vector per thread per tile row
#ifndef RS_MSS_LUNROLL
#define RS_MSS_LUNROLL 1
#endif
constexpr int kMssLUnroll = RS_MSS_LUNROLL;   // pass L: row vectors in flight per thread (a slice in one round)

struct MssSmem {
    unsigned long long childw[RS_MAX_TREE];   // current w of child x's token (owner CTA only)
    unsigned long long childq[RS_MAX_TREE];   // qw of child x's token
};

// Block + cluster all-reduce of three u64 values (ops op[0..2]); same result in every thread.
__device__ __forceinline__ void allreduce3(unsigned long long v[3], const int op[3], Smem& sm, int& phase) {
    unsigned long long a[3] = {v[0], v[1], v[2]};
    const int o[3] = {op[0], op[1], op[2]};
    allreduce_n<3>(a, o, sm, phase);
    v[0] = a[0];
    v[1] = a[1];
    v[2] = a[2];
}

__device__ __forceinline__ uint64_t wdec(uint32_t x) { return x == 0xFFFFFFFFu ? (1ull << 32) : (uint64_t)x; }

// trunc(e * 2^32) for e in [0, 1], ENCODED as u32 (2^32 -> 0xFFFFFFFF): e * 2^32 is exact and
// cvt.rzi.u32.f32 saturates, so e = 1 gives 0xFFFFFFFF and every e < 1 its exact truncation
// (<= 2^32 - 2^8); 0, -0 and subnormals give 0 (= __float2ull_rz(e * 2^32) for all e in [0, 1]).
__device__ __forceinline__ uint32_t f2w(float e) { return __float2uint_rz(__fmul_rn(e, 4294967296.0f)); }
// sum of 8 encoded weights as the true 64-bit sum
__device__ __forceinline__ unsigned long long wsum8(const uint32_t e[8]) {
    const unsigned long long s = ((unsigned long long)e[0] + e[1] + e[2]) + ((unsigned long long)e[3] + e[4] + e[5]) +
                                 ((unsigned long long)e[6] + e[7]);
    const uint32_t mn = min(min(min(~e[0], ~e[1]), min(~e[2], ~e[3])), min(min(~e[4], ~e[5]), min(~e[6], ~e[7])));
    if (mn != 0u) return s;                     // no 0xFFFFFFFF code in the vector (the usual case)
    uint32_t tops = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) tops += e[j] == 0xFFFFFFFFu ? 1u : 0u;
    return s + tops;
}

// r = max(x*S - y*T, 0) for ENCODED 33-bit weights x, y (0xFFFFFFFF = 2^32) and S, T < 2^64 with
// x*S, y*T < 2^95: three 32-bit limbs (r2:r1:r0) with carry chains (exact; DESIGN "Bit-exact
// sampling": r_v = max(w_v Zq - qw_v Z, 0)).
struct R96 {
    uint32_t r0, r1, r2;
};
__device__ __forceinline__ R96 resid96(uint32_t x, bool xtop, uint64_t S, uint32_t y, bool ytop, uint64_t T) {
    const uint32_t s0 = (uint32_t)S, s1 = (uint32_t)(S >> 32), t0 = (uint32_t)T, t1 = (uint32_t)(T >> 32);
    // x = 2^32 is encoded 0xFFFFFFFF: x*S = enc*S + S (the +S is added at limb 0)
    const uint32_t xs0 = xtop ? s0 : 0u, xs1 = xtop ? s1 : 0u;
    const uint32_t yt0 = ytop ? t0 : 0u, yt1 = ytop ? t1 : 0u;
    uint32_t a0, a1, a2, b0, b1, b2;
    asm("{\n\t"
        "mul.lo.u32 %0, %6, %7;\n\t"
        "mul.hi.u32 %1, %6, %7;\n\t"
        "mad.lo.cc.u32 %1, %6, %8, %1;\n\t"
        "madc.hi.u32 %2, %6, %8, 0;\n\t"
        "add.cc.u32 %0, %0, %9;\n\t"
        "addc.cc.u32 %1, %1, %10;\n\t"
        "addc.u32 %2, %2, 0;\n\t"
        "mul.lo.u32 %3, %11, %12;\n\t"
        "mul.hi.u32 %4, %11, %12;\n\t"
        "mad.lo.cc.u32 %4, %11, %13, %4;\n\t"
        "madc.hi.u32 %5, %11, %13, 0;\n\t"
        "add.cc.u32 %3, %3, %14;\n\t"
        "addc.cc.u32 %4, %4, %15;\n\t"
        "addc.u32 %5, %5, 0;\n\t"
        "}"
        : "=&r"(a0), "=&r"(a1), "=&r"(a2), "=&r"(b0), "=&r"(b1), "=&r"(b2)
        : "r"(x), "r"(s0), "r"(s1), "r"(xs0), "r"(xs1), "r"(y), "r"(t0), "r"(t1), "r"(yt0), "r"(yt1));
    uint32_t d0, d1, d2;
    asm("{\n\t"
        "sub.cc.u32 %0, %3, %6;\n\t"
        "subc.cc.u32 %1, %4, %7;\n\t"
        "subc.u32 %2, %5, %8;\n\t"
        "}"
        : "=r"(d0), "=r"(d1), "=r"(d2)
        : "r"(a0), "r"(a1), "r"(a2), "r"(b0), "r"(b1), "r"(b2));
    const uint32_t keep = (uint32_t)((int32_t)d2 >> 31) ^ 0xFFFFFFFFu;   // 0 if A < B
    return R96{d0 & keep, d1 & keep, d2 & keep};
}
__device__ __forceinline__ int r96_bitlen(const R96& r) {
    return r.r2 ? 96 - __clz(r.r2) : (r.r1 ? 64 - __clz(r.r1) : 32 - __clz(r.r0));
}
// low 32 bits of r >> t, 0 <= t < 64
__device__ __forceinline__ uint32_t r96_shr32(const R96& r, int t) {
    return t < 32 ? __funnelshift_rc(r.r0, r.r1, t) : __funnelshift_rc(r.r1, r.r2, t - 32);
}

// 3 CTAs per SM (registers and 65 KB of shared memory each); with bf16 drafts 49 KB, so 4 fit
// when the kernel stays within 64 registers (more clusters in flight: the kernel is latency-bound)
#ifndef RS_MSS_MINB_BF16
#define RS_MSS_MINB_BF16 4
#endif
template <int DT, int DQ, typename CA>   // DT: logits dtype, DQ: draft-probability dtype (bf16 values are exact fp32)
__global__ void __launch_bounds__(kMssThreads, DQ == RS_DTYPE_BF16 ? RS_MSS_MINB_BF16 : 3)
mss_accept_kernel(const void* __restrict__ logits, const void* __restrict__ draft,
                  const int32_t* __restrict__ draft_row, const int32_t* __restrict__ parent, const int32_t* __restrict__ token,
                  const int32_t* __restrict__ tree_off, const int64_t* __restrict__ gid, int V, float inv_tau,
                  uint64_t seed, uint64_t step, int32_t* __restrict__ acc_out, int32_t* __restrict__ path_out,
                  int32_t* __restrict__ bonus_out, int32_t* __restrict__ flags_out, bool logits_vec_ok,
                  bool draft_vec_ok, const __grid_constant__ CA ca) {
    __shared__ Smem sm;
    __shared__ MssSmem ms;
    extern __shared__ __align__(16) uint4 mss_dyn[];
    const uint32_t cs = cluster_size();
    const uint32_t crank = cluster_rank();
    const int b = blockIdx.x / cs;
    const int tid = threadIdx.x;
    const bool leader = crank == 0;
    const int off = tree_off[b];
    const int T = tree_off[b + 1] - off;
    int32_t* pth = path_out + (int64_t)b * RS_MAX_TREE;
    int phase = 0;
    if (leader && tid < RS_MAX_TREE) pth[tid] = -1;
    bool bad_node = !(T >= 1 && T <= RS_MAX_TREE);
    if (tid == 0) sm.kids = 0ull;
    __syncthreads();
    if (!bad_node && tid < T) {
        const int pp = parent[off + tid];
        const int tk = token[off + tid];
        sm.parent[tid] = pp;
        sm.token[tid] = tk;
        bad_node = tid == 0 ? pp != -1 : !(pp >= 0 && pp < tid && tk >= 0 && tk < V);
        if (!bad_node && tid > 0) atomicOr(&sm.kids, 1ull << pp);
        sm.qrow[tid] = draft_row ? draft_row[off + tid] : off + tid;
    }
    __syncthreads();
    // with a row map, every node with children needs its draft row (else the tree is malformed)
    if (draft_row && !bad_node && tid < T && ((sm.kids >> tid) & 1ull) && draft_row[off + tid] < 0) bad_node = true;
    if (__syncthreads_or(bad_node)) {
        if (leader && tid == 0) { acc_out[b] = 0; bonus_out[b] = -1; flags_out[b] = RS_FLAG_MALFORMED; }
        if constexpr (CA::kOn) fused_commit(ca, b, 0, sm);   // accepted_len 0: new_len only
        return;
    }
    const int64_t g = gid[b];
    const int nvec = (V + 7) / 8;
    const int per = (nvec + (int)cs - 1) / (int)cs;
    const int vbeg = min(nvec, (int)crank * per), vend = min(nvec, vbeg + per);
    uint32_t* wsl = reinterpret_cast<uint32_t*>(mss_dyn);   // [per * 8]
    // draft: qw words [per * 8] (fp32 drafts), or the raw bf16 values [per * 8] (bf16 drafts: half
    // the shared memory, qw = trunc(q * 2^32) recomputed where used)
    uint32_t* qsl = wsl + (size_t)per * 8;
    uint16_t* qsl16 = reinterpret_cast<uint16_t*>(qsl);
    uint8_t* vex = reinterpret_cast<uint8_t*>(qsl) + (size_t)per * 8 * (DQ == RS_DTYPE_BF16 ? 2 : 4);   // [per]
    int c = 0, a = 0, bonus = -1, flags = 0;
    bool bonus_mine = leader;
    if (leader && tid == 0) pth[0] = 0;
    if (tid == 0) sm.path_s[0] = 0;
    __syncthreads();
    // owner CTA: publish the current (w, qw) of the children x > after of node c (tid < T)
    auto publish = [&](int after, bool resid_state) {
        __syncthreads();   // this CTA's shared-memory weights are complete
        const int x = tid;
        if (x < T && x > after && sm.parent[x] == c) {
            const int tk = sm.token[x];
            const int ti = tk >> 3;
            if (ti >= vbeg && ti < vend) {
                const int lo = tk - vbeg * 8;
                ms.childw[x] = resid_state ? (uint64_t)wsl[lo] : wdec(wsl[lo]);
                ms.childq[x] = DQ == RS_DTYPE_BF16 ? wdec(f2w(__uint_as_float((uint32_t)qsl16[lo] << 16)))
                                                   : wdec(qsl[lo]);
            }
        }
    };
    for (;;) {
        const RowView lv{logits, (int64_t)(off + c), V, DT, logits_vec_ok};
        // reading Z29: the draft row is read only for a node with children (a leaf's q is unused:
        // no child tests, no residual; its bonus is drawn from the target weights alone)
        const bool with_q = (sm.kids >> c) & 1ull;   // (read here: no register held across the walk)
        const RowView qv{draft, (int64_t)sm.qrow[c], V, DQ, draft_vec_ok};   // (the row from shared memory)
        // ---- pass L: the row from HBM into shared memory; max, validity, Zq
        // (bf16 logits stay packed: the first 16 bytes of the vector's w words hold the 8 raw
        // values until pass E expands them)
        unsigned long long red[3] = {0, 0, 0};
        {
            float fmx = -INFINITY;
            uint32_t amag = 0, qbad = 0;
            unsigned long long zq = 0;
            for (int i0 = vbeg + tid; i0 < vend; i0 += kMssLUnroll * kMssThreads) {
                Raw8 x[kMssLUnroll], q[kMssLUnroll];
#pragma unroll
                for (int u = 0; u < kMssLUnroll; ++u) {
                    const int i = i0 + u * kMssThreads;
                    if (i < vend) {
                        x[u] = load_raw(lv, i);
                        q[u] = with_q ? load_raw(qv, i) : Raw8{make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
                    }
                }
#pragma unroll
                for (int u = 0; u < kMssLUnroll; ++u) {
                    const int i = i0 + u * kMssThreads;
                    if (i >= vend) continue;
                    const bool full = (i + 1) * 8 <= V;
                    uint4* wp = reinterpret_cast<uint4*>(wsl + (size_t)(i - vbeg) * 8);
                    {   // the draft row (zeros at a leaf: its row is not read, Z29)
                        uint32_t qb[8];
                        if (DQ == RS_DTYPE_BF16) {   // bf16 -> the fp32 bit pattern of the same value
                            const uint32_t h4[4] = {q[u].a.x, q[u].a.y, q[u].a.z, q[u].a.w};
    #pragma unroll
                            for (int k = 0; k < 4; ++k) { qb[2 * k] = h4[k] << 16; qb[2 * k + 1] = h4[k] & 0xFFFF0000u; }
                        } else {
                            qb[0] = q[u].a.x; qb[1] = q[u].a.y; qb[2] = q[u].a.z; qb[3] = q[u].a.w;
                            qb[4] = q[u].b.x; qb[5] = q[u].b.y; qb[6] = q[u].b.z; qb[7] = q[u].b.w;
                        }
                        uint32_t qe[8], qu[8];
                        if (full) {
    #pragma unroll
                            for (int j = 0; j < 8; ++j) qu[j] = qb[j];
                        } else {
    #pragma unroll
                            for (int j = 0; j < 8; ++j) qu[j] = i * 8 + j < V ? qb[j] : 0u;
                        }
    #pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            // a probability: bits <= 1.0f, or -0
                            qbad |= (qu[j] > 0x3F800000u && qu[j] != 0x80000000u) ? 1u : 0u;
                            qe[j] = f2w(__uint_as_float(qu[j]));
                        }
                        zq += wsum8(qe);
                        if (DQ == RS_DTYPE_BF16) {   // the raw values back (padding lanes zero)
                            *reinterpret_cast<uint4*>(qsl16 + (size_t)(i - vbeg) * 8) =
                                make_uint4((qu[0] >> 16) | (qu[1] & 0xFFFF0000u), (qu[2] >> 16) | (qu[3] & 0xFFFF0000u),
                                           (qu[4] >> 16) | (qu[5] & 0xFFFF0000u), (qu[6] >> 16) | (qu[7] & 0xFFFF0000u));
                        } else {
                            uint4* qp = reinterpret_cast<uint4*>(qsl + (size_t)(i - vbeg) * 8);
                            qp[0] = make_uint4(qe[0], qe[1], qe[2], qe[3]);
                            qp[1] = make_uint4(qe[4], qe[5], qe[6], qe[7]);
                        }
                    }
                    if (DT == RS_DTYPE_BF16) {
                        uint32_t w4[4] = {x[u].a.x, x[u].a.y, x[u].a.z, x[u].a.w};
                        uint32_t wm[4] = {w4[0], w4[1], w4[2], w4[3]};   // for the validity check
                        if (!full) {
#pragma unroll
                            for (int j = 0; j < 8; ++j)   // padding: -inf (weight 0), not checked
                                if (i * 8 + j >= V) {
                                    const uint32_t keepm = (j & 1) ? 0x0000FFFFu : 0xFFFF0000u;
                                    w4[j >> 1] = (w4[j >> 1] & keepm) | ((j & 1) ? 0xFF800000u : 0x0000FF80u);
                                    wm[j >> 1] &= keepm;
                                }
                        }
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint32_t wv = w4[k];
                            amag = __vmaxu2(amag, wm[k] & 0x7FFF7FFFu);
                            fmx = fmaxf(fmx, fmaxf(__uint_as_float(wv << 16), __uint_as_float(wv & 0xFFFF0000u)));
                        }
                        wp[0] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
                    } else {
                        uint32_t lw[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const float l = (full || i * 8 + j < V) ? raw_elem(x[u], DT, j) : -INFINITY;
                            qbad |= ((full || i * 8 + j < V) && !isfinite(l)) ? 1u : 0u;
                            fmx = fmaxf(fmx, l);
                            lw[j] = __float_as_uint(l);
                        }
                        wp[0] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
                        wp[1] = make_uint4(lw[4], lw[5], lw[6], lw[7]);
                    }
                }
            }
            // bf16: magnitude bits >= 0x7F80 <=> inf or NaN (padding lanes are not in amag)
            const bool lbad = DT == RS_DTYPE_BF16 ? ((amag & 0xFFFFu) >= 0x7F80u || (amag >> 16) >= 0x7F80u) : false;
            red[0] = fkey(fmx);
            red[1] = (qbad || lbad) ? 1ull : 0ull;
            red[2] = zq;
        }
        {
            const int ops[3] = {OP_MAX, OP_OR, OP_SUM};
            allreduce3(red, ops, sm, phase);
        }
        if (red[1]) { flags |= RS_FLAG_NONFINITE; break; }
        const float m = fkey_inv((uint32_t)red[0]);
        const uint64_t Zq = red[2];
        // ---- pass E (shared memory): w_v = trunc(exp_spec((l_v - m) * inv_tau) * 2^32) and Z
        // (the inverse-CDF tile sums are built only for the bonus draw, below)
        unsigned long long zs = 0, dummy = 0;
        for (int base = vbeg; base < vend; base += kMssThreads) {
            const int i = base + tid;
            unsigned long long s8 = 0;
            if (i < vend) {
                uint4* wp = reinterpret_cast<uint4*>(wsl + (size_t)(i - vbeg) * 8);
                uint32_t lw[8];
                if (DT == RS_DTYPE_BF16) {
                    const uint4 a0 = wp[0];
                    const uint32_t w4[4] = {a0.x, a0.y, a0.z, a0.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) { lw[2 * k] = w4[k] << 16; lw[2 * k + 1] = w4[k] & 0xFFFF0000u; }
                } else {
                    const uint4 a0 = wp[0], a1 = wp[1];
                    lw[0] = a0.x; lw[1] = a0.y; lw[2] = a0.z; lw[3] = a0.w;
                    lw[4] = a1.x; lw[5] = a1.y; lw[6] = a1.z; lw[7] = a1.w;
                }
                uint32_t en[8];
#pragma unroll
                for (int j = 0; j < 8; ++j)   // w = trunc(exp_spec((l - m) * inv_tau) * 2^32)
                    en[j] = rs::exp_spec_w32(__fmul_rn(__fsub_rn(__uint_as_float(lw[j]), m), inv_tau));
                s8 = wsum8(en);
                wp[0] = make_uint4(en[0], en[1], en[2], en[3]);
                wp[1] = make_uint4(en[4], en[5], en[6], en[7]);
            }
            zs += s8;
        }
        publish(c, false);
        allreduce2(zs, OP_SUM, dummy, OP_OR, sm, phase);   // (cluster barrier: published values visible)
        uint64_t Z = zs;
        bool resid = false;
        int rank = 0, next = -1;
        for (int x = c + 1; x < T && next < 0; ++x) {
            if (sm.parent[x] != c) continue;
            const int tk = sm.token[x];
            if (tid == 0) {
                const uint32_t owner = (uint32_t)((tk >> 3) / per);
                const uint64_t wt = ld_dsmem_u64(&ms.childw[x], owner);
                const uint64_t qw = ld_dsmem_u64(&ms.childq[x], owner);
                const uint32_t U = rs::uniform_word(seed, step, g, (uint32_t)rank, (uint32_t)c);
                const bool acc = qw == 0 ? wt > 0 : ((u128)U * ((u128)qw * Z)) < (((u128)wt * Zq) << 32);
                sm.bcast_i = acc ? 1 : 0;
            }
            __syncthreads();
            const bool accepted = sm.bcast_i != 0;
            __syncthreads();
            if (accepted) { next = x; break; }
            ++rank;
            // pass A: r_v in 128 bits, once; stored per vector as r >> t with t in vex
            unsigned long long bl = 0, dummy2 = 0;
            for (int i = vbeg + tid; i < vend; i += kMssThreads) {
                uint4* wp = reinterpret_cast<uint4*>(wsl + (size_t)(i - vbeg) * 8);
                const uint4 a0 = wp[0], a1 = wp[1];
                const uint32_t ww[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                uint32_t qq[8];
                if (DQ == RS_DTYPE_BF16) {
                    const uint4 h = *reinterpret_cast<const uint4*>(qsl16 + (size_t)(i - vbeg) * 8);
                    const uint32_t h4[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        qq[2 * k] = f2w(__uint_as_float(h4[k] << 16));
                        qq[2 * k + 1] = f2w(__uint_as_float(h4[k] & 0xFFFF0000u));
                    }
                } else {
                    const uint4* qp = reinterpret_cast<const uint4*>(qsl + (size_t)(i - vbeg) * 8);
                    const uint4 b0 = qp[0], b1 = qp[1];
                    qq[0] = b0.x; qq[1] = b0.y; qq[2] = b0.z; qq[3] = b0.w;
                    qq[4] = b1.x; qq[5] = b1.y; qq[6] = b1.z; qq[7] = b1.w;
                }
                R96 r[8];
                R96 ro{0, 0, 0};   // bitlen(max_j r_j) = bitlen(OR_j r_j)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    r[j] = resid96(ww[j], !resid && ww[j] == 0xFFFFFFFFu, Zq, qq[j], qq[j] == 0xFFFFFFFFu, Z);
                    ro.r0 |= r[j].r0;
                    ro.r1 |= r[j].r1;
                    ro.r2 |= r[j].r2;
                }
                const int vb = r96_bitlen(ro);
                bl = bl > (unsigned long long)vb ? bl : (unsigned long long)vb;
                if (vb == 0) {
                    vex[i - vbeg] = 0xFF;                // all-zero vector: old words kept
                } else {
                    const int t = vb > 32 ? vb - 32 : 0;
                    vex[i - vbeg] = (uint8_t)t;
                    uint32_t mt[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) mt[j] = r96_shr32(r[j], t);
                    wp[0] = make_uint4(mt[0], mt[1], mt[2], mt[3]);
                    wp[1] = make_uint4(mt[4], mt[5], mt[6], mt[7]);
                }
            }
            allreduce2(bl, OP_MAX, dummy2, OP_OR, sm, phase);
            if (bl != 0) {
                // pass B: w <- (r >> t) >> (s - t) = r >> s, s = max(0, bitlen - 32); Z, tile sums
                const int sh = (int)bl > 32 ? (int)bl - 32 : 0;
                unsigned long long zn = 0, dummy3 = 0;
                for (int base = vbeg; base < vend; base += kMssThreads) {
                    const int i = base + tid;
                    unsigned long long s8 = 0;
                    if (i < vend) {
                        uint4* wp = reinterpret_cast<uint4*>(wsl + (size_t)(i - vbeg) * 8);
                        const int t = vex[i - vbeg];
                        uint32_t wn[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                        if (t != 0xFF) {
                            const uint4 a0 = wp[0], a1 = wp[1];
                            const uint32_t ww[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                            const int d = sh - t;
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                wn[j] = d >= 32 ? 0u : (ww[j] >> d);
                                s8 += wn[j];
                            }
                        }
                        wp[0] = make_uint4(wn[0], wn[1], wn[2], wn[3]);
                        wp[1] = make_uint4(wn[4], wn[5], wn[6], wn[7]);
                    }
                    zn += s8;
                }
                resid = true;
                publish(x, true);
                allreduce2(zn, OP_SUM, dummy3, OP_OR, sm, phase);   // (cluster barrier: visible)
                Z = zn;
            }
            __syncthreads();
        }
        if (next < 0) {
            const uint32_t U2 = rs::uniform_word(seed, step, g, 0xFFFFFFFFu, (uint32_t)c);
            const uint64_t t = (uint64_t)(((u128)U2 * Z) >> 32);
            const bool rs_ = resid;
            // per-tile sums of the current weights (this CTA's slice), then the inverse CDF
            clear_tiles(sm);
            for (int base = vbeg; base < vend; base += kMssThreads) {
                const int i = base + tid;
                unsigned long long s8 = 0;
                if (i < vend) {
                    const uint4* wp = reinterpret_cast<const uint4*>(wsl + (size_t)(i - vbeg) * 8);
                    const uint4 a0 = wp[0], a1 = wp[1];
                    const uint32_t ww[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                    if (rs_) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) s8 += ww[j];
                    } else {
                        s8 = wsum8(ww);
                    }
                }
                tile_add(sm, (base - vbeg) / kMssThreads, s8);
            }
            bonus = draw_bonus(sm, phase, t, vbeg, vend, V, bonus_mine, [&](int i, uint64_t w8[8]) {
                const uint4* wp = reinterpret_cast<const uint4*>(wsl + (size_t)(i - vbeg) * 8);
                const uint4 a0 = wp[0], a1 = wp[1];
                const uint32_t ww[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
                for (int j = 0; j < 8; ++j) w8[j] = rs_ ? (uint64_t)ww[j] : wdec(ww[j]);
            });
            break;
        }
        c = next;
        ++a;
        if (leader && tid == 0) pth[a] = c;
        if (tid == 0) sm.path_s[a] = c;
        __syncthreads();
    }
    if (tid == 0) {
        if (leader) {
            acc_out[b] = a;
            flags_out[b] = flags;
            if (flags & RS_FLAG_NONFINITE) bonus_out[b] = -1;
        }
        if (!(flags & RS_FLAG_NONFINITE) && bonus_mine) bonus_out[b] = bonus;
    }
    if constexpr (CA::kOn) fused_commit(ca, b, a, sm);
    // no final cluster barrier: every DSMEM access (pushes, the child tests' reads of published
    // weights) is followed in every CTA by at least one cluster barrier (the next pass's reduction or
    // the bonus draw's exchange), so no CTA touches a peer's shared memory after the peer exits
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

extern "C" size_t rs_tree_accept_workspace_bytes(int32_t mode, int32_t B, int32_t V) {
    (void)mode; (void)B; (void)V;
    return 0;   // MSS keeps the residual on chip (mss_accept_kernel); no mode needs workspace
}

// per CTA: w and qw words (64 B per 8-token vector) + one residual shift byte per vector
static size_t mss_smem_bytes(int nvec, int cs, bool qbf) {
    const size_t per = (size_t)((nvec + cs - 1) / cs);
    return (per * (qbf ? 49 : 65) + 15) / 16 * 16;
}

// MSS launch: cluster size = 16 (non-portable) when the device can co-schedule it, else 8, and
// never more CTAs than give every CTA >= 256 vectors; dynamic shared memory = per * 64 bytes.
template <typename CA>
static rs_status launch_mss(const CA& ca, bool bf, bool qbf, const void* logits, const void* draft,
                            const int32_t* draft_row, const int32_t* parent,
                            const int32_t* token, const int32_t* tree_off, const int64_t* gid, int B, int V,
                            float inv_tau, uint64_t seed, uint64_t step, int32_t* acc, int32_t* path, int32_t* bonus,
                            int32_t* flags, bool lvec, bool dvec, cudaStream_t st) {
    auto kern = bf ? (qbf ? mss_accept_kernel<RS_DTYPE_BF16, RS_DTYPE_BF16, CA> : mss_accept_kernel<RS_DTYPE_BF16, RS_DTYPE_F32, CA>)
                   : (qbf ? mss_accept_kernel<RS_DTYPE_F32, RS_DTYPE_BF16, CA> : mss_accept_kernel<RS_DTYPE_F32, RS_DTYPE_F32, CA>);
    const int nvec = (V + 7) / 8;
    static int max_cs = 0;            // 16 if a 16-CTA cluster of this kernel can be resident, else 8
    static size_t attr_smem[4] = {0, 0, 0, 0};
    int cs = 1;
    while (cs < 16 && nvec / (cs * 2) >= kMssThreads) cs *= 2;
#ifdef RS_MSS_CS
    cs = cs > RS_MSS_CS ? RS_MSS_CS : cs;   // (profiling variant: smaller clusters)
#endif
    const size_t smem = mss_smem_bytes(nvec, cs, qbf);
    size_t& cur = attr_smem[(bf ? 0 : 1) + (qbf ? 2 : 0)];
    if (cur < smem) {
        RS_REQUIRE(smem <= 200 * 1024, RS_ERR_UNSUPPORTED, "rs_tree_accept: V=%d too large for MSS", V);
        RS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cur = smem;
    }
    static bool nonportable[4] = {false, false, false, false};
    if (!nonportable[(bf ? 0 : 1) + (qbf ? 2 : 0)]) {   // per template instance
        nonportable[(bf ? 0 : 1) + (qbf ? 2 : 0)] = true;
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaGetLastError();
    }
    if (max_cs == 0) {
        max_cs = 8;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3(16);
            q.blockDim = dim3(kMssThreads);
            q.dynamicSmemBytes = mss_smem_bytes(nvec, 16, qbf);
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = 16;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            q.attrs = qa;
            q.numAttrs = 1;
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, kern, &q) == cudaSuccess && n > 0) max_cs = 16;
        }
        cudaGetLastError();
    }
    if (cs > max_cs) {
        cs = max_cs;
        const size_t sm2 = mss_smem_bytes(nvec, cs, qbf);
        if (cur < sm2) {
            RS_REQUIRE(sm2 <= 200 * 1024, RS_ERR_UNSUPPORTED, "rs_tree_accept: V=%d too large for MSS", V);
            RS_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
            cur = sm2;
        }
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(B * cs));
    cfg.blockDim = dim3(kMssThreads);
    cfg.dynamicSmemBytes = mss_smem_bytes(nvec, cs, qbf);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    RS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, logits, draft, draft_row, parent, token, tree_off, gid, V, inv_tau,
                                     seed, step,
                                     acc, path, bonus, flags, lvec, dvec, ca));
    return RS_OK;
}

extern "C" rs_status rs_tree_accept_ex(int32_t mode, const void* logits, int32_t logits_dtype,
                                       const void* draft_probs, int32_t draft_dtype, const int32_t* parent,
                                       const int32_t* token, const int32_t* tree_off,
                                       const int64_t* gid, int32_t B, int32_t V, float temperature,
                                       uint64_t seed, uint64_t step, int32_t* accepted_len,
                                       int32_t* path, int32_t* bonus_token, int32_t* status_flags,
                                       void* ws, size_t ws_bytes, void* stream);

extern "C" rs_status rs_tree_accept(int32_t mode, const void* logits, int32_t logits_dtype,
                                    const float* draft_probs, const int32_t* parent,
                                    const int32_t* token, const int32_t* tree_off,
                                    const int64_t* gid, int32_t B, int32_t V, float temperature,
                                    uint64_t seed, uint64_t step, int32_t* accepted_len,
                                    int32_t* path, int32_t* bonus_token, int32_t* status_flags,
                                    void* ws, size_t ws_bytes, void* stream) {
    return rs_tree_accept_ex(mode, logits, logits_dtype, draft_probs, RS_DTYPE_F32, parent, token, tree_off, gid, B,
                             V, temperature, seed, step, accepted_len, path, bonus_token, status_flags, ws, ws_bytes,
                             stream);
}

template <typename CA>
static rs_status accept_launch(const CA& ca, int32_t mode, const void* logits, int32_t logits_dtype,
                               const void* draft_probs, int32_t draft_dtype, const int32_t* draft_row,
                               const int32_t* parent,
                               const int32_t* token, const int32_t* tree_off, const int64_t* gid, int32_t B,
                               int32_t V, float temperature, uint64_t seed, uint64_t step, int32_t* accepted_len,
                               int32_t* path, int32_t* bonus_token, int32_t* status_flags, void* ws, size_t ws_bytes,
                               void* stream) {
    RS_REQUIRE(mode == RS_ACCEPT_GREEDY || mode == RS_ACCEPT_SAMPLE_DELTA ||
                   mode == RS_ACCEPT_SAMPLE_MSS,
               RS_ERR_INVALID_ARG, "rs_tree_accept: bad mode %d", mode);
    RS_REQUIRE(logits_dtype == RS_DTYPE_BF16 || logits_dtype == RS_DTYPE_F32, RS_ERR_INVALID_ARG,
               "rs_tree_accept: bad logits dtype %d", logits_dtype);
    RS_REQUIRE(draft_dtype == RS_DTYPE_BF16 || draft_dtype == RS_DTYPE_F32, RS_ERR_INVALID_ARG,
               "rs_tree_accept: bad draft dtype %d", draft_dtype);
    RS_REQUIRE(B >= 0 && V >= 1, RS_ERR_INVALID_ARG, "rs_tree_accept: B=%d V=%d", B, V);
    RS_REQUIRE((mode == RS_ACCEPT_SAMPLE_MSS) == (draft_probs != nullptr), RS_ERR_INVALID_ARG,
               "rs_tree_accept: draft_probs must be given for MSS only");
    RS_REQUIRE(mode == RS_ACCEPT_SAMPLE_MSS || draft_row == nullptr, RS_ERR_INVALID_ARG,
               "rs_tree_accept: draft_row is an MSS argument");
    RS_REQUIRE(mode == RS_ACCEPT_GREEDY || temperature > 0.0f, RS_ERR_INVALID_ARG,
               "rs_tree_accept: temperature must be > 0");
    if (B == 0) return RS_OK;
    RS_REQUIRE(logits && parent && token && tree_off && gid && accepted_len && path && bonus_token &&
                   status_flags,
               RS_ERR_INVALID_ARG, "rs_tree_accept: null pointer");
    const size_t need = rs_tree_accept_workspace_bytes(mode, B, V);
    RS_REQUIRE(ws_bytes >= need && (need == 0 || (ws && (reinterpret_cast<uintptr_t>(ws) & 15) == 0)), RS_ERR_WORKSPACE,
               "rs_tree_accept: workspace %zu < %zu bytes (16-byte aligned)", ws_bytes, need);
    // cluster size: enough CTAs per sample that one row streams in ~a microsecond, without
    // exceeding ~2 waves of the GPU when B is large
    const int nvec = (V + 7) / 8;
    int cs = 1;
    while (cs < kMaxCluster && nvec / (cs * 2) >= kThreads * 2 && (int64_t)B * cs * 2 <= 148 * 4) cs *= 2;
    if (RS_ACC_CS == 1 || RS_ACC_CS == 2 || RS_ACC_CS == 4 || RS_ACC_CS == 8) cs = RS_ACC_CS;   // variant builds
    const int per = (nvec + cs - 1) / cs;
    RS_REQUIRE((per + kTileVecs - 1) / kTileVecs <= kMaxTiles, RS_ERR_UNSUPPORTED, "rs_tree_accept: V=%d too large", V);
    const float inv_tau = (mode == RS_ACCEPT_GREEDY) ? 1.0f : 1.0f / temperature;
    const int esz = logits_dtype == RS_DTYPE_BF16 ? 2 : 4;
    const bool lvec = ((reinterpret_cast<uintptr_t>(logits) & 15) == 0) && ((int64_t)V * esz % 16 == 0);
    const bool dvec = draft_probs && ((reinterpret_cast<uintptr_t>(draft_probs) & 15) == 0) &&
                      (V % (draft_dtype == RS_DTYPE_BF16 ? 8 : 4) == 0);
    // -DRS_ACC_PF=1: speculative L2 prefetch of the children rows (greedy). Measured on config 2:
    // 34.7 -> 38.1 us (2.2x the DRAM bytes; the walk is bound by the cluster barriers), so off.
    constexpr int pf = RS_ACC_PF;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(B * cs));
    cfg.blockDim = dim3(kThreads);
    cfg.stream = rs::as_stream(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const bool bf = logits_dtype == RS_DTYPE_BF16;
    if (mode == RS_ACCEPT_SAMPLE_MSS) return launch_mss(ca, bf, draft_dtype == RS_DTYPE_BF16, logits, draft_probs,
                                                        draft_row, parent, token, tree_off, gid, B, V,
                                                        inv_tau, seed, step, accepted_len, path, bonus_token,
                                                        status_flags, lvec, dvec, cfg.stream);
    auto kern = mode == RS_ACCEPT_GREEDY
                    ? (bf ? tree_accept_kernel<RS_ACCEPT_GREEDY, RS_DTYPE_BF16, CA>
                          : tree_accept_kernel<RS_ACCEPT_GREEDY, RS_DTYPE_F32, CA>)
                    : (bf ? tree_accept_kernel<RS_ACCEPT_SAMPLE_DELTA, RS_DTYPE_BF16, CA>
                          : tree_accept_kernel<RS_ACCEPT_SAMPLE_DELTA, RS_DTYPE_F32, CA>);
    RS_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, (int)mode, logits, (int)logits_dtype, static_cast<const float*>(draft_probs), parent, token,
                                     tree_off, gid, (int)V, inv_tau, seed, step, accepted_len, path, bonus_token,
                                     status_flags, lvec, dvec, static_cast<uint32_t*>(need ? ws : nullptr), pf, ca));
    return RS_OK;
}

extern "C" rs_status rs_tree_accept_ex(int32_t mode, const void* logits, int32_t logits_dtype,
                                       const void* draft_probs, int32_t draft_dtype, const int32_t* parent,
                                       const int32_t* token, const int32_t* tree_off,
                                       const int64_t* gid, int32_t B, int32_t V, float temperature,
                                       uint64_t seed, uint64_t step, int32_t* accepted_len,
                                       int32_t* path, int32_t* bonus_token, int32_t* status_flags,
                                       void* ws, size_t ws_bytes, void* stream) {
    rs::bind_device(logits);
    return accept_launch(rs::NoCompact{}, mode, logits, logits_dtype, draft_probs, draft_dtype, nullptr, parent,
                         token, tree_off, gid, B, V, temperature, seed, step, accepted_len, path, bonus_token,
                         status_flags, ws, ws_bytes, stream);
}

extern "C" rs_status rs_tree_accept_compact(int32_t mode, const void* logits, int32_t logits_dtype,
                                            const void* draft_probs, int32_t draft_dtype,
                                            const int32_t* draft_row, const int32_t* parent,
                                            const int32_t* token, const int32_t* tree_off, const int64_t* gid,
                                            int32_t B, int32_t V, float temperature, uint64_t seed, uint64_t step,
                                            int32_t* accepted_len, int32_t* path, int32_t* bonus_token,
                                            int32_t* status_flags, void* ws, size_t ws_bytes,
                                            void* const* k_layers_host, void* const* v_layers_host, int32_t L,
                                            int32_t Hkv, int32_t head_dim, int32_t page_size,
                                            const int32_t* block_table, int32_t max_pages, const int32_t* prefix_len,
                                            int32_t* new_len, int32_t* moves, void* stream) {
    rs::bind_device(logits);
    RS_REQUIRE(L >= 0 && L <= rs::kCompactMaxLayers && Hkv > 0 && page_size > 0 && max_pages >= 0,
               RS_ERR_INVALID_ARG, "rs_tree_accept_compact: bad KV sizes (L=%d, at most %d layers)", L,
               rs::kCompactMaxLayers);
    RS_REQUIRE(head_dim > 0 && head_dim % 8 == 0, RS_ERR_UNSUPPORTED, "rs_tree_accept_compact: head_dim %% 8 != 0");
    if (B == 0) return RS_OK;
    RS_REQUIRE((L == 0 || (k_layers_host && v_layers_host)) && block_table && prefix_len && new_len,
               RS_ERR_INVALID_ARG, "rs_tree_accept_compact: null pointer");
    rs::CompactArgs A;
    for (int i = 0; i < L; ++i) {
        RS_REQUIRE(k_layers_host[i] && v_layers_host[i], RS_ERR_INVALID_ARG,
                   "rs_tree_accept_compact: null layer pointer");
        A.k[i] = k_layers_host[i];
        A.v[i] = v_layers_host[i];
    }
    A.nl = L;
    A.Hkv = Hkv;
    A.d = head_dim;
    A.ps = page_size;
    A.max_pages = max_pages;
    A.block_table = block_table;
    A.prefix_len = prefix_len;
    A.new_len = new_len;
    A.moves = moves;
    return accept_launch(A, mode, logits, logits_dtype, draft_probs, draft_dtype, draft_row, parent, token, tree_off,
                         gid, B, V, temperature, seed, step, accepted_len, path, bonus_token, status_flags, ws,
                         ws_bytes, stream);
}


extern "C" rs_status rs_philox4x32_10(const uint32_t* ctr, int64_t n, const uint32_t* key_host,
                                      uint32_t* out, void* stream) {
    rs::bind_device(ctr);
    RS_REQUIRE(n >= 0 && key_host, RS_ERR_INVALID_ARG, "rs_philox4x32_10: bad args");
    if (n == 0) return RS_OK;
    philox_kernel<<<(unsigned)((n + 255) / 256), 256, 0, rs::as_stream(stream)>>>(
        reinterpret_cast<const uint4*>(ctr), n, make_uint2(key_host[0], key_host[1]),
        reinterpret_cast<uint4*>(out));
    RS_LAUNCH_CHECK();
    return RS_OK;
}

extern "C" rs_status rs_exp_spec(const float* x, int64_t n, float* y, void* stream) {
    rs::bind_device(x);
    RS_REQUIRE(n >= 0, RS_ERR_INVALID_ARG, "rs_exp_spec: n < 0");
    if (n == 0) return RS_OK;
    exp_spec_kernel<<<(unsigned)((n + 255) / 256), 256, 0, rs::as_stream(stream)>>>(x, n, y);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

#ifdef RS_ACC_TRACE
extern "C" int rs_debug_acc_trace(unsigned long long* host, int n_samples) {
    return (int)cudaMemcpyFromSymbol(host, g_acc_trace, sizeof(unsigned long long) * 8 * (size_t)n_samples);
}
#endif
