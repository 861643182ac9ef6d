// a2: tree-verification attention on sm_100a (P:76-80 single-pass tree verification; P:213
// "attention primarily incurs cost due to KVCache loading"). Readings Z1-Z4.
//
// Work unit = (sample b, kv head, M tile of 128 query rows). Query rows of a unit are the
// T_b*g (node, head-in-group) pairs, node-major, padded to 128 (UMMA M = 128). Keys are the
// sample's logical slots 0..P_b+T_b-1 in 64-key blocks = one KV page each.
//
// Persistent kernel, one CTA per SM (grid = plan.n_ctas), warp-specialised:
//   warp 0      TMA producer: Q tile (3-D tensor map, 2 buffers), per block one K and one V
//               page tile (2-D tensor map over [pages*Hkv*64, D], SWIZZLE_128B), 4-stage ring.
//   warp 1      MMA issuer (one thread): S_j = Q K_j^T -> TMEM (2 buffers, 64 fp32 columns);
//               O += P_j V_j -> TMEM (D fp32 columns), tcgen05.mma kind::f16, M=128.
//   warp 2      TMEM allocator.
//   warps 4..7  softmax + epilogue, one query row per thread: tcgen05.ld S, ancestor mask,
//               online softmax in the exp2 domain with lazy (threshold 2^8) rescaling of O in
//               TMEM, P (bf16) -> shared memory in the UMMA K-major SW128 layout, final
//               normalisation and store (or a split-KV partial + combine kernel).
// The schedule (which units/key ranges each CTA processes, split-KV cuts for load balance)
// is built on the host by rs_attn_plan_create from the step's lengths and reused by all layers.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace {

using namespace rs::ptx;

constexpr int kBlockN = 64;      // keys per KV block (= page_size)
constexpr int kM = 128;          // query rows per work item (UMMA M)
constexpr int kStages = 4;
constexpr int kQBufs = 2;
constexpr int kThreads = 256;    // 8 warps
constexpr int kOvhBlocks = 2;    // per-item fixed cost in block units (planning)
constexpr int kMinPart = 4;      // smallest split-KV part, in blocks

struct WorkItem {
    int32_t b, kvh, mtile, blk_begin, blk_end, part;  // part: -1 = direct, else partial slot
};
struct SplitUnit {
    int32_t b, kvh, mtile, n_parts, part_base, pad;
};

template <int D>
struct Cfg {
    static constexpr int kBoxes = D / 64;                    // 64-element (128 B) SW128 boxes
    static constexpr int kQBytes = kM * D * 2;
    static constexpr int kKVBytes = kBlockN * D * 2;         // one of K or V per block
    static constexpr int kStageBytes = 2 * kKVBytes;
    static constexpr int kPBytes = kM * kBlockN * 2;
    static constexpr int kOffQ = 0;
    static constexpr int kOffStage = kOffQ + kQBufs * kQBytes;
    static constexpr int kOffP = kOffStage + kStages * kStageBytes;
    static constexpr int kOffBar = kOffP + 2 * kPBytes;
    static constexpr int kSmemBytes = kOffBar + 256 + 1024;  // + barriers + alignment slack
    static constexpr int kTmemCols = 256;                    // O: D cols, S: 2 x 64 cols
    static constexpr int kColS = D;
};

struct Bars {
    uint64_t q_full[kQBufs], q_empty[kQBufs];
    uint64_t kv_full[kStages], kv_empty[kStages];
    uint64_t s_full[2], s_free[2];
    uint64_t p_full[2], pv_done[2];
    uint64_t o_free;
    uint32_t tmem_base;
};

struct Params {
    const int32_t* cta_off;
    const WorkItem* items;
    float* part_o;      // [n_parts][kM][D] fp32
    float* part_lse;    // [n_parts][kM] fp32 (log2 domain)
    const int32_t* prefix_len;
    const int32_t* tree_off;
    const uint64_t* tree_mask;
    const int32_t* block_table;
    int max_pages;
    int Hq, Hkv, g;
    float scale_log2;   // sm_scale * log2(e)
    __nv_bfloat16* out;
    float* lse;
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
tree_attn_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmV, const Params p) {
    using C = Cfg<D>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Bars* bars = reinterpret_cast<Bars*>(smem + C::kOffBar);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int item_begin = p.cta_off[blockIdx.x];
    const int item_end = p.cta_off[blockIdx.x + 1];

    if (threadIdx.x == 0) {
        for (int i = 0; i < kQBufs; ++i) { mbar_init(&bars->q_full[i], 1); mbar_init(&bars->q_empty[i], 1); }
        for (int i = 0; i < kStages; ++i) { mbar_init(&bars->kv_full[i], 1); mbar_init(&bars->kv_empty[i], 1); }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->s_full[i], 1);
            mbar_init(&bars->s_free[i], 4);
            mbar_init(&bars->p_full[i], 4);
            mbar_init(&bars->pv_done[i], 1);
        }
        mbar_init(&bars->o_free, 4);
        fence_mbar_init();
        prefetch_tmap(&tmQ);
        prefetch_tmap(&tmK);
        prefetch_tmap(&tmV);
    }
    if (warp == 2) tmem_alloc<C::kTmemCols>(&bars->tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem_base;

    if (warp == 0) {
        // ============================ TMA producer ============================
        if (lane == 0) {
            uint32_t J = 0;
            int it = 0;
            for (int w = item_begin; w < item_end; ++w, ++it) {
                const WorkItem wi = p.items[w];
                const int qb = it % kQBufs;
                mbar_wait(&bars->q_empty[qb], ((it / kQBufs) & 1) ^ 1);
                mbar_arrive_expect_tx(&bars->q_full[qb], C::kQBytes);
                const int node0 = p.tree_off[wi.b] + wi.mtile * (kM / p.g);
                uint8_t* qs = smem + C::kOffQ + qb * C::kQBytes;
#pragma unroll
                for (int bx = 0; bx < C::kBoxes; ++bx)
                    tma_load_3d(qs + bx * (kM * 128), &tmQ, &bars->q_full[qb], bx * 64, wi.kvh * p.g, node0);
                const int32_t* bt = p.block_table + (int64_t)wi.b * p.max_pages;
                for (int blk = wi.blk_begin; blk < wi.blk_end; ++blk, ++J) {
                    const int s = J % kStages;
                    mbar_wait(&bars->kv_empty[s], ((J / kStages) & 1) ^ 1);
                    const int page = bt[blk];
                    const int row = (page * p.Hkv + wi.kvh) * kBlockN;
                    uint8_t* ks = smem + C::kOffStage + s * C::kStageBytes;
                    uint8_t* vs = ks + C::kKVBytes;
                    mbar_arrive_expect_tx(&bars->kv_full[s], C::kStageBytes);
#pragma unroll
                    for (int bx = 0; bx < C::kBoxes; ++bx) {
                        tma_load_2d(ks + bx * (kBlockN * 128), &tmK, &bars->kv_full[s], bx * 64, row);
                        tma_load_2d(vs + bx * (kBlockN * 128), &tmV, &bars->kv_full[s], bx * 64, row);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ============================ MMA issuer ============================
        if (lane == 0) {
            constexpr uint32_t idS = idesc_bf16_f32(kM, kBlockN, 0);
            constexpr uint32_t idPV = idesc_bf16_f32(kM, D, 1);
            const uint32_t sbase = smem_u32(smem);
            uint32_t J = 0;
            int it = 0;
            auto issue_pv = [&](uint32_t Jp, bool first, int item_idx) {
                mbar_wait(&bars->p_full[Jp & 1], (Jp >> 1) & 1);
                if (first) mbar_wait(&bars->o_free, (item_idx & 1) ^ 1);
                tc_fence_after();
                const uint32_t pa = sbase + C::kOffP + (Jp & 1) * C::kPBytes;
                const uint32_t va = sbase + C::kOffStage + (Jp % kStages) * C::kStageBytes + C::kKVBytes;
#pragma unroll
                for (int kk = 0; kk < kBlockN / 16; ++kk) {
                    uint64_t ad = smem_desc_sw128(pa + kk * 32, 16, 1024);
                    uint64_t bd = smem_desc_sw128(va + kk * 2048, kBlockN * 128, 1024);
                    umma_f16(tmem, ad, bd, idPV, (first && kk == 0) ? 0u : 1u);
                }
                umma_commit(&bars->pv_done[Jp & 1]);
                umma_commit(&bars->kv_empty[Jp % kStages]);
            };
            for (int w = item_begin; w < item_end; ++w, ++it) {
                const WorkItem wi = p.items[w];
                const int qb = it % kQBufs;
                const int nblk = wi.blk_end - wi.blk_begin;
                mbar_wait(&bars->q_full[qb], (it / kQBufs) & 1);
                const uint32_t qa = sbase + C::kOffQ + qb * C::kQBytes;
                for (int j = 0; j < nblk; ++j) {
                    const uint32_t Jj = J + j;
                    const int s = Jj % kStages;
                    mbar_wait(&bars->kv_full[s], (Jj / kStages) & 1);
                    mbar_wait(&bars->s_free[Jj & 1], ((Jj >> 1) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t ka = sbase + C::kOffStage + s * C::kStageBytes;
                    const uint32_t sd = tmem + C::kColS + (Jj & 1) * kBlockN;
#pragma unroll
                    for (int k = 0; k < D / 16; ++k) {
                        const int bx = k >> 2, within = (k & 3) * 32;
                        uint64_t ad = smem_desc_sw128(qa + bx * (kM * 128) + within, 16, 1024);
                        uint64_t bd = smem_desc_sw128(ka + bx * (kBlockN * 128) + within, 16, 1024);
                        umma_f16(sd, ad, bd, idS, k > 0 ? 1u : 0u);
                    }
                    umma_commit(&bars->s_full[Jj & 1]);
                    if (j == nblk - 1) umma_commit(&bars->q_empty[qb]);
                    if (j >= 1) issue_pv(Jj - 1, j - 1 == 0, it);
                }
                issue_pv(J + nblk - 1, nblk == 1, it);
                J += nblk;
            }
        }
    } else if (warp >= 4) {
        // ============================ softmax + epilogue ============================
        const int wq = warp - 4;                 // TMEM sub-partition == warp % 4
        const int r = wq * 32 + lane;            // query row within the tile
        const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
        uint32_t J = 0;
        int it = 0;
        for (int w = item_begin; w < item_end; ++w, ++it) {
            const WorkItem wi = p.items[w];
            const int b = wi.b;
            const int P = p.prefix_len[b];
            const int off = p.tree_off[b];
            const int T = p.tree_off[b + 1] - off;
            const int rows = min(kM, T * p.g - wi.mtile * kM);
            const bool warp_active = wq * 32 < rows;
            const bool row_valid = r < rows;
            const int grow = wi.mtile * kM + r;          // row within the unit
            const int node = grow / p.g;
            const uint64_t mask = row_valid ? p.tree_mask[off + node] : 0ull;
            const int key_end = P + T;                   // keys >= key_end do not exist
            float m_run = -INFINITY, l_run = 0.0f;
            const int nblk = wi.blk_end - wi.blk_begin;
            for (int j = 0; j < nblk; ++j) {
                const uint32_t Jj = J + j;
                const int blk = wi.blk_begin + j;
                const int kbase = blk * kBlockN;
                mbar_wait(&bars->s_full[Jj & 1], (Jj >> 1) & 1);
                tc_fence_after();
                // sr: raw S bits -> masked S (float bits) -> packed bf16 P in sr[0..31]
                uint32_t sr[64];
                if (warp_active) {
                    const uint32_t sa = tmem + lane_base + C::kColS + (Jj & 1) * kBlockN;
                    tmem_ld32(sa, reinterpret_cast<uint32_t(&)[32]>(sr[0]));
                    tmem_ld32(sa + 32, reinterpret_cast<uint32_t(&)[32]>(sr[32]));
                    tmem_wait_ld();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->s_free[Jj & 1]);
                if (warp_active) {
                    // ancestor mask (only blocks that reach the tree slots need it)
                    float mx = -INFINITY;
                    if (kbase + kBlockN <= P) {
#pragma unroll
                        for (int c = 0; c < 64; ++c) mx = fmaxf(mx, __uint_as_float(sr[c]));
                    } else {
#pragma unroll
                        for (int c = 0; c < 64; ++c) {
                            const int key = kbase + c;
                            const int t = key - P;
                            bool ok = key < P || (key < key_end && ((mask >> (t & 63)) & 1ull));
                            sr[c] = ok ? sr[c] : 0xFF800000u;   // -inf
                            mx = fmaxf(mx, __uint_as_float(sr[c]));
                        }
                    }
                    const float m_blk = mx * p.scale_log2;
                    bool need_o = false;
                    float alpha = 1.0f;
                    if (m_blk > m_run + 8.0f) {          // lazy rescale (values stay <= 2^8)
                        alpha = ex2(m_run - m_blk);      // m_run = -inf -> 0
                        need_o = (j > 0) && (m_run != -INFINITY);
                        l_run *= alpha;
                        m_run = m_blk;
                    }
                    if (__any_sync(0xffffffffu, need_o)) {
                        // O rows in TMEM *= alpha, after the previous PV has landed
                        const uint32_t Jp = Jj - 1;
                        mbar_wait(&bars->pv_done[Jp & 1], (Jp >> 1) & 1);
                        tc_fence_after();
                        const float f = need_o ? alpha : 1.0f;
#pragma unroll 1
                        for (int c0 = 0; c0 < D; c0 += 32) {
                            uint32_t o[32];
                            tmem_ld32(tmem + lane_base + c0, o);
                            tmem_wait_ld();
#pragma unroll
                            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
                            tmem_st32(tmem + lane_base + c0, o);
                        }
                        tmem_wait_st();
                    }
                    const float mo = (m_run == -INFINITY) ? 0.0f : m_run;
                    float ls = 0.0f;
#pragma unroll
                    for (int c = 0; c < 64; c += 2) {
                        float e0 = ex2(fmaf(__uint_as_float(sr[c]), p.scale_log2, -mo));
                        float e1 = ex2(fmaf(__uint_as_float(sr[c + 1]), p.scale_log2, -mo));
                        uint32_t pk = pack_bf16(e0, e1);
                        sr[c >> 1] = pk;
                        ls += __uint_as_float(pk << 16) + __uint_as_float(pk & 0xFFFF0000u);
                    }
                    l_run += ls;
                }
                // P buffer (Jj & 1) was last read by PV_{Jj-2}
                if (Jj >= 2) mbar_wait(&bars->pv_done[Jj & 1], ((Jj - 2) >> 1) & 1);
                // keys past the end of the sample in its last page: zero those V rows so that
                // garbage (possibly NaN) bytes never meet a zero probability in the MMA
                const int nvalid = key_end - kbase;
                if (nvalid < kBlockN) {
                    const uint32_t s = Jj % kStages;
                    mbar_wait(&bars->kv_full[s], (Jj / kStages) & 1);
                    if (r < kBlockN && r >= nvalid) {
                        uint8_t* vs = smem + C::kOffStage + s * C::kStageBytes + C::kKVBytes;
#pragma unroll
                        for (int bx = 0; bx < C::kBoxes; ++bx) {
                            uint4* row = reinterpret_cast<uint4*>(vs + bx * (kBlockN * 128) + r * 128);
#pragma unroll
                            for (int c = 0; c < 8; ++c) row[c] = make_uint4(0, 0, 0, 0);
                        }
                    }
                }
                if (warp_active) {
                    uint8_t* prow = smem + C::kOffP + (Jj & 1) * C::kPBytes + r * 128;
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        uint4 v = make_uint4(sr[4 * c], sr[4 * c + 1], sr[4 * c + 2], sr[4 * c + 3]);
                        *reinterpret_cast<uint4*>(prow + ((c ^ (r & 7)) << 4)) = v;
                    }
                }
                fence_proxy_async_smem();
                tc_fence_before();
                // all softmax threads must be done with V-row zeroing before any warp arrives
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (lane == 0) mbar_arrive(&bars->p_full[Jj & 1]);
            }
            // ---------------- epilogue ----------------
            const uint32_t Jl = J + nblk - 1;
            mbar_wait(&bars->pv_done[Jl & 1], (Jl >> 1) & 1);
            tc_fence_after();
            if (warp_active) {
                const float inv_l = (l_run > 0.0f) ? 1.0f / l_run : 0.0f;
                const int h = wi.kvh * p.g + (grow % p.g);
                const bool direct = wi.part < 0;
                __nv_bfloat16* orow = p.out + ((int64_t)(off + node) * p.Hq + h) * D;
                float* prow = direct ? nullptr : p.part_o + ((int64_t)wi.part * kM + r) * D;
#pragma unroll 1
                for (int c0 = 0; c0 < D; c0 += 32) {
                    uint32_t o[32];
                    tmem_ld32(tmem + lane_base + c0, o);
                    tmem_wait_ld();
                    if (row_valid) {
                        if (direct) {
#pragma unroll
                            for (int c = 0; c < 32; c += 8) {
                                uint4 v;
                                v.x = pack_bf16(__uint_as_float(o[c]) * inv_l, __uint_as_float(o[c + 1]) * inv_l);
                                v.y = pack_bf16(__uint_as_float(o[c + 2]) * inv_l, __uint_as_float(o[c + 3]) * inv_l);
                                v.z = pack_bf16(__uint_as_float(o[c + 4]) * inv_l, __uint_as_float(o[c + 5]) * inv_l);
                                v.w = pack_bf16(__uint_as_float(o[c + 6]) * inv_l, __uint_as_float(o[c + 7]) * inv_l);
                                *reinterpret_cast<uint4*>(orow + c0 + c) = v;
                            }
                        } else {
#pragma unroll
                            for (int c = 0; c < 32; c += 4) {
                                float4 v = make_float4(__uint_as_float(o[c]) * inv_l, __uint_as_float(o[c + 1]) * inv_l,
                                                       __uint_as_float(o[c + 2]) * inv_l, __uint_as_float(o[c + 3]) * inv_l);
                                *reinterpret_cast<float4*>(prow + c0 + c) = v;
                            }
                        }
                    }
                }
                if (row_valid) {
                    const float lse2 = (l_run > 0.0f) ? m_run + __log2f(l_run) : -INFINITY;
                    if (direct) {
                        if (p.lse) p.lse[(int64_t)(off + node) * p.Hq + h] = lse2 * 0.6931471805599453f;
                    } else {
                        p.part_lse[(int64_t)wi.part * kM + r] = lse2;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->o_free);
            J += nblk;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<C::kTmemCols>(tmem);
}

// Merge split-KV partials: o = sum_p 2^(lse_p - M) o_p / sum_p 2^(lse_p - M).
template <int D>
__global__ void __launch_bounds__(128)
combine_kernel(const SplitUnit* __restrict__ units, const float* __restrict__ part_o,
               const float* __restrict__ part_lse, const int32_t* __restrict__ tree_off, int Hq,
               int g, __nv_bfloat16* __restrict__ out, float* __restrict__ lse) {
    const SplitUnit u = units[blockIdx.x];
    const int off = tree_off[u.b];
    const int T = tree_off[u.b + 1] - off;
    const int rows = min(kM, T * g - u.mtile * kM);
    for (int r = blockIdx.y; r < rows; r += gridDim.y) {
        float M = -INFINITY;
        for (int q = 0; q < u.n_parts; ++q) M = fmaxf(M, part_lse[(int64_t)(u.part_base + q) * kM + r]);
        float wsum = 0.0f, acc = 0.0f;
        for (int q = 0; q < u.n_parts; ++q) {
            const float lq = part_lse[(int64_t)(u.part_base + q) * kM + r];
            const float wq = (lq == -INFINITY) ? 0.0f : exp2f(lq - M);
            wsum += wq;
            if (threadIdx.x < D) acc += wq * part_o[((int64_t)(u.part_base + q) * kM + r) * D + threadIdx.x];
        }
        const int grow = u.mtile * kM + r;
        const int node = grow / g;
        const int h = u.kvh * g + grow % g;
        if (threadIdx.x < D)
            out[((int64_t)(off + node) * Hq + h) * D + threadIdx.x] = __float2bfloat16_rn(acc / wsum);
        if (threadIdx.x == 0 && lse) lse[(int64_t)(off + node) * Hq + h] = (M + log2f(wsum)) * 0.6931471805599453f;
    }
}

// ---------------------------------------------------------------- host: tensor maps
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(ptr);
    }
    return fn;
}

}  // namespace

// ---------------------------------------------------------------- plan
struct rs_attn_plan {
    int B, Hq, Hkv, D, ps, g, n_ctas, NT;
    std::vector<int32_t> cta_off;
    std::vector<WorkItem> items;
    std::vector<SplitUnit> units;
    int n_parts;
    size_t off_cta, off_items, off_units, off_part_o, off_part_lse, ws_bytes;
    std::vector<uint8_t> blob;  // [0, off_part_o): header tables, uploaded verbatim
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

extern "C" rs_status rs_attn_plan_create(const int32_t* prefix_len_host, const int32_t* tree_off_host,
                                         int32_t B, int32_t Hq, int32_t Hkv, int32_t head_dim,
                                         int32_t page_size, int32_t num_ctas,
                                         rs_attn_plan** plan_out) {
    RS_REQUIRE(plan_out && (B == 0 || (prefix_len_host && tree_off_host)), RS_ERR_INVALID_ARG,
               "rs_attn_plan_create: null pointer");
    RS_REQUIRE(B >= 0 && Hq > 0 && Hkv > 0 && Hq % Hkv == 0, RS_ERR_INVALID_ARG,
               "rs_attn_plan_create: bad heads Hq=%d Hkv=%d", Hq, Hkv);
    RS_REQUIRE(head_dim == 64 || head_dim == 128, RS_ERR_UNSUPPORTED,
               "rs_attn_plan_create: head_dim %d (supported: 64, 128)", head_dim);
    RS_REQUIRE(page_size == kBlockN, RS_ERR_UNSUPPORTED, "rs_attn_plan_create: page_size %d != 64",
               page_size);
    const int g = Hq / Hkv;
    RS_REQUIRE(g <= kM && (kM % g) == 0, RS_ERR_UNSUPPORTED, "rs_attn_plan_create: group size %d", g);
    if (num_ctas <= 0) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
        cudaGetLastError();
        num_ctas = sms;
    }
    auto* pl = new rs_attn_plan();
    pl->B = B; pl->Hq = Hq; pl->Hkv = Hkv; pl->D = head_dim; pl->ps = page_size; pl->g = g;
    pl->NT = B ? tree_off_host[B] : 0;
    // units
    struct U { int b, kvh, mtile, nblk; };
    std::vector<U> units;
    long long W = 0;
    for (int b = 0; b < B; ++b) {
        const int T = tree_off_host[b + 1] - tree_off_host[b];
        const int P = prefix_len_host[b];
        if (T < 1 || T > RS_MAX_TREE || P < 0 || T * g > 4 * kM) {
            delete pl;
            rs::set_error("rs_attn_plan_create: sample %d has T=%d P=%d (need 1<=T<=64, T*g<=512)", b, T, P);
            return (T < 1 || T > RS_MAX_TREE) ? RS_ERR_MALFORMED_TREE : RS_ERR_UNSUPPORTED;
        }
        const int nblk = (P + T + kBlockN - 1) / kBlockN;
        const int mt = (T * g + kM - 1) / kM;
        for (int kvh = 0; kvh < Hkv; ++kvh)
            for (int m = 0; m < mt; ++m) {
                units.push_back({b, kvh, m, nblk});
                W += nblk + kOvhBlocks;
            }
    }
    const int n_ctas = std::max(1, std::min<int>(num_ctas, (int)std::max<size_t>(units.size(), 1)));
    // balanced contiguous fill with split-KV cuts (load balance over heavy-tailed lengths)
    // Greedy contiguous fill: units are poured, in order, into CTAs of capacity `target`
    // (block units incl. a per-item overhead); a unit that overflows a CTA is cut (split-KV)
    // and continues on the next one. Parts are never smaller than kMinPart blocks.
    // CTA c owns the work interval [c*W/n, (c+1)*W/n) of the concatenated unit stream, so
    // rounding never accumulates: a CTA that is left slightly under/over full is absorbed by
    // the next boundary.
    // (Each extra split part costs another kOvhBlocks, so the remaining work is re-divided over
    // the remaining CTAs whenever a new CTA is entered.)
    long long W_eff = W;
    std::vector<std::vector<WorkItem>> per_cta(n_ctas);
    int cta = 0;
    long long pos = 0;
    long long end = (W_eff + n_ctas - 1) / n_ctas;
    auto next_cta = [&]() {
        ++cta;
        end = pos + (W_eff - pos + (n_ctas - cta) - 1) / (n_ctas - cta);
    };
    int n_parts = 0;
    for (const U& u : units) {
        int rem = u.nblk, start = 0;
        std::vector<std::pair<int, int>> where;   // (cta, index) of this unit's parts
        while (rem > 0) {
            if (cta < n_ctas - 1 && pos >= end) { next_cta(); continue; }
            const long long room = (cta == n_ctas - 1) ? (1ll << 60) : end - pos - kOvhBlocks;
            int take;
            if (room >= rem) {
                take = rem;
            } else if (room < kMinPart) {
                if (per_cta[cta].empty()) {
                    take = rem;               // never leave a CTA without work
                } else {
                    next_cta();               // too little room for a useful part: next CTA
                    continue;
                }
            } else {
                take = (int)room;
                if (rem - take < kMinPart) take = (rem >= 2 * kMinPart) ? rem - kMinPart : rem;
            }
            if (!where.empty()) W_eff += kOvhBlocks;   // an extra part of a split unit
            where.push_back({cta, (int)per_cta[cta].size()});
            per_cta[cta].push_back({u.b, u.kvh, u.mtile, start, start + take, -1});
            pos += take + kOvhBlocks;
            start += take;
            rem -= take;
        }
        if (where.size() > 1) {
            pl->units.push_back({u.b, u.kvh, u.mtile, (int)where.size(), n_parts, 0});
            for (auto& wc : where) per_cta[wc.first][wc.second].part = n_parts++;
        }
    }
    pl->cta_off.assign(n_ctas + 1, 0);
    for (int c = 0; c < n_ctas; ++c) {
        pl->cta_off[c] = (int)pl->items.size();
        pl->items.insert(pl->items.end(), per_cta[c].begin(), per_cta[c].end());
    }
    pl->cta_off[n_ctas] = (int)pl->items.size();
    pl->n_ctas = n_ctas;
    pl->n_parts = n_parts;
    pl->off_cta = 0;
    pl->off_items = align_up(sizeof(int32_t) * (n_ctas + 1), 256);
    pl->off_units = align_up(pl->off_items + sizeof(WorkItem) * pl->items.size(), 256);
    pl->off_part_o = align_up(pl->off_units + sizeof(SplitUnit) * pl->units.size(), 256);
    pl->off_part_lse = align_up(pl->off_part_o + sizeof(float) * (size_t)n_parts * kM * head_dim, 256);
    pl->ws_bytes = align_up(pl->off_part_lse + sizeof(float) * (size_t)n_parts * kM, 256);
    pl->blob.assign(pl->off_part_o, 0);
    memcpy(pl->blob.data() + pl->off_cta, pl->cta_off.data(), sizeof(int32_t) * (n_ctas + 1));
    if (!pl->items.empty())
        memcpy(pl->blob.data() + pl->off_items, pl->items.data(), sizeof(WorkItem) * pl->items.size());
    if (!pl->units.empty())
        memcpy(pl->blob.data() + pl->off_units, pl->units.data(), sizeof(SplitUnit) * pl->units.size());
    *plan_out = pl;
    return RS_OK;
}

extern "C" size_t rs_attn_plan_workspace_bytes(const rs_attn_plan* plan) {
    return plan ? plan->ws_bytes : 0;
}

extern "C" rs_status rs_attn_plan_upload(const rs_attn_plan* plan, void* ws, size_t ws_bytes, void* stream) {
    RS_REQUIRE(plan && ws, RS_ERR_INVALID_ARG, "rs_attn_plan_upload: null pointer");
    RS_REQUIRE(ws_bytes >= plan->ws_bytes, RS_ERR_WORKSPACE, "rs_attn_plan_upload: workspace %zu < %zu",
               ws_bytes, plan->ws_bytes);
    RS_REQUIRE((reinterpret_cast<uintptr_t>(ws) & 255) == 0, RS_ERR_INVALID_ARG,
               "rs_attn_plan_upload: workspace not 256-byte aligned");
    RS_CUDA_CHECK(cudaMemcpyAsync(ws, plan->blob.data(), plan->blob.size(), cudaMemcpyHostToDevice,
                                  rs::as_stream(stream)));
    return RS_OK;
}

extern "C" rs_status rs_attn_plan_info(const rs_attn_plan* plan, int32_t* num_ctas, int32_t* num_items,
                                       int32_t* num_split_units) {
    RS_REQUIRE(plan, RS_ERR_INVALID_ARG, "rs_attn_plan_info: null plan");
    if (num_ctas) *num_ctas = plan->n_ctas;
    if (num_items) *num_items = (int32_t)plan->items.size();
    if (num_split_units) *num_split_units = (int32_t)plan->units.size();
    return RS_OK;
}

extern "C" rs_status rs_attn_plan_items(const rs_attn_plan* plan, int32_t* cta_off, int32_t* items) {
    RS_REQUIRE(plan, RS_ERR_INVALID_ARG, "rs_attn_plan_items: null plan");
    if (cta_off) memcpy(cta_off, plan->cta_off.data(), sizeof(int32_t) * plan->cta_off.size());
    if (items && !plan->items.empty()) memcpy(items, plan->items.data(), sizeof(WorkItem) * plan->items.size());
    return RS_OK;
}

extern "C" void rs_attn_plan_destroy(rs_attn_plan* plan) { delete plan; }

template <int D>
static rs_status launch_attn(const rs_attn_plan* pl, const void* q, const void* k_pages, const void* v_pages,
                             int64_t num_pages, const int32_t* block_table, int32_t max_pages,
                             const int32_t* prefix_len, const int32_t* tree_off, const uint64_t* tree_mask,
                             float sm_scale, void* out, float* lse, void* ws, cudaStream_t st) {
    using C = Cfg<D>;
    PFN_encodeTiled enc = get_encode();
    RS_REQUIRE(enc, RS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap tmQ, tmK, tmV;
    {
        cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)pl->Hq, (cuuint64_t)std::max(pl->NT, 1)};
        cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)pl->Hq * D * 2};
        cuuint32_t box[3] = {64, (cuuint32_t)pl->g, (cuuint32_t)(kM / pl->g)};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = enc(&tmQ, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(q), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        RS_REQUIRE(r == CUDA_SUCCESS, RS_ERR_CUDA, "tensor map Q failed (%d)", (int)r);
    }
    const void* kv[2] = {k_pages, v_pages};
    CUtensorMap* tm[2] = {&tmK, &tmV};
    for (int i = 0; i < 2; ++i) {
        cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)num_pages * pl->Hkv * kBlockN};
        cuuint64_t strides[1] = {(cuuint64_t)D * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)kBlockN};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(tm[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(kv[i]), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        RS_REQUIRE(r == CUDA_SUCCESS, RS_ERR_CUDA, "tensor map KV failed (%d)", (int)r);
    }
    Params prm;
    uint8_t* w = static_cast<uint8_t*>(ws);
    prm.cta_off = reinterpret_cast<const int32_t*>(w + pl->off_cta);
    prm.items = reinterpret_cast<const WorkItem*>(w + pl->off_items);
    prm.part_o = reinterpret_cast<float*>(w + pl->off_part_o);
    prm.part_lse = reinterpret_cast<float*>(w + pl->off_part_lse);
    prm.prefix_len = prefix_len;
    prm.tree_off = tree_off;
    prm.tree_mask = tree_mask;
    prm.block_table = block_table;
    prm.max_pages = max_pages;
    prm.Hq = pl->Hq;
    prm.Hkv = pl->Hkv;
    prm.g = pl->g;
    prm.scale_log2 = sm_scale * 1.4426950408889634f;
    prm.out = static_cast<__nv_bfloat16*>(out);
    prm.lse = lse;
    static bool attr_set[2] = {false, false};
    if (!attr_set[D == 128]) {
        RS_CUDA_CHECK(cudaFuncSetAttribute(tree_attn_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           C::kSmemBytes));
        attr_set[D == 128] = true;
    }
    tree_attn_kernel<D><<<pl->n_ctas, kThreads, C::kSmemBytes, st>>>(tmQ, tmK, tmV, prm);
    RS_LAUNCH_CHECK();
    if (!pl->units.empty()) {
        dim3 grid((unsigned)pl->units.size(), 16);
        combine_kernel<D><<<grid, 128, 0, st>>>(reinterpret_cast<const SplitUnit*>(w + pl->off_units),
                                                prm.part_o, prm.part_lse, tree_off, pl->Hq, pl->g,
                                                prm.out, lse);
        RS_LAUNCH_CHECK();
    }
    return RS_OK;
}

extern "C" rs_status rs_tree_verify_attention(const rs_attn_plan* plan, const void* q, const void* k_pages,
                                              const void* v_pages, int64_t num_pages,
                                              const int32_t* block_table, int32_t max_pages,
                                              const int32_t* prefix_len, const int32_t* tree_off,
                                              const uint64_t* tree_mask, int32_t B, int32_t Hq,
                                              int32_t Hkv, int32_t head_dim, int32_t page_size,
                                              float sm_scale, void* out, float* lse, void* ws,
                                              size_t ws_bytes, void* stream) {
    RS_REQUIRE(plan, RS_ERR_INVALID_ARG, "rs_tree_verify_attention: null plan");
    RS_REQUIRE(plan->B == B && plan->Hq == Hq && plan->Hkv == Hkv && plan->D == head_dim &&
                   plan->ps == page_size,
               RS_ERR_INVALID_ARG, "rs_tree_verify_attention: arguments differ from the plan");
    RS_REQUIRE(ws && ws_bytes >= plan->ws_bytes, RS_ERR_WORKSPACE,
               "rs_tree_verify_attention: workspace %zu < %zu", ws_bytes, plan->ws_bytes);
    if (B == 0 || plan->items.empty()) return RS_OK;
    RS_REQUIRE(q && k_pages && v_pages && block_table && prefix_len && tree_off && tree_mask && out,
               RS_ERR_INVALID_ARG, "rs_tree_verify_attention: null pointer");
    RS_REQUIRE(num_pages > 0 && num_pages * Hkv * kBlockN < (1ll << 31), RS_ERR_UNSUPPORTED,
               "rs_tree_verify_attention: num_pages out of range");
    RS_REQUIRE(((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k_pages) |
                 reinterpret_cast<uintptr_t>(v_pages) | reinterpret_cast<uintptr_t>(out)) & 15) == 0,
               RS_ERR_INVALID_ARG, "rs_tree_verify_attention: pointers must be 16-byte aligned");
    cudaStream_t st = rs::as_stream(stream);
    if (head_dim == 128)
        return launch_attn<128>(plan, q, k_pages, v_pages, num_pages, block_table, max_pages, prefix_len,
                                tree_off, tree_mask, sm_scale, out, lse, ws, st);
    return launch_attn<64>(plan, q, k_pages, v_pages, num_pages, block_table, max_pages, prefix_len, tree_off,
                           tree_mask, sm_scale, out, lse, ws, st);
}
