// f2: the LM head fused with greedy acceptance.
//
// Verification scores all tree nodes in one target pass and the LM head is one of
// its GEMMs. Greedy acceptance needs, per tree node, only the
// arg-max of logits[r, :] = hidden[r, :] · W^T. This file computes that arg-max inside the
// GEMM's epilogue so the [rows, V] logits (263 MB at config 2) are never written:
//
//   lm_head_argmax_kernel  persistent tcgen05 GEMM, tile 128 rows x 256 vocab, K by 64;
//                          warp 0 = TMA producer (hidden + W tiles, SWIZZLE_128B, 4-stage
//                          ring), warp 1 = TMEM allocator + MMA issuer (one elected thread,
//                          kind::f16, M=128 N=256 K=16, fp32 accumulator in TMEM, double
//                          buffered across tiles), warps 2-5 = epilogue: each thread owns one
//                          accumulator row, streams its 256 columns out of TMEM and keeps
//                          (max, lowest index); the tile's winner is merged into a per-row
//                          64-bit key by atomicMax (orderable float bits << 32 | ~vocab id,
//                          so equal values resolve to the lowest id, Z6).
//   lm_head_finalize_kernel  key -> (token, max logit).
//   greedy_walk_kernel     c-2's walk over the per-node arg-max tokens, one warp per sample.
//
// Tile order: tile t -> (m = t % num_m, n = t / num_m); CTAs sweep t in steps of gridDim, so the
// num_m row tiles of one vocab tile run concurrently and W streams from HBM about once.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>

#include "common.cuh"
#include "compact_tail.cuh"
#include "sm100_ptx.cuh"

namespace {

using namespace rs::ptx;

constexpr int kBM = 128;                    // tree-node rows per tile (MMA M)
constexpr int kBN = 256;                    // vocabulary entries per tile (MMA N)
constexpr int kBK = 64;                     // K per stage: one 128-byte swizzle row
constexpr int kStages = 4;
constexpr int kABytes = kBM * kBK * 2;      // 16 KB
constexpr int kBBytes = kBN * kBK * 2;      // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kThreads = 192;
constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256;

struct Bars {
    uint64_t full[kStages], empty[kStages], acc_full[2], acc_empty[2];
    uint32_t tmem;
};

__device__ __forceinline__ unsigned long long argmax_key(float x, int v) {
    uint32_t b = __float_as_uint(__fadd_rn(x, 0.0f));   // -0 -> +0: equal values tie on the id
    b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return ((unsigned long long)b << 32) | (unsigned long long)(~(uint32_t)v);
}

// kLogits: the epilogue writes the bf16 logits tile instead (the LM head feeding the sampling
// modes, which need whole rows: rs_lm_head_logits).
template <bool kLogits>
__global__ void __launch_bounds__(kThreads, 1)
lm_head_argmax_kernel(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmW,
                      int rows, int V, int Dm, unsigned long long* __restrict__ keys,
                      __nv_bfloat16* __restrict__ logits) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Bars* bars = reinterpret_cast<Bars*>(smem + kStages * kStageBytes);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int num_m = (rows + kBM - 1) / kBM, num_n = (V + kBN - 1) / kBN;
    const int ntiles = num_m * num_n, nk = Dm / kBK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&bars->full[s], 1);
            mbar_init(&bars->empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&bars->acc_full[a], 1);
            mbar_init(&bars->acc_empty[a], 4);
        }
        fence_mbar_init();
        prefetch_tmap(&tmH);
        prefetch_tmap(&tmW);
    }
    if (warp == 1) tmem_alloc<512>(&bars->tmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = bars->tmem;

    if (warp == 0) {
        // ---------------------------------------------------------------- TMA producer
        if (elect_one()) {
            uint32_t it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int m = t % num_m, n = t / num_m;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % kStages;
                    mbar_wait(&bars->empty[s], ((it / kStages) & 1) ^ 1);
                    uint8_t* sa = smem + s * kStageBytes;
                    mbar_arrive_expect_tx(&bars->full[s], kStageBytes);
                    tma_load_2d(sa, &tmH, &bars->full[s], kb * kBK, m * kBM);
                    tma_load_2d(sa + kABytes, &tmW, &bars->full[s], kb * kBK, n * kBN);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA issuer
        constexpr uint32_t idesc = idesc_bf16_f32(kBM, kBN, 0);
        const uint32_t sbase = smem_u32(smem);
        uint32_t it = 0, i = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const uint32_t a = i & 1;
            mbar_wait(&bars->acc_empty[a], ((i >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d = tmem + a * kBN;
            for (int kb = 0; kb < nk; ++kb, ++it) {
                const int s = it % kStages;
                mbar_wait(&bars->full[s], (it / kStages) & 1);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t sa = sbase + s * kStageBytes, sb = sa + kABytes;
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) {
                        const uint64_t ad = smem_desc_sw128(sa + k * 32, 16, 1024);
                        const uint64_t bd = smem_desc_sw128(sb + k * 32, 16, 1024);
                        umma_f16(d, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
                    }
                    umma_commit(&bars->empty[s]);
                    if (kb == nk - 1) umma_commit(&bars->acc_full[a]);
                }
                __syncwarp();
            }
        }
    } else {
        // ---------------------------------------------------------------- epilogue (warps 2-5)
        const int q = warp & 3;                  // TMEM sub-partition this warp may access
        uint32_t i = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const int m = t % num_m, n = t / num_m;
            const uint32_t a = i & 1;
            mbar_wait(&bars->acc_full[a], (i >> 1) & 1);
            tc_fence_after();
            const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + a * kBN;
            const int v0 = n * kBN;
            const bool full_tile = v0 + kBN <= V;
            if constexpr (kLogits) {
                // one accumulator row per thread: 64 columns per round out of TMEM, rounded to
                // bf16 (RN) and stored as 8 x 16-byte vectors (V % 8 == 0: rows stay aligned)
                const int row = m * kBM + q * 32 + lane;
                __nv_bfloat16* dst = logits + (size_t)row * V + v0;
#pragma unroll 1
                for (int c = 0; c < kBN; c += 64) {
                    uint32_t r0[32], r1[32];
                    tmem_ld32(base + c, r0);
                    tmem_ld32(base + c + 32, r1);
                    tmem_wait_ld();
                    if (row < rows) {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const uint32_t* rr = h ? r1 : r0;
#pragma unroll
                            for (int j8 = 0; j8 < 32; j8 += 8) {
                                const int v = c + 32 * h + j8;
                                if (full_tile || v0 + v + 8 <= V) {
                                    uint32_t pk[4];
#pragma unroll
                                    for (int e = 0; e < 4; ++e) {
                                        const __nv_bfloat162 b2 = __floats2bfloat162_rn(__uint_as_float(rr[j8 + 2 * e]),
                                                                                        __uint_as_float(rr[j8 + 2 * e + 1]));
                                        pk[e] = *reinterpret_cast<const uint32_t*>(&b2);
                                    }
                                    *reinterpret_cast<uint4*>(dst + v) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                                }
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->acc_empty[a]);
                continue;
            }
            float best = -INFINITY;
            int bi = -1;
            uint32_t amag = 0;   // max |x| bits of the row's valid columns: >= 0x7F800000 <=> Inf / NaN
#pragma unroll 1
            for (int c = 0; c < kBN; c += 64) {
                uint32_t r0[32], r1[32];
                tmem_ld32(base + c, r0);
                tmem_ld32(base + c + 32, r1);
                tmem_wait_ld();
                if (full_tile) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float x = __uint_as_float(r0[j]);
                        amag = max(amag, r0[j] & 0x7FFFFFFFu);
                        if (x > best) { best = x; bi = v0 + c + j; }
                    }
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float x = __uint_as_float(r1[j]);
                        amag = max(amag, r1[j] & 0x7FFFFFFFu);
                        if (x > best) { best = x; bi = v0 + c + 32 + j; }
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float x = __uint_as_float(r0[j]);
                        if (v0 + c + j < V) amag = max(amag, r0[j] & 0x7FFFFFFFu);
                        if (v0 + c + j < V && x > best) { best = x; bi = v0 + c + j; }
                    }
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float x = __uint_as_float(r1[j]);
                        if (v0 + c + 32 + j < V) amag = max(amag, r1[j] & 0x7FFFFFFFu);
                        if (v0 + c + 32 + j < V && x > best) { best = x; bi = v0 + c + 32 + j; }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->acc_empty[a]);
            const int row = m * kBM + q * 32 + lane;
            // a non-finite logit anywhere in the row: the all-ones key (above every real key) marks
            // it and finalize reports no arg-max (-1), as rs_tree_accept flags such a row (Z15)
            if (row < rows && amag >= 0x7F800000u) atomicMax(&keys[row], ~0ull);
            else if (row < rows && bi >= 0) atomicMax(&keys[row], argmax_key(best, bi));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<512>(tmem);
}

__global__ void lm_head_finalize_kernel(const unsigned long long* __restrict__ keys, int rows,
                                        int32_t* __restrict__ tok, float* __restrict__ mx) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const unsigned long long k = keys[r];
    if (k == 0 || k == ~0ull) {                // a non-finite logit in the row (or no columns): no arg-max
        tok[r] = -1;
        if (mx) mx[r] = __uint_as_float(0x7fc00000u);
        return;
    }
    tok[r] = (int32_t)(~(uint32_t)(k & 0xffffffffu));
    if (mx) {
        uint32_t b = (uint32_t)(k >> 32);
        b = (b & 0x80000000u) ? (b & 0x7fffffffu) : ~b;
        mx[r] = __uint_as_float(b);
    }
}

// One warp per sample: validate the tree, then walk (c-2). At the current node c the lanes
// test nodes x > c for (parent == c, token == argmax[c]); the lowest such x wins (ballot).
// write: this warp writes the outputs; path_s (optional, shared memory): the path for a fused
// commit. Returns the accepted length (all lanes).
__device__ __forceinline__ int greedy_walk_warp(const int32_t* __restrict__ amax, const int32_t* __restrict__ parent,
                                                const int32_t* __restrict__ token,
                                                const int32_t* __restrict__ tree_off, int b, bool write,
                                                int32_t* __restrict__ acc, int32_t* __restrict__ path,
                                                int32_t* __restrict__ bonus, int32_t* __restrict__ flags,
                                                int* path_s) {
    const int lane = threadIdx.x & 31;
    const int s = tree_off[b], T = tree_off[b + 1] - s;
    int32_t* pb = path + (size_t)b * RS_MAX_TREE;
    bool ok = T >= 1 && T <= RS_MAX_TREE;
    int p0 = -1, p1 = -1;
    if (ok) {
        if (lane < T) p0 = parent[s + lane];
        if (lane + 32 < T) p1 = parent[s + lane + 32];
        const bool bad0 = lane < T && (lane == 0 ? p0 != -1 : (p0 < 0 || p0 >= lane));
        const bool bad1 = lane + 32 < T && (p1 < 0 || p1 >= lane + 32);
        ok = !__any_sync(0xffffffffu, bad0 || bad1);
    }
    const int t0 = (ok && lane < T) ? token[s + lane] : 0;
    const int t1 = (ok && lane + 32 < T) ? token[s + lane + 32] : 0;
    int c = 0, n = 0, fl = ok ? 0 : RS_FLAG_MALFORMED;
    if (write) {
        pb[lane] = -1;
        pb[lane + 32] = -1;
    }
    if (path_s && lane == 0) path_s[0] = 0;
    __syncwarp();
    if (ok) {
        for (;;) {
            const int t = amax[s + c];
            if (t < 0) { fl |= RS_FLAG_NONFINITE; break; }
            const unsigned m0 = __ballot_sync(0xffffffffu, lane > c && lane < T && p0 == c && t0 == t);
            const unsigned m1 = __ballot_sync(0xffffffffu, lane + 32 > c && lane + 32 < T && p1 == c && t1 == t);
            const int nx = m0 ? __ffs(m0) - 1 : (m1 ? 32 + __ffs(m1) - 1 : -1);
            if (nx < 0) break;
            c = nx;
            ++n;
            if (write && lane == 0) pb[n] = c;
            if (path_s && lane == 0) path_s[n] = c;
        }
    }
    if (write && lane == 0) {
        pb[0] = 0;
        acc[b] = ok ? n : 0;
        bonus[b] = (ok && !(fl & RS_FLAG_NONFINITE)) ? amax[s + c] : -1;
        flags[b] = fl;
    }
    return ok ? n : 0;
}

__global__ void greedy_walk_kernel(const int32_t* __restrict__ amax, const int32_t* __restrict__ parent,
                                   const int32_t* __restrict__ token, const int32_t* __restrict__ tree_off,
                                   int B, int32_t* __restrict__ acc, int32_t* __restrict__ path,
                                   int32_t* __restrict__ bonus, int32_t* __restrict__ flags) {
    const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (b >= B) return;
    greedy_walk_warp(amax, parent, token, tree_off, b, true, acc, path, bonus, flags, nullptr);
}

// The walk fused with the KV commit (rs_tree_accept_greedy_tokens_compact): a CTA per (sample,
// group of layers) as kv_compact_kernel; its warp 0 walks the sample's tree (cheap: a ballot per
// node over the per-node arg-max tokens), group 0 writes the walk's outputs, and every CTA then
// commits the path for its layer group (rs::compact_sample).
__global__ void __launch_bounds__(256)
greedy_walk_compact_kernel(const __grid_constant__ rs::CompactArgs A, const int32_t* __restrict__ amax,
                           const int32_t* __restrict__ parent, const int32_t* __restrict__ token,
                           const int32_t* __restrict__ tree_off, int32_t* __restrict__ acc,
                           int32_t* __restrict__ path, int32_t* __restrict__ bonus, int32_t* __restrict__ flags) {
    __shared__ rs::CompactSmem cm;
    __shared__ int path_s[RS_MAX_TREE];
    __shared__ int a_s;
    const int b = blockIdx.x;
    if (threadIdx.x < 32) {
        const int a = greedy_walk_warp(amax, parent, token, tree_off, b, blockIdx.y == 0, acc, path, bonus, flags,
                                       path_s);
        if (threadIdx.x == 0) a_s = a;
    }
    __syncthreads();
    rs::compact_sample(A, b, a_s, [&](int k) { return path_s[k]; }, blockIdx.y, gridDim.y, blockIdx.y == 0, cm);
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled encode_fn() {
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

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

}  // namespace

extern "C" size_t rs_lm_head_argmax_workspace_bytes(int32_t rows) {
    return rows > 0 ? (size_t)rows * sizeof(unsigned long long) : 0;
}

extern "C" rs_status rs_lm_head_argmax(const void* hidden, const void* weight, int32_t rows, int32_t V, int32_t Dm,
                                       int32_t* argmax_token, float* max_logit, void* ws, size_t ws_bytes,
                                       void* stream) {
    rs::bind_device(hidden);
    RS_REQUIRE(rows >= 0 && V >= 1 && Dm >= kBK && Dm % kBK == 0, RS_ERR_INVALID_ARG,
               "rs_lm_head_argmax: rows=%d V=%d Dm=%d (Dm must be a positive multiple of 64)", rows, V, Dm);
    if (rows == 0) return RS_OK;
    RS_REQUIRE(hidden && weight && argmax_token, RS_ERR_INVALID_ARG, "rs_lm_head_argmax: null pointer");
    RS_REQUIRE((reinterpret_cast<uintptr_t>(hidden) & 15) == 0 && (reinterpret_cast<uintptr_t>(weight) & 15) == 0,
               RS_ERR_INVALID_ARG, "rs_lm_head_argmax: hidden/weight must be 16-byte aligned");
    const size_t need = rs_lm_head_argmax_workspace_bytes(rows);
    RS_REQUIRE(ws && ws_bytes >= need && (reinterpret_cast<uintptr_t>(ws) & 7) == 0, RS_ERR_WORKSPACE,
               "rs_lm_head_argmax: workspace %zu < %zu bytes (8-byte aligned)", ws_bytes, need);
    PFN_encodeTiled enc = encode_fn();
    RS_REQUIRE(enc, RS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap tmH, tmW;
    const void* src[2] = {hidden, weight};
    CUtensorMap* tm[2] = {&tmH, &tmW};
    const cuuint64_t nrow[2] = {(cuuint64_t)rows, (cuuint64_t)V};
    const cuuint32_t brow[2] = {kBM, kBN};
    for (int i = 0; i < 2; ++i) {
        cuuint64_t dims[2] = {(cuuint64_t)Dm, nrow[i]};
        cuuint64_t strides[1] = {(cuuint64_t)Dm * 2};
        cuuint32_t box[2] = {kBK, brow[i]};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(tm[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(src[i]), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        RS_REQUIRE(r == CUDA_SUCCESS, RS_ERR_CUDA, "rs_lm_head_argmax: tensor map %d failed (%d)", i, (int)r);
    }
    cudaStream_t st = rs::as_stream(stream);
    auto* keys = static_cast<unsigned long long*>(ws);
    RS_CUDA_CHECK(cudaMemsetAsync(keys, 0, need, st));
    static bool attr = false;
    if (!attr) {
        RS_CUDA_CHECK(cudaFuncSetAttribute(lm_head_argmax_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kSmemBytes));
        attr = true;
    }
    const int ntiles = ((rows + kBM - 1) / kBM) * ((V + kBN - 1) / kBN);
    const int grid = std::min(ntiles, num_sms());
    lm_head_argmax_kernel<false><<<grid, kThreads, kSmemBytes, st>>>(tmH, tmW, rows, V, Dm, keys, nullptr);
    RS_LAUNCH_CHECK();
    lm_head_finalize_kernel<<<(rows + 255) / 256, 256, 0, st>>>(keys, rows, argmax_token, max_logit);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

extern "C" rs_status rs_tree_accept_greedy_tokens(const int32_t* argmax_token, const int32_t* parent,
                                                  const int32_t* token, const int32_t* tree_off, int32_t B,
                                                  int32_t* accepted_len, int32_t* path, int32_t* bonus_token,
                                                  int32_t* status_flags, void* stream) {
    rs::bind_device(argmax_token);
    RS_REQUIRE(B >= 0, RS_ERR_INVALID_ARG, "rs_tree_accept_greedy_tokens: B=%d", B);
    if (B == 0) return RS_OK;
    RS_REQUIRE(argmax_token && parent && token && tree_off && accepted_len && path && bonus_token && status_flags,
               RS_ERR_INVALID_ARG, "rs_tree_accept_greedy_tokens: null pointer");
    const int wpb = 4;
    greedy_walk_kernel<<<(B + wpb - 1) / wpb, 32 * wpb, 0, rs::as_stream(stream)>>>(
        argmax_token, parent, token, tree_off, B, accepted_len, path, bonus_token, status_flags);
    RS_LAUNCH_CHECK();
    return RS_OK;
}

extern "C" rs_status rs_lm_head_logits(const void* hidden, const void* weight, int32_t rows, int32_t V, int32_t Dm,
                                       void* logits, void* stream) {
    rs::bind_device(hidden);
    RS_REQUIRE(rows >= 0 && V >= 8 && V % 8 == 0 && Dm >= kBK && Dm % kBK == 0, RS_ERR_INVALID_ARG,
               "rs_lm_head_logits: rows=%d V=%d Dm=%d (V a multiple of 8, Dm a positive multiple of 64)", rows, V,
               Dm);
    if (rows == 0) return RS_OK;
    RS_REQUIRE(hidden && weight && logits, RS_ERR_INVALID_ARG, "rs_lm_head_logits: null pointer");
    RS_REQUIRE((reinterpret_cast<uintptr_t>(hidden) & 15) == 0 && (reinterpret_cast<uintptr_t>(weight) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(logits) & 15) == 0,
               RS_ERR_INVALID_ARG, "rs_lm_head_logits: hidden/weight/logits must be 16-byte aligned");
    PFN_encodeTiled enc = encode_fn();
    RS_REQUIRE(enc, RS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap tmH, tmW;
    const void* src[2] = {hidden, weight};
    CUtensorMap* tm[2] = {&tmH, &tmW};
    const cuuint64_t nrow[2] = {(cuuint64_t)rows, (cuuint64_t)V};
    const cuuint32_t brow[2] = {kBM, kBN};
    for (int i = 0; i < 2; ++i) {
        cuuint64_t dims[2] = {(cuuint64_t)Dm, nrow[i]};
        cuuint64_t strides[1] = {(cuuint64_t)Dm * 2};
        cuuint32_t box[2] = {kBK, brow[i]};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(tm[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(src[i]), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        RS_REQUIRE(r == CUDA_SUCCESS, RS_ERR_CUDA, "rs_lm_head_logits: tensor map %d failed (%d)", i, (int)r);
    }
    cudaStream_t st = rs::as_stream(stream);
    static bool attr = false;
    if (!attr) {
        RS_CUDA_CHECK(cudaFuncSetAttribute(lm_head_argmax_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           kSmemBytes));
        attr = true;
    }
    const int ntiles = ((rows + kBM - 1) / kBM) * ((V + kBN - 1) / kBN);
    const int grid = std::min(ntiles, num_sms());
    lm_head_argmax_kernel<true><<<grid, kThreads, kSmemBytes, st>>>(tmH, tmW, rows, V, Dm, nullptr,
                                                                    static_cast<__nv_bfloat16*>(logits));
    RS_LAUNCH_CHECK();
    return RS_OK;
}

extern "C" rs_status rs_tree_accept_greedy_tokens_compact(
    const int32_t* argmax_token, const int32_t* parent, const int32_t* token, const int32_t* tree_off, int32_t B,
    int32_t* accepted_len, int32_t* path, int32_t* bonus_token, int32_t* status_flags, void* const* k_layers_host,
    void* const* v_layers_host, int32_t L, int32_t Hkv, int32_t head_dim, int32_t page_size, const int32_t* block_table,
    int32_t max_pages, const int32_t* prefix_len, int32_t* new_len, int32_t* moves, void* stream) {
    rs::bind_device(argmax_token);
    RS_REQUIRE(B >= 0 && L >= 0 && L <= rs::kCompactMaxLayers && Hkv > 0 && page_size > 0 && max_pages >= 0,
               RS_ERR_INVALID_ARG, "rs_tree_accept_greedy_tokens_compact: bad sizes (L=%d, at most %d layers)", L,
               rs::kCompactMaxLayers);
    RS_REQUIRE(head_dim > 0 && head_dim % 8 == 0, RS_ERR_UNSUPPORTED,
               "rs_tree_accept_greedy_tokens_compact: head_dim %% 8 != 0");
    if (B == 0) return RS_OK;
    RS_REQUIRE(argmax_token && parent && token && tree_off && accepted_len && path && bonus_token && status_flags &&
                   block_table && prefix_len && new_len && (L == 0 || (k_layers_host && v_layers_host)),
               RS_ERR_INVALID_ARG, "rs_tree_accept_greedy_tokens_compact: null pointer");
    rs::CompactArgs A;
    for (int i = 0; i < L; ++i) {
        RS_REQUIRE(k_layers_host[i] && v_layers_host[i], RS_ERR_INVALID_ARG,
                   "rs_tree_accept_greedy_tokens_compact: null layer pointer");
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
    const int groups = L > 0 ? (L + 1) / 2 : 1;   // two layers per CTA, as rs_kv_compact
    greedy_walk_compact_kernel<<<dim3((unsigned)B, (unsigned)groups), 256, 0, rs::as_stream(stream)>>>(
        A, argmax_token, parent, token, tree_off, accepted_len, path, bonus_token, status_flags);
    RS_LAUNCH_CHECK();
    return RS_OK;
}
