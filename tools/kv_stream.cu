// Microbenchmark: stream paged K and V tiles exactly as the attention kernel does (two tensors
// [pages, Hkv, 64, 128] bf16, per-CTA list of (page, kvh) blocks, K and V of a block loaded by
// two producer warps with 4-slot rings each), no compute. Variants probe the address pattern.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2512_04752_b200/csrc -o kv_stream kv_stream.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <numeric>
#include <random>
#include <vector>

#include "sm100_ptx.cuh"

using namespace rs::ptx;
constexpr int SLOTS = 4;
constexpr int kTile = 64 * 256;

__global__ void __launch_bounds__(128, 1) kv_kernel(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
                                                    const int* rows_k, const int* rows_v, int n, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * SLOTS * kTile);   // full[2][S], empty[2][S]
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4 * SLOTS; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp < 2 && lane == 0) {   // producers: warp 0 K, warp 1 V
        const int* rows = (warp == 0 ? rows_k : rows_v) + (size_t)blockIdx.x * n;
        const CUtensorMap* tm = warp == 0 ? &tk : &tv;
        uint64_t* full = bars + warp * SLOTS;
        uint64_t* empty = bars + 2 * SLOTS + warp * SLOTS;
        for (int j = 0; j < n; ++j) {
            const int s = j % SLOTS;
            mbar_wait(&empty[s], ((j / SLOTS) & 1) ^ 1);
            mbar_arrive_expect_tx(&full[s], kTile);
            uint8_t* dst = smem + (warp * SLOTS + s) * kTile;
            tma_load_2d(dst, tm, &full[s], 0, rows[j]);
            tma_load_2d(dst + kTile / 2, tm, &full[s], 64, rows[j]);
        }
    } else if (warp >= 2 && lane == 0) {   // consumers: warp 2 K, warp 3 V
        const int which = warp - 2;
        uint64_t* full = bars + which * SLOTS;
        uint64_t* empty = bars + 2 * SLOTS + which * SLOTS;
        unsigned long long acc = 0;
        for (int j = 0; j < n; ++j) {
            const int s = j % SLOTS;
            mbar_wait(&full[s], (j / SLOTS) & 1);
            acc += *reinterpret_cast<volatile uint32_t*>(smem + (which * SLOTS + s) * kTile);
            mbar_arrive(&empty[s]);
        }
        if (acc == 0x12345) sink[0] = acc;
    }
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int Hkv = 8, B = 64, P = 1040, sms = 148;
    const int npg = (P + 63) / 64;                  // 17 pages per sample
    const int num_pages = B * npg;
    size_t bytes = (size_t)num_pages * Hkv * kTile;
    void *k, *v, *big;
    cudaMalloc(&k, bytes);
    cudaMalloc(&v, bytes);
    cudaMalloc(&big, 2 * bytes + (1 << 20) * 3);    // for the "offset" variant
    cudaMemset(k, 1, bytes); cudaMemset(v, 1, bytes); cudaMemset(big, 1, 2 * bytes + (1 << 20) * 3);
    PFN_encodeTiled enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    auto mk = [&](void* base, size_t rows) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {128, rows};
        cuuint64_t strides[1] = {256};
        cuuint32_t box[2] = {64, 64};
        cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        return tm;
    };
    std::mt19937 rng(1);
    std::vector<int> perm(num_pages), perm2(num_pages);
    std::iota(perm.begin(), perm.end(), 0);
    std::shuffle(perm.begin(), perm.end(), rng);
    std::iota(perm2.begin(), perm2.end(), 0);
    std::shuffle(perm2.begin(), perm2.end(), rng);
    // units (b, kvh) in order, 17 blocks each; contiguous split over CTAs (~58.8 blocks per CTA)
    const int total = B * Hkv * npg;
    const int per = (total + sms - 1) / sms;
    auto run = [&](const char* name, const CUtensorMap& tk, const CUtensorMap& tv, bool vperm2, bool shuffle_all) {
        std::vector<int> rk((size_t)sms * per, 0), rv((size_t)sms * per, 0);
        std::vector<std::pair<int,int>> blocks;   // (page, kvh)
        for (int b = 0; b < B; ++b)
            for (int h = 0; h < Hkv; ++h)
                for (int j = 0; j < npg; ++j) blocks.push_back({b * npg + j, h});
        if (shuffle_all) std::shuffle(blocks.begin(), blocks.end(), rng);
        for (int i = 0; i < total; ++i) {
            const int pg = blocks[i].first, h = blocks[i].second;
            rk[i] = (perm[pg] * Hkv + h) * 64;
            rv[i] = ((vperm2 ? perm2[pg] : perm[pg]) * Hkv + h) * 64;
        }
        int *dk, *dv;
        cudaMalloc(&dk, rk.size() * 4); cudaMalloc(&dv, rv.size() * 4);
        cudaMemcpy(dk, rk.data(), rk.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dv, rv.data(), rv.size() * 4, cudaMemcpyHostToDevice);
        unsigned long long* sink; cudaMalloc(&sink, 8);
        const int smem = 2 * SLOTS * kTile + 2048;
        cudaFuncSetAttribute(kv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaEvent_t a, e; cudaEventCreate(&a); cudaEventCreate(&e);
        for (int w = 0; w < 3; ++w) kv_kernel<<<sms, 128, smem>>>(tk, tv, dk, dv, per, sink);
        float best = 1e9;
        for (int r = 0; r < 10; ++r) {
            cudaEventRecord(a);
            kv_kernel<<<sms, 128, smem>>>(tk, tv, dk, dv, per, sink);
            cudaEventRecord(e);
            cudaEventSynchronize(e);
            float ms; cudaEventElapsedTime(&ms, a, e);
            best = std::min(best, ms);
        }
        const double by = 2.0 * sms * per * kTile;
        printf("%-44s %7.1f us  %7.1f GB/s  err=%s\n", name, best * 1e3, by / (best * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
        cudaFree(dk); cudaFree(dv); cudaFree(sink);
    };
    const size_t rows = (size_t)num_pages * Hkv * 64;
    CUtensorMap tk = mk(k, rows), tv = mk(v, rows);
    run("K,V separate allocs, same page perm", tk, tv, false, false);
    run("K,V separate allocs, independent perms", tk, tv, true, false);
    run("K,V separate, blocks shuffled globally", tk, tv, false, true);
    CUtensorMap tk2 = mk(big, rows), tv2 = mk((char*)big + bytes + (1 << 20) * 3 + 4096 * 5, rows);
    run("K,V in one alloc, V offset by odd amount", tk2, tv2, false, false);
    // like the verify step: every launch reads a different layer's cache (8 layers rotating)
    {
        std::vector<CUtensorMap> tks, tvs;
        for (int l = 0; l < 8; ++l) {
            void *kk, *vv;
            cudaMalloc(&kk, bytes);
            cudaMalloc(&vv, bytes);
            cudaMemset(kk, 1, bytes);
            cudaMemset(vv, 1, bytes);
            tks.push_back(mk(kk, rows));
            tvs.push_back(mk(vv, rows));
        }
        std::vector<int> rk((size_t)sms * per, 0), rv((size_t)sms * per, 0);
        for (int i = 0; i < total; ++i) {
            const int b = i / (Hkv * npg), h = (i / npg) % Hkv, j = i % npg;
            rk[i] = (perm[b * npg + j] * Hkv + h) * 64;
            rv[i] = rk[i];
        }
        int *dk, *dv;
        cudaMalloc(&dk, rk.size() * 4); cudaMalloc(&dv, rv.size() * 4);
        cudaMemcpy(dk, rk.data(), rk.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dv, rv.data(), rv.size() * 4, cudaMemcpyHostToDevice);
        unsigned long long* sink; cudaMalloc(&sink, 8);
        const int smem = 2 * SLOTS * kTile + 2048;
        cudaEvent_t a, e; cudaEventCreate(&a); cudaEventCreate(&e);
        for (int w = 0; w < 8; ++w) kv_kernel<<<sms, 128, smem>>>(tks[w], tvs[w], dk, dv, per, sink);
        cudaEventRecord(a);
        for (int r = 0; r < 32; ++r) kv_kernel<<<sms, 128, smem>>>(tks[r % 8], tvs[r % 8], dk, dv, per, sink);
        cudaEventRecord(e);
        cudaEventSynchronize(e);
        float ms; cudaEventElapsedTime(&ms, a, e);
        const double by = 2.0 * sms * per * kTile;
        printf("%-44s %7.1f us  %7.1f GB/s  err=%s\n", "8 rotating layers (32 launches, mean)", ms * 1e3 / 32,
               by / (ms * 1e-3 / 32) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
