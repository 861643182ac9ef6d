// Microbenchmark: how fast can a persistent kernel stream paged KV tiles with TMA on this
// B200, as a function of ring depth / tile size? (Ceiling for the attention kernel's loads.)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2512_04752_b200/csrc
//        -o tma_stream tma_stream.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "sm100_ptx.cuh"

using namespace rs::ptx;

template <int SLOTS, int TILE_ROWS>
__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, const int* order,
                                                        int n_tiles_per_cta, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int kTileBytes = TILE_ROWS * 128 * 2;   // two 64-col boxes (d = 128)
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + SLOTS * kTileBytes);
    uint64_t* empty = full + SLOTS;
    if (threadIdx.x == 0) {
        for (int i = 0; i < SLOTS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        fence_mbar_init();
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int* ord = order + (size_t)blockIdx.x * n_tiles_per_cta;
    if (warp == 0 && lane == 0) {
        for (int j = 0; j < n_tiles_per_cta; ++j) {
            int s = j % SLOTS;
            mbar_wait(&empty[s], ((j / SLOTS) & 1) ^ 1);
            mbar_arrive_expect_tx(&full[s], kTileBytes);
            int row = ord[j] * TILE_ROWS;
            uint8_t* dst = smem + s * kTileBytes;
            tma_load_2d(dst, &tm, &full[s], 0, row);
            tma_load_2d(dst + TILE_ROWS * 128, &tm, &full[s], 64, row);
        }
    } else if (warp == 1 && lane == 0) {
        unsigned long long acc = 0;
        for (int j = 0; j < n_tiles_per_cta; ++j) {
            int s = j % SLOTS;
            mbar_wait(&full[s], (j / SLOTS) & 1);
            acc += *reinterpret_cast<volatile uint32_t*>(smem + s * kTileBytes);
            mbar_arrive(&empty[s]);
        }
        if (acc == 0x12345) sink[0] = acc;
    }
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int SLOTS, int TILE_ROWS>
void run(void* buf, size_t rows, int ctas, int tiles_per_cta, CUtensorMapL2promotion promo, const char* name) {
    PFN_encodeTiled enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {128, rows};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, TILE_ROWS};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    size_t n_tiles_total = rows / TILE_ROWS;
    std::vector<int> order((size_t)ctas * tiles_per_cta);
    srand(1);
    for (auto& o : order) o = (int)(((size_t)rand() * 7919u) % n_tiles_total);
    int* d_order;
    cudaMalloc(&d_order, order.size() * 4);
    cudaMemcpy(d_order, order.data(), order.size() * 4, cudaMemcpyHostToDevice);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    int smem = SLOTS * TILE_ROWS * 256 + 1024 + 256;
    cudaFuncSetAttribute(stream_kernel<SLOTS, TILE_ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) stream_kernel<SLOTS, TILE_ROWS><<<ctas, 128, smem>>>(tm, d_order, tiles_per_cta, sink);
    cudaEventRecord(a);
    stream_kernel<SLOTS, TILE_ROWS><<<ctas, 128, smem>>>(tm, d_order, tiles_per_cta, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    double bytes = (double)ctas * tiles_per_cta * TILE_ROWS * 256;
    printf("%-28s slots=%2d tile=%5d B  smem=%6d  %8.1f GB/s  (%.1f us)  err=%s\n", name, SLOTS, TILE_ROWS * 256, smem,
           bytes / (ms * 1e-3) / 1e9, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d_order);
    cudaFree(sink);
}

int main(int argc, char** argv) {
    size_t bytes = 8ull << 30;
    void* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    size_t rows = bytes / 256;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int tiles = argc > 1 ? atoi(argv[1]) : 400;
    run<4, 64>(buf, rows, sms, tiles, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, "64-row tiles");
    run<8, 64>(buf, rows, sms, tiles, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, "64-row tiles");
    run<12, 64>(buf, rows, sms, tiles, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, "64-row tiles");
    run<6, 128>(buf, rows, sms, tiles / 2, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, "128-row tiles");
    return 0;
}
