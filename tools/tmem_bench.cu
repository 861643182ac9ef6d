// Microbenchmark: TMEM load/store throughput and latency on this B200 (tcgen05.ld/st 32x32b).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2512_04752_b200/csrc -o tmem_bench tmem_bench.cu
#include <cuda_runtime.h>
#include <stdio.h>

#include "sm100_ptx.cuh"

using namespace rs::ptx;

template <int NWARPS, int MODE>   // MODE 0: ld.x16 + wait each; 1: 4 x ld.x16 then wait; 2: ld.x32 + wait; 3: st.x32
__global__ void __launch_bounds__(NWARPS * 32, 1) tmem_kernel(unsigned long long* out, int iters) {
    __shared__ uint32_t base;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<512>(&base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t = base + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
    uint32_t acc = 0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (MODE == 0) {
            uint32_t r[16];
            tmem_ld16(t + (i & 3) * 16, r);
            tmem_wait_ld();
            acc += r[0] ^ r[15];
        } else if (MODE == 1) {
            uint32_t r[4][16];
#pragma unroll
            for (int k = 0; k < 4; ++k) tmem_ld16(t + k * 16, r[k]);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 4; ++k) acc += r[k][0] ^ r[k][15];
        } else if (MODE == 2) {
            uint32_t r[32];
            tmem_ld32(t + (i & 1) * 32, r);
            tmem_wait_ld();
            acc += r[0] ^ r[31];
        } else {
            uint32_t r[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) r[k] = acc + k;
            tmem_st32(t + (i & 1) * 32, r);
            tmem_wait_st();
            acc += 1;
        }
    }
    const unsigned long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 0x12345) out[1 << 20] = acc;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<512>(base);
}

template <int NW, int MODE>
void run(const char* name, unsigned long long* d, int bytes_per_iter_per_warp) {
    const int iters = 2000;
    tmem_kernel<NW, MODE><<<148, NW * 32>>>(d, iters);
    cudaDeviceSynchronize();
    unsigned long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    double cyc_per_iter = (double)c / iters;
    printf("%-28s warps=%2d  %7.1f cycles/iter  -> %7.1f B/cycle/SM  err=%s\n", name, NW, cyc_per_iter,
           NW * (double)bytes_per_iter_per_warp / cyc_per_iter, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, (1 << 20) * 8 + 64);
    run<4, 0>("ld.x16 + wait", d, 32 * 16 * 4);
    run<8, 0>("ld.x16 + wait", d, 32 * 16 * 4);
    run<4, 1>("4 x ld.x16, 1 wait", d, 4 * 32 * 16 * 4);
    run<8, 1>("4 x ld.x16, 1 wait", d, 4 * 32 * 16 * 4);
    run<4, 2>("ld.x32 + wait", d, 32 * 32 * 4);
    run<8, 2>("ld.x32 + wait", d, 32 * 32 * 4);
    run<1, 2>("ld.x32 + wait (1 warp)", d, 32 * 32 * 4);
    run<4, 3>("st.x32 + wait", d, 32 * 32 * 4);
    run<8, 3>("st.x32 + wait", d, 32 * 32 * 4);
    return 0;
}
