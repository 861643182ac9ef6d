// Test-only kernel (not part of the product library): an UPSTREAM writer of tree-slot K/V that
// lets the next kernel on the stream start early. It executes griddepcontrol.launch_dependents
// first (so a PDL-launched rs_tree_verify_attention may begin at once), spins for `spin_ns`,
// then writes rows of the K and V page pools. Used by tests/test_gpu_pdl.py to check that the
// attention kernel reads no tree-slot K/V before griddepcontrol.wait (header: PDL).
#include <cstdint>
#include <cuda_runtime.h>

__global__ void pdl_write_rows(uint4* __restrict__ k, uint4* __restrict__ v, const int64_t* __restrict__ rows,
                               int n_rows, int row_vecs, const uint4* __restrict__ src_k,
                               const uint4* __restrict__ src_v, unsigned long long spin_ns) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < spin_ns);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)n_rows * row_vecs;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / row_vecs, c = i % row_vecs;
        k[rows[r] * row_vecs + c] = src_k[i];
        v[rows[r] * row_vecs + c] = src_v[i];
    }
}

extern "C" int pdl_test_write_rows(void* k_pages, void* v_pages, const int64_t* rows, int n_rows, int row_bytes,
                                   const void* src_k, const void* src_v, unsigned long long spin_ns, void* stream) {
    if (row_bytes % 16) return 1;
    pdl_write_rows<<<64, 128, 0, (cudaStream_t)stream>>>((uint4*)k_pages, (uint4*)v_pages, rows, n_rows,
                                                         row_bytes / 16, (const uint4*)src_k, (const uint4*)src_v,
                                                         spin_ns);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
