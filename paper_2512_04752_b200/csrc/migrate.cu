// a5: KV migration between generation instances (§6.2).
//   phase 1: pack the samples' KV from the paged store into ONE pre-allocated contiguous
//            buffer, hierarchically model -> layer -> sample (reading Z18: per segment
//            K then V, each [Hkv][len][d]);
//   phase 2: allocation handshake — the source sends a request with the memory needed, the
//            destination reserves pages all-or-nothing and answers; on refusal the source
//            keeps its samples and the call reports RS_ERR_NO_MEMORY;
//   phase 3: transfer (NCCL send/recv over NVLink) and unpack into the reserved pages.
// Migration is blocking in this build (reading Z14): the sample is paused during its transfer.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#ifdef RS_HAVE_NCCL
#include <nccl.h>
#endif

namespace {

constexpr int kMaxLayers = 256;
constexpr int kThreads = 256;

struct LayerPtrs {
    void* k[kMaxLayers];
    void* v[kMaxLayers];
};

// One CTA per (sample, layer, K|V). Buffer segment of (layer l, sample s):
//   base + l * 2*Hkv*d*sum(lens) + 2*Hkv*d*prefix(lens, s) ; K first, then V, each [Hkv][len][d].
// For one (page, head) the cache holds the page's rows contiguously ([pages][Hkv][ps][d]) and the
// buffer holds that head's tokens contiguously, so the copy is a sequence of contiguous runs of
// up to ps*d*2 bytes (16 KB at d = 128): all 256 threads stream 16-byte vectors of one run at a
// time, with the index arithmetic done once per run.
template <bool PACK>
__global__ void __launch_bounds__(kThreads)
kv_pack_kernel(LayerPtrs layers, int Hkv, int d, int ps, const int32_t* __restrict__ block_table, int max_pages,
               const int32_t* __restrict__ rows, const int32_t* __restrict__ starts, const int32_t* __restrict__ lens,
               int n, uint4* buf) {
    const int s = blockIdx.x, l = blockIdx.y, kv = blockIdx.z;
    long long total = 0, before = 0;
    for (int i = 0; i < n; ++i) {
        const int li = __ldg(lens + i);
        if (i < s) before += li;
        total += li;
    }
    const int len = __ldg(lens + s);                          // tokens [st0, st0 + len) of the sample
    const int st0 = starts ? __ldg(starts + s) : 0;
    if (len <= 0) return;
    const int vpr = d / 8;                                   // 16-byte vectors per token row
    uint4* seg = buf + ((long long)l * 2 * Hkv * total + 2LL * Hkv * before + (long long)kv * Hkv * len) * vpr;
    uint4* cache = reinterpret_cast<uint4*>(kv ? layers.v[l] : layers.k[l]);
    const int32_t* bt = block_table + (int64_t)__ldg(rows + s) * max_pages;
    const int pg0 = st0 / ps, npg = (st0 + len - 1) / ps - pg0 + 1;
    for (int run = 0; run < npg * Hkv; ++run) {
        const int pg = pg0 + run / Hkv, h = run % Hkv;
        const int t0 = max(st0, pg * ps);
        const int nt = min(st0 + len, (pg + 1) * ps) - t0;   // tokens of the range on this page
        uint4* c = cache + (((long long)__ldg(bt + pg) * Hkv + h) * ps + (t0 - pg * ps)) * vpr;
        uint4* bsg = seg + ((long long)h * len + (t0 - st0)) * vpr;
        const int nv = nt * vpr;
        const uint4* src = PACK ? c : bsg;
        uint4* dst = PACK ? bsg : c;
        for (int e0 = threadIdx.x; e0 < nv; e0 += 4 * kThreads) {   // 4 loads in flight, then 4 stores
            uint4 x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (e0 + u * kThreads < nv) x[u] = src[e0 + u * kThreads];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (e0 + u * kThreads < nv) dst[e0 + u * kThreads] = x[u];
        }
    }
}

template <bool PACK>
rs_status launch_pack(void* const* k_layers, void* const* v_layers, int32_t L, int32_t Hkv, int32_t d, int32_t ps,
                      const int32_t* block_table, int32_t max_pages, const int32_t* rows, const int32_t* starts,
                      const int32_t* lens, int32_t n, void* buf, int64_t off, cudaStream_t st) {
    RS_REQUIRE(L >= 0 && L <= kMaxLayers && Hkv > 0 && d % 8 == 0 && ps > 0 && n >= 0, RS_ERR_INVALID_ARG,
               "rs_kv_pack/unpack: bad sizes");
    RS_REQUIRE(off % 8 == 0 && (reinterpret_cast<uintptr_t>(buf) & 15) == 0, RS_ERR_INVALID_ARG,
               "rs_kv_pack/unpack: buffer offset must be 16-byte aligned");
    if (n == 0 || L == 0) return RS_OK;
    RS_REQUIRE(k_layers && v_layers && block_table && rows && lens && buf, RS_ERR_INVALID_ARG,
               "rs_kv_pack/unpack: null pointer");
    LayerPtrs lp;
    for (int i = 0; i < L; ++i) {
        lp.k[i] = k_layers[i];
        lp.v[i] = v_layers[i];
    }
    dim3 grid(n, L, 2);
    kv_pack_kernel<PACK><<<grid, kThreads, 0, st>>>(lp, Hkv, d, ps, block_table, max_pages, rows, starts, lens, n,
                                                    reinterpret_cast<uint4*>(static_cast<uint16_t*>(buf) + off));
    RS_LAUNCH_CHECK();
    return RS_OK;
}

}  // namespace

extern "C" int64_t rs_kv_pack_elems(int32_t L, int32_t Hkv, int32_t head_dim, const int32_t* lens_host, int32_t n) {
    int64_t tok = 0;
    for (int i = 0; i < n; ++i) tok += lens_host[i];
    return (int64_t)L * 2 * Hkv * head_dim * tok;
}

extern "C" rs_status rs_kv_pack(void* const* k_layers_host, void* const* v_layers_host, int32_t L, int32_t Hkv,
                                int32_t head_dim, int32_t page_size, const int32_t* block_table, int32_t max_pages,
                                const int32_t* sample_rows, const int32_t* lens, int32_t n, void* buf,
                                int64_t buf_offset_elems, void* stream) {
    rs::bind_device(block_table);
    return launch_pack<true>(k_layers_host, v_layers_host, L, Hkv, head_dim, page_size, block_table, max_pages,
                             sample_rows, nullptr, lens, n, buf, buf_offset_elems, rs::as_stream(stream));
}

extern "C" rs_status rs_kv_pack_range(void* const* k_layers_host, void* const* v_layers_host, int32_t L, int32_t Hkv,
                                      int32_t head_dim, int32_t page_size, const int32_t* block_table,
                                      int32_t max_pages, const int32_t* sample_rows, const int32_t* starts,
                                      const int32_t* lens, int32_t n, void* buf, int64_t buf_offset_elems,
                                      void* stream) {
    rs::bind_device(block_table);
    return launch_pack<true>(k_layers_host, v_layers_host, L, Hkv, head_dim, page_size, block_table, max_pages,
                             sample_rows, starts, lens, n, buf, buf_offset_elems, rs::as_stream(stream));
}

extern "C" rs_status rs_kv_unpack_range(void* const* k_layers_host, void* const* v_layers_host, int32_t L,
                                        int32_t Hkv, int32_t head_dim, int32_t page_size, const int32_t* block_table,
                                        int32_t max_pages, const int32_t* sample_rows, const int32_t* starts,
                                        const int32_t* lens, int32_t n, const void* buf, int64_t buf_offset_elems,
                                        void* stream) {
    rs::bind_device(block_table);
    return launch_pack<false>(k_layers_host, v_layers_host, L, Hkv, head_dim, page_size, block_table, max_pages,
                              sample_rows, starts, lens, n, const_cast<void*>(buf), buf_offset_elems,
                              rs::as_stream(stream));
}

extern "C" rs_status rs_kv_unpack(void* const* k_layers_host, void* const* v_layers_host, int32_t L, int32_t Hkv,
                                  int32_t head_dim, int32_t page_size, const int32_t* block_table, int32_t max_pages,
                                  const int32_t* sample_rows, const int32_t* lens, int32_t n, const void* buf,
                                  int64_t buf_offset_elems, void* stream) {
    rs::bind_device(block_table);
    return launch_pack<false>(k_layers_host, v_layers_host, L, Hkv, head_dim, page_size, block_table, max_pages,
                              sample_rows, nullptr, lens, n, const_cast<void*>(buf), buf_offset_elems,
                              rs::as_stream(stream));
}

// ------------------------------------------------------------------ page pool (host)
struct rs_page_pool {
    std::vector<int32_t> free_list;   // LIFO stack of free page ids
    std::vector<uint8_t> in_use;
};

extern "C" rs_status rs_page_pool_create(int32_t num_pages, rs_page_pool** out) {
    RS_REQUIRE(out && num_pages >= 0, RS_ERR_INVALID_ARG, "rs_page_pool_create: bad args");
    auto* p = new rs_page_pool();
    p->in_use.assign(num_pages, 0);
    p->free_list.resize(num_pages);
    for (int i = 0; i < num_pages; ++i) p->free_list[i] = num_pages - 1 - i;   // pops 0, 1, 2, ...
    *out = p;
    return RS_OK;
}

extern "C" void rs_page_pool_destroy(rs_page_pool* pool) { delete pool; }

extern "C" int32_t rs_page_pool_free_count(const rs_page_pool* pool) {
    return pool ? (int32_t)pool->free_list.size() : 0;
}

extern "C" rs_status rs_page_pool_alloc(rs_page_pool* pool, int32_t n, int32_t* pages_out) {
    RS_REQUIRE(pool && n >= 0 && (n == 0 || pages_out), RS_ERR_INVALID_ARG, "rs_page_pool_alloc: bad args");
    if ((size_t)n > pool->free_list.size()) {
        rs::set_error("rs_page_pool_alloc: %d pages requested, %zu free", n, pool->free_list.size());
        return RS_ERR_NO_MEMORY;   // all-or-nothing: nothing reserved
    }
    for (int i = 0; i < n; ++i) {
        const int32_t pg = pool->free_list.back();
        pool->free_list.pop_back();
        pool->in_use[pg] = 1;
        pages_out[i] = pg;
    }
    return RS_OK;
}

extern "C" rs_status rs_page_pool_free(rs_page_pool* pool, const int32_t* pages, int32_t n) {
    RS_REQUIRE(pool && n >= 0 && (n == 0 || pages), RS_ERR_INVALID_ARG, "rs_page_pool_free: bad args");
    for (int i = 0; i < n; ++i) {
        const int32_t pg = pages[i];
        RS_REQUIRE(pg >= 0 && pg < (int32_t)pool->in_use.size() && pool->in_use[pg], RS_ERR_INVALID_ARG,
                   "rs_page_pool_free: page %d not allocated", pg);
        pool->in_use[pg] = 0;
        pool->free_list.push_back(pg);
    }
    return RS_OK;
}

// Destination side of the allocation handshake: reserve the pages for every sample of
// the request, all-or-nothing, and build the destination block-table rows.
extern "C" rs_status rs_migrate_reserve(rs_page_pool* pool, const int32_t* lens_host, int32_t n, int32_t page_size,
                                        int32_t max_pages, int32_t* block_table_rows_out) {
    RS_REQUIRE(pool && n >= 0 && page_size > 0 && max_pages > 0, RS_ERR_INVALID_ARG, "rs_migrate_reserve: bad args");
    int64_t need = 0;
    for (int i = 0; i < n; ++i) {
        const int np = (lens_host[i] + page_size - 1) / page_size;
        RS_REQUIRE(np <= max_pages, RS_ERR_INVALID_ARG, "rs_migrate_reserve: sample %d needs %d pages > %d", i, np,
                   max_pages);
        need += np;
    }
    std::vector<int32_t> pages(need);
    rs_status st = rs_page_pool_alloc(pool, (int32_t)need, pages.data());
    if (st != RS_OK) return st;
    int64_t o = 0;
    for (int i = 0; i < n; ++i) {
        const int np = (lens_host[i] + page_size - 1) / page_size;
        for (int k = 0; k < max_pages; ++k)
            block_table_rows_out[(int64_t)i * max_pages + k] = k < np ? pages[o + k] : (np ? pages[o + np - 1] : 0);
        o += np;
    }
    return RS_OK;
}

// ------------------------------------------------------------------ NCCL communicator
struct rs_comm {
    int rank = 0, world = 1;
#ifdef RS_HAVE_NCCL
    ncclComm_t nccl = nullptr;
#endif
    int64_t* d_hdr = nullptr;   // device scratch for header / status messages
    int64_t* h_hdr = nullptr;   // pinned host mirror
};

extern "C" rs_status rs_comm_unique_id(uint8_t* id_out_128) {
#ifdef RS_HAVE_NCCL
    RS_REQUIRE(id_out_128, RS_ERR_INVALID_ARG, "rs_comm_unique_id: null");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    RS_REQUIRE(r == ncclSuccess, RS_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    memcpy(id_out_128, &id, 128);
    return RS_OK;
#else
    (void)id_out_128;
    rs::set_error("built without NCCL");
    return RS_ERR_UNSUPPORTED;
#endif
}

static constexpr int kHdrMax = 4 + 2 * 4096;   // n, total, status, reserved, lens[...], gids[...]

extern "C" rs_status rs_comm_create(const uint8_t* id_128, int32_t rank, int32_t world, rs_comm** out) {
#ifdef RS_HAVE_NCCL
    RS_REQUIRE(id_128 && out && world >= 1 && rank >= 0 && rank < world, RS_ERR_INVALID_ARG,
               "rs_comm_create: bad args");
    auto* c = new rs_comm();
    c->rank = rank;
    c->world = world;
    ncclUniqueId id;
    memcpy(&id, id_128, 128);
    ncclResult_t r = ncclCommInitRank(&c->nccl, world, id, rank);
    if (r != ncclSuccess) {
        delete c;
        rs::set_error("ncclCommInitRank: %s", ncclGetErrorString(r));
        return RS_ERR_NCCL;
    }
    if (cudaMalloc(&c->d_hdr, sizeof(int64_t) * kHdrMax) != cudaSuccess ||
        cudaMallocHost(&c->h_hdr, sizeof(int64_t) * kHdrMax) != cudaSuccess) {
        ncclCommDestroy(c->nccl);
        delete c;
        rs::set_error("rs_comm_create: scratch allocation failed");
        return RS_ERR_CUDA;
    }
    *out = c;
    return RS_OK;
#else
    (void)id_128; (void)rank; (void)world; (void)out;
    rs::set_error("built without NCCL");
    return RS_ERR_UNSUPPORTED;
#endif
}

extern "C" rs_status rs_comm_destroy(rs_comm* c) {
    if (!c) return RS_OK;
#ifdef RS_HAVE_NCCL
    if (c->nccl) ncclCommDestroy(c->nccl);
#endif
    if (c->d_hdr) cudaFree(c->d_hdr);
    if (c->h_hdr) cudaFreeHost(c->h_hdr);
    delete c;
    return RS_OK;
}

#ifdef RS_HAVE_NCCL
// Point-to-point message from src to dst (both ranks call; src == dst is a local copy).
static rs_status p2p(rs_comm* c, int src, int dst, void* buf, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return RS_OK;
    ncclResult_t r = ncclGroupStart();
    if (r == ncclSuccess && c->rank == src) r = ncclSend(buf, bytes, ncclUint8, dst, c->nccl, st);
    if (r == ncclSuccess && c->rank == dst) r = ncclRecv(buf, bytes, ncclUint8, src, c->nccl, st);
    ncclResult_t r2 = ncclGroupEnd();
    RS_REQUIRE(r == ncclSuccess && r2 == ncclSuccess, RS_ERR_NCCL, "NCCL p2p %d->%d: %s", src, dst,
               ncclGetErrorString(r != ncclSuccess ? r : r2));
    return RS_OK;
}
#endif

extern "C" rs_status rs_migrate_samples(rs_comm* c, int32_t src_rank, int32_t dst_rank, const rs_kv_desc* kv,
                                        rs_page_pool* pool, const int64_t* gids_host, const int32_t* lens_host,
                                        int32_t n, const int32_t* src_block_table, int32_t max_pages,
                                        int32_t* dst_block_table_host, void* staging, size_t staging_bytes,
                                        int32_t* device_scratch, void* stream) {
    rs::bind_device(device_scratch);
#ifdef RS_HAVE_NCCL
    RS_REQUIRE(c && kv && n >= 0 && n <= 4096 && src_rank >= 0 && dst_rank >= 0 && src_rank < c->world &&
                   dst_rank < c->world,
               RS_ERR_INVALID_ARG, "rs_migrate_samples: bad args");
    const bool is_src = c->rank == src_rank, is_dst = c->rank == dst_rank;
    if (!is_src && !is_dst) return RS_OK;
    cudaStream_t st = rs::as_stream(stream);
    // ---- phase 2a: request header src -> dst: [n, bytes, -, -, lens..., gids...]
    const int64_t hdr_len = 4 + 2 * (int64_t)n;
    int64_t bytes = 0;
    if (is_src) {
        RS_REQUIRE(lens_host && gids_host, RS_ERR_INVALID_ARG, "rs_migrate_samples: src needs lens and gids");
        const int64_t e_ssm = kv->L_ssm ? rs_kv_pack_elems(kv->L_ssm, kv->Hkv_ssm, kv->d_ssm, lens_host, n) : 0;
        const int64_t e_llm = rs_kv_pack_elems(kv->L_llm, kv->Hkv_llm, kv->d_llm, lens_host, n);
        bytes = 2 * (e_ssm + e_llm);
        c->h_hdr[0] = n;
        c->h_hdr[1] = bytes;
        c->h_hdr[2] = 0;
        c->h_hdr[3] = 0;
        for (int i = 0; i < n; ++i) {
            c->h_hdr[4 + i] = lens_host[i];
            c->h_hdr[4 + n + i] = gids_host[i];
        }
        RS_CUDA_CHECK(cudaMemcpyAsync(c->d_hdr, c->h_hdr, sizeof(int64_t) * hdr_len, cudaMemcpyHostToDevice, st));
    }
    rs_status s = p2p(c, src_rank, dst_rank, c->d_hdr, sizeof(int64_t) * hdr_len, st);
    if (s != RS_OK) return s;
    std::vector<int32_t> lens(n);
    int64_t status = RS_OK;
    if (is_dst) {
        RS_CUDA_CHECK(cudaMemcpyAsync(c->h_hdr, c->d_hdr, sizeof(int64_t) * hdr_len, cudaMemcpyDeviceToHost, st));
        RS_CUDA_CHECK(cudaStreamSynchronize(st));
        RS_REQUIRE(c->h_hdr[0] == n, RS_ERR_LAYOUT_MISMATCH, "rs_migrate_samples: header n %lld != %d",
                   (long long)c->h_hdr[0], n);
        bytes = c->h_hdr[1];
        for (int i = 0; i < n; ++i) lens[i] = (int32_t)c->h_hdr[4 + i];
        // ---- phase 2b: reserve (all-or-nothing) and answer; every refusal is answered so the
        // source never blocks on a transfer that will not come
        if ((size_t)bytes > staging_bytes || !staging || !pool || !dst_block_table_host)
            status = RS_ERR_WORKSPACE;
        else
            status = rs_migrate_reserve(pool, lens.data(), n, kv->page_size, max_pages, dst_block_table_host);
        c->h_hdr[2] = status;
        RS_CUDA_CHECK(cudaMemcpyAsync(c->d_hdr + 2, c->h_hdr + 2, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    } else {
        for (int i = 0; i < n; ++i) lens[i] = lens_host[i];
    }
    s = p2p(c, dst_rank, src_rank, c->d_hdr + 2, sizeof(int64_t), st);
    if (s != RS_OK) return s;
    if (is_src && !is_dst) {
        RS_CUDA_CHECK(cudaMemcpyAsync(c->h_hdr + 2, c->d_hdr + 2, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        RS_CUDA_CHECK(cudaStreamSynchronize(st));
        status = c->h_hdr[2];
    }
    if (status != RS_OK) {
        rs::set_error("rs_migrate_samples: destination refused the request (status %lld)", (long long)status);
        return status == RS_ERR_NO_MEMORY ? RS_ERR_NO_MEMORY : RS_ERR_WORKSPACE;   // source unchanged
    }
    RS_REQUIRE(device_scratch, RS_ERR_INVALID_ARG, "rs_migrate_samples: device_scratch required");
    RS_REQUIRE((size_t)bytes <= staging_bytes && staging, RS_ERR_WORKSPACE, "rs_migrate_samples: staging too small");
    // device scratch: [n] rows (0..n-1) | [n] lens | [n*max_pages] dst block-table rows
    int32_t* d_rows = device_scratch;
    int32_t* d_lens = device_scratch + n;
    int32_t* d_bt = device_scratch + 2 * n;
    std::vector<int32_t> rows(n);
    for (int i = 0; i < n; ++i) rows[i] = i;
    RS_CUDA_CHECK(cudaMemcpyAsync(d_rows, rows.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    RS_CUDA_CHECK(cudaMemcpyAsync(d_lens, lens.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    const int64_t e_ssm = kv->L_ssm ? rs_kv_pack_elems(kv->L_ssm, kv->Hkv_ssm, kv->d_ssm, lens.data(), n) : 0;
    // ---- phase 1: pack (model order SSM, LLM)
    if (is_src) {
        RS_REQUIRE(src_block_table, RS_ERR_INVALID_ARG, "rs_migrate_samples: src block table required");
        if (kv->L_ssm) {
            s = rs_kv_pack(kv->k_ssm, kv->v_ssm, kv->L_ssm, kv->Hkv_ssm, kv->d_ssm, kv->page_size, src_block_table,
                           max_pages, d_rows, d_lens, n, staging, 0, stream);
            if (s != RS_OK) return s;
        }
        s = rs_kv_pack(kv->k_llm, kv->v_llm, kv->L_llm, kv->Hkv_llm, kv->d_llm, kv->page_size, src_block_table,
                       max_pages, d_rows, d_lens, n, staging, e_ssm, stream);
        if (s != RS_OK) return s;
    }
    // ---- phase 2c: one contiguous transfer
    s = p2p(c, src_rank, dst_rank, staging, (size_t)bytes, st);
    if (s != RS_OK) return s;
    // ---- phase 3: unpack into the reserved pages
    if (is_dst) {
        RS_CUDA_CHECK(cudaMemcpyAsync(d_bt, dst_block_table_host, sizeof(int32_t) * n * max_pages,
                                      cudaMemcpyHostToDevice, st));
        if (kv->L_ssm) {
            s = rs_kv_unpack(kv->k_ssm, kv->v_ssm, kv->L_ssm, kv->Hkv_ssm, kv->d_ssm, kv->page_size, d_bt, max_pages,
                             d_rows, d_lens, n, staging, 0, stream);
            if (s != RS_OK) return s;
        }
        s = rs_kv_unpack(kv->k_llm, kv->v_llm, kv->L_llm, kv->Hkv_llm, kv->d_llm, kv->page_size, d_bt, max_pages,
                         d_rows, d_lens, n, staging, e_ssm, stream);
        if (s != RS_OK) return s;
    }
    RS_CUDA_CHECK(cudaStreamSynchronize(st));
    return RS_OK;
#else
    (void)c; (void)src_rank; (void)dst_rank; (void)kv; (void)pool; (void)gids_host; (void)lens_host; (void)n;
    (void)src_block_table; (void)max_pages; (void)dst_block_table_host; (void)staging; (void)staging_bytes;
    (void)device_scratch; (void)stream;
    rs::set_error("built without NCCL");
    return RS_ERR_UNSUPPORTED;
#endif
}

// ------------------------------------------------------------------ f1: two-stage migration
// P:303-318. Stage 1 moves the KV of the tokens verified before the trigger while both instances
// keep computing: later verification steps only write slots beyond them (Markov property), so
// the transfer is enqueued on a side stream and the call returns. Stage 2 moves the tokens
// verified meanwhile with the SSM part first (the destination can resume drafting once it has
// landed) and the LLM part behind it.
#ifdef RS_HAVE_NCCL
namespace {
// Request src -> dst: [n, bytes, status, -, A[n], B[n]]; the destination decides and answers
// one status word. Returns RS_OK when the transfer may proceed (on both ranks).
template <class Decide>
rs_status handshake(rs_comm* c, int src, int dst, int n, int64_t bytes_src, const int32_t* A_src,
                    const int32_t* B_src, std::vector<int32_t>& A, std::vector<int32_t>& B, cudaStream_t st,
                    Decide decide, const char* what) {
    const bool is_src = c->rank == src, is_dst = c->rank == dst;
    const int64_t len = 4 + 2 * (int64_t)n;
    A.assign(n, 0);
    B.assign(n, 0);
    if (is_src) {
        c->h_hdr[0] = n;
        c->h_hdr[1] = bytes_src;
        c->h_hdr[2] = 0;
        c->h_hdr[3] = 0;
        for (int i = 0; i < n; ++i) {
            c->h_hdr[4 + i] = A_src[i];
            c->h_hdr[4 + n + i] = B_src[i];
            A[i] = A_src[i];
            B[i] = B_src[i];
        }
        RS_CUDA_CHECK(cudaMemcpyAsync(c->d_hdr, c->h_hdr, sizeof(int64_t) * len, cudaMemcpyHostToDevice, st));
    }
    rs_status s = p2p(c, src, dst, c->d_hdr, sizeof(int64_t) * len, st);
    if (s != RS_OK) return s;
    int64_t status = RS_OK;
    if (is_dst) {
        RS_CUDA_CHECK(cudaMemcpyAsync(c->h_hdr, c->d_hdr, sizeof(int64_t) * len, cudaMemcpyDeviceToHost, st));
        RS_CUDA_CHECK(cudaStreamSynchronize(st));
        RS_REQUIRE(c->h_hdr[0] == n, RS_ERR_LAYOUT_MISMATCH, "%s: header n %lld != %d", what, (long long)c->h_hdr[0], n);
        for (int i = 0; i < n; ++i) {
            A[i] = (int32_t)c->h_hdr[4 + i];
            B[i] = (int32_t)c->h_hdr[4 + n + i];
        }
        status = decide(c->h_hdr[1], A, B);
        c->h_hdr[2] = status;
        RS_CUDA_CHECK(cudaMemcpyAsync(c->d_hdr + 2, c->h_hdr + 2, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    }
    s = p2p(c, dst, src, c->d_hdr + 2, sizeof(int64_t), st);
    if (s != RS_OK) return s;
    if (is_src && !is_dst) {
        RS_CUDA_CHECK(cudaMemcpyAsync(c->h_hdr + 2, c->d_hdr + 2, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        RS_CUDA_CHECK(cudaStreamSynchronize(st));
        status = c->h_hdr[2];
    }
    if (status != RS_OK) {
        rs::set_error("%s: destination refused the request (status %lld)", what, (long long)status);
        return status == RS_ERR_NO_MEMORY ? RS_ERR_NO_MEMORY : RS_ERR_WORKSPACE;
    }
    return RS_OK;
}

int64_t model_elems(int L, int Hkv, int d, const std::vector<int32_t>& lens) {
    return L ? rs_kv_pack_elems(L, Hkv, d, lens.data(), (int32_t)lens.size()) : 0;
}
}  // namespace
#endif

extern "C" rs_status rs_migrate_stage1(rs_comm* c, int32_t src_rank, int32_t dst_rank, const rs_kv_desc* kv,
                                       rs_page_pool* pool, const int64_t* gids_host, const int32_t* lens_host,
                                       const int32_t* reserve_lens_host, int32_t n, const int32_t* src_block_table,
                                       int32_t max_pages, int32_t* dst_block_table_host, void* staging,
                                       size_t staging_bytes, int32_t* device_scratch, void* stream) {
    rs::bind_device(device_scratch);
#ifdef RS_HAVE_NCCL
    RS_REQUIRE(c && kv && n >= 0 && n <= 4096 && src_rank >= 0 && dst_rank >= 0 && src_rank < c->world &&
                   dst_rank < c->world,
               RS_ERR_INVALID_ARG, "rs_migrate_stage1: bad args");
    const bool is_src = c->rank == src_rank, is_dst = c->rank == dst_rank;
    if (!is_src && !is_dst) return RS_OK;
    cudaStream_t st = rs::as_stream(stream);
    int64_t bytes = 0;
    if (is_src) {
        RS_REQUIRE(lens_host && reserve_lens_host && gids_host, RS_ERR_INVALID_ARG,
                   "rs_migrate_stage1: src needs lens, reserve_lens and gids");
        for (int i = 0; i < n; ++i)
            RS_REQUIRE(reserve_lens_host[i] >= lens_host[i], RS_ERR_INVALID_ARG,
                       "rs_migrate_stage1: reserve_lens[%d] < lens", i);
        std::vector<int32_t> ln(lens_host, lens_host + n);
        bytes = 2 * (model_elems(kv->L_ssm, kv->Hkv_ssm, kv->d_ssm, ln) +
                     model_elems(kv->L_llm, kv->Hkv_llm, kv->d_llm, ln));
    }
    std::vector<int32_t> lens, reserve;
    rs_status s = handshake(
        c, src_rank, dst_rank, n, bytes, lens_host, reserve_lens_host, lens, reserve, st,
        [&](int64_t b, std::vector<int32_t>&, std::vector<int32_t>& rsv) -> int64_t {
            bytes = b;
            if ((size_t)b > staging_bytes || !staging || !pool || !dst_block_table_host) return RS_ERR_WORKSPACE;
            return rs_migrate_reserve(pool, rsv.data(), n, kv->page_size, max_pages, dst_block_table_host);
        },
        "rs_migrate_stage1");
    if (s != RS_OK) return s;
    RS_REQUIRE(device_scratch && staging && (size_t)bytes <= staging_bytes, RS_ERR_WORKSPACE,
               "rs_migrate_stage1: staging / device_scratch");
    int32_t* d_rows = device_scratch;
    int32_t* d_lens = device_scratch + n;
    int32_t* d_bt = device_scratch + 2 * n;
    std::vector<int32_t> rows(n);
    for (int i = 0; i < n; ++i) rows[i] = i;
    RS_CUDA_CHECK(cudaMemcpyAsync(d_rows, rows.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    RS_CUDA_CHECK(cudaMemcpyAsync(d_lens, lens.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    const int64_t e_ssm = model_elems(kv->L_ssm, kv->Hkv_ssm, kv->d_ssm, lens);
    if (is_src) {
        RS_REQUIRE(src_block_table, RS_ERR_INVALID_ARG, "rs_migrate_stage1: src block table required");
        if (kv->L_ssm) {
            s = rs_kv_pack(kv->k_ssm, kv->v_ssm, kv->L_ssm, kv->Hkv_ssm, kv->d_ssm, kv->page_size, src_block_table,
                           max_pages, d_rows, d_lens, n, staging, 0, stream);
            if (s != RS_OK) return s;
        }
        s = rs_kv_pack(kv->k_llm, kv->v_llm, kv->L_llm, kv->Hkv_llm, kv->d_llm, kv->page_size, src_block_table,
                       max_pages, d_rows, d_lens, n, staging, e_ssm, stream);
        if (s != RS_OK) return s;
    }
    s = p2p(c, src_rank, dst_rank, staging, (size_t)bytes, st);
    if (s != RS_OK) return s;
    if (is_dst) {
        RS_CUDA_CHECK(cudaMemcpyAsync(d_bt, dst_block_table_host, sizeof(int32_t) * n * max_pages,
                                      cudaMemcpyHostToDevice, st));
        if (kv->L_ssm) {
            s = rs_kv_unpack(kv->k_ssm, kv->v_ssm, kv->L_ssm, kv->Hkv_ssm, kv->d_ssm, kv->page_size, d_bt, max_pages,
                             d_rows, d_lens, n, staging, 0, stream);
            if (s != RS_OK) return s;
        }
        s = rs_kv_unpack(kv->k_llm, kv->v_llm, kv->L_llm, kv->Hkv_llm, kv->d_llm, kv->page_size, d_bt, max_pages,
                         d_rows, d_lens, n, staging, e_ssm, stream);
        if (s != RS_OK) return s;
    }
    return RS_OK;   // enqueued; the caller waits on `stream` before stage 2
#else
    (void)c; (void)src_rank; (void)dst_rank; (void)kv; (void)pool; (void)gids_host; (void)lens_host;
    (void)reserve_lens_host; (void)n; (void)src_block_table; (void)max_pages; (void)dst_block_table_host;
    (void)staging; (void)staging_bytes; (void)device_scratch; (void)stream;
    rs::set_error("built without NCCL");
    return RS_ERR_UNSUPPORTED;
#endif
}

extern "C" rs_status rs_migrate_stage2(rs_comm* c, int32_t src_rank, int32_t dst_rank, const rs_kv_desc* kv,
                                       rs_page_pool* pool, const int32_t* starts_host, const int32_t* lens_host,
                                       int32_t n, const int32_t* src_block_table, int32_t max_pages,
                                       int32_t* dst_block_table_host, int32_t* dst_capacity_host, void* staging,
                                       size_t staging_bytes, int32_t* device_scratch, void* ssm_ready_event,
                                       void* stream) {
    rs::bind_device(device_scratch);
#ifdef RS_HAVE_NCCL
    RS_REQUIRE(c && kv && n >= 0 && n <= 4096 && src_rank >= 0 && dst_rank >= 0 && src_rank < c->world &&
                   dst_rank < c->world,
               RS_ERR_INVALID_ARG, "rs_migrate_stage2: bad args");
    const bool is_src = c->rank == src_rank, is_dst = c->rank == dst_rank;
    if (!is_src && !is_dst) return RS_OK;
    cudaStream_t st = rs::as_stream(stream);
    int64_t bytes = 0;
    if (is_src) {
        RS_REQUIRE(starts_host && lens_host, RS_ERR_INVALID_ARG, "rs_migrate_stage2: src needs starts and lens");
        std::vector<int32_t> ln(lens_host, lens_host + n);
        bytes = 2 * (model_elems(kv->L_ssm, kv->Hkv_ssm, kv->d_ssm, ln) +
                     model_elems(kv->L_llm, kv->Hkv_llm, kv->d_llm, ln));
    }
    const int ps = kv->page_size;
    std::vector<int32_t> starts, lens;
    rs_status s = handshake(
        c, src_rank, dst_rank, n, bytes, starts_host, lens_host, starts, lens, st,
        [&](int64_t b, std::vector<int32_t>& stt, std::vector<int32_t>& ln) -> int64_t {
            bytes = b;
            if ((size_t)b > staging_bytes || !staging || !pool || !dst_block_table_host || !dst_capacity_host)
                return RS_ERR_WORKSPACE;
            // pages beyond each row's reservation, all-or-nothing
            int64_t extra = 0;
            for (int i = 0; i < n; ++i) {
                const int need = (stt[i] + ln[i] + ps - 1) / ps, have = (dst_capacity_host[i] + ps - 1) / ps;
                if (need > max_pages) return RS_ERR_INVALID_ARG;
                extra += std::max(0, need - have);
            }
            if (extra == 0) return RS_OK;
            std::vector<int32_t> pages(extra);
            const rs_status a = rs_page_pool_alloc(pool, (int32_t)extra, pages.data());
            if (a != RS_OK) return a;
            int64_t o = 0;
            for (int i = 0; i < n; ++i) {
                const int need = (stt[i] + ln[i] + ps - 1) / ps, have = (dst_capacity_host[i] + ps - 1) / ps;
                int32_t* row = dst_block_table_host + (int64_t)i * max_pages;
                for (int k = have; k < need; ++k) row[k] = pages[o++];
                if (need > have)
                    for (int k = need; k < max_pages; ++k) row[k] = row[need - 1];
                if (need * ps > dst_capacity_host[i]) dst_capacity_host[i] = std::max(dst_capacity_host[i], need * ps);
            }
            return RS_OK;
        },
        "rs_migrate_stage2");
    if (s != RS_OK) return s;
    RS_REQUIRE(device_scratch && staging && (size_t)bytes <= staging_bytes, RS_ERR_WORKSPACE,
               "rs_migrate_stage2: staging / device_scratch");
    int32_t* d_rows = device_scratch;
    int32_t* d_starts = device_scratch + n;
    int32_t* d_lens = device_scratch + 2 * n;
    int32_t* d_bt = device_scratch + 3 * n;
    std::vector<int32_t> rows(n);
    for (int i = 0; i < n; ++i) rows[i] = i;
    RS_CUDA_CHECK(cudaMemcpyAsync(d_rows, rows.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    RS_CUDA_CHECK(cudaMemcpyAsync(d_starts, starts.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    RS_CUDA_CHECK(cudaMemcpyAsync(d_lens, lens.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    if (is_dst)
        RS_CUDA_CHECK(cudaMemcpyAsync(d_bt, dst_block_table_host, sizeof(int32_t) * n * max_pages,
                                      cudaMemcpyHostToDevice, st));
    RS_REQUIRE(!is_src || src_block_table, RS_ERR_INVALID_ARG, "rs_migrate_stage2: src block table required");
    const int64_t e_ssm = model_elems(kv->L_ssm, kv->Hkv_ssm, kv->d_ssm, lens);
    // SSM part first: drafting resumes on the destination as soon as it has landed
    if (kv->L_ssm) {
        if (is_src) {
            s = rs_kv_pack_range(kv->k_ssm, kv->v_ssm, kv->L_ssm, kv->Hkv_ssm, kv->d_ssm, ps, src_block_table,
                                 max_pages, d_rows, d_starts, d_lens, n, staging, 0, stream);
            if (s != RS_OK) return s;
        }
        s = p2p(c, src_rank, dst_rank, staging, (size_t)(2 * e_ssm), st);
        if (s != RS_OK) return s;
        if (is_dst) {
            s = rs_kv_unpack_range(kv->k_ssm, kv->v_ssm, kv->L_ssm, kv->Hkv_ssm, kv->d_ssm, ps, d_bt, max_pages,
                                   d_rows, d_starts, d_lens, n, staging, 0, stream);
            if (s != RS_OK) return s;
        }
    }
    if (is_dst && ssm_ready_event) RS_CUDA_CHECK(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ssm_ready_event), st));
    if (is_src) {
        s = rs_kv_pack_range(kv->k_llm, kv->v_llm, kv->L_llm, kv->Hkv_llm, kv->d_llm, ps, src_block_table, max_pages,
                             d_rows, d_starts, d_lens, n, staging, e_ssm, stream);
        if (s != RS_OK) return s;
    }
    s = p2p(c, src_rank, dst_rank, static_cast<uint16_t*>(staging) + e_ssm, (size_t)(bytes - 2 * e_ssm), st);
    if (s != RS_OK) return s;
    if (is_dst) {
        s = rs_kv_unpack_range(kv->k_llm, kv->v_llm, kv->L_llm, kv->Hkv_llm, kv->d_llm, ps, d_bt, max_pages, d_rows,
                               d_starts, d_lens, n, staging, e_ssm, stream);
        if (s != RS_OK) return s;
    }
    return RS_OK;   // enqueued; the destination verifies the samples after `stream` reaches here
#else
    (void)c; (void)src_rank; (void)dst_rank; (void)kv; (void)pool; (void)starts_host; (void)lens_host; (void)n;
    (void)src_block_table; (void)max_pages; (void)dst_block_table_host; (void)dst_capacity_host; (void)staging;
    (void)staging_bytes; (void)device_scratch; (void)ssm_ready_event; (void)stream;
    rs::set_error("built without NCCL");
    return RS_ERR_UNSUPPORTED;
#endif
}
