// a5 over peer memory: KV migration between generation instances as ONE copy kernel that reads
// the source's pages from local HBM and stores them straight into the destination's reserved
// pages through a CUDA-IPC mapping of the destination's KV pools (NVLink P2P stores over
// NVSwitch when the instances sit on different GPUs; a device-local copy when two instance
// processes share one GPU). PAPER.md §6.2 describes migration as pack into one
// contiguous buffer -> transfer -> unpack; on B200 the pages are directly addressable from the
// peer, so the three phases collapse into one pass with no staging buffer: every 16 KB
// (page, head) run leaves the source once and lands in its final place, and the transfer is
// pipelined by construction (the first pages arrive while later ones are still being read).
// The allocation handshake is unchanged and stays with the caller (rs_migrate_reserve on
// the destination, rows sent back over the control plane). Completion travels as an
// inter-process CUDA event recorded by the source after its push and waited on by the
// destination's stream (no host synchronisation on either side).
#include <unistd.h>

#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"

namespace {

constexpr int kMaxLayers = 256;
constexpr int kThreads = 256;
constexpr int kMaxPeers = 64;
constexpr uint32_t kMagic = 0x52535052u;   // "RSPR"

struct LayerPtrs {
    void* k[kMaxLayers];
    void* v[kMaxLayers];
};

// Grid (n, L, 2*Hkv): one CTA per (sample, layer, K|V x kv head). The sample's token range
// [st0, st0 + len) covers logical pages pg0..pg1; on both sides logical slot j sits in row j % ps
// of page bt[j / ps] and a (page, head) tile is ps*d contiguous bf16, so the range is a sequence
// of contiguous runs (up to 16 KB at d = 128) at the same row offsets on both sides.
__global__ void __launch_bounds__(kThreads)
kv_push_kernel(LayerPtrs src, LayerPtrs dst, int Hkv, int d, int ps, const int32_t* __restrict__ src_bt,
               const int32_t* __restrict__ dst_bt, int max_pages, const int32_t* __restrict__ starts,
               const int32_t* __restrict__ lens) {
    const int s = blockIdx.x, l = blockIdx.y, kv = blockIdx.z / Hkv, h = blockIdx.z % Hkv;
    const int len = __ldg(lens + s);
    if (len <= 0) return;
    const int st0 = starts ? __ldg(starts + s) : 0;
    const int vpr = d / 8;   // 16-byte vectors per token row
    const uint4* sc = reinterpret_cast<const uint4*>(kv ? src.v[l] : src.k[l]);
    uint4* dc = reinterpret_cast<uint4*>(kv ? dst.v[l] : dst.k[l]);
    const int32_t* sbt = src_bt + (int64_t)s * max_pages;
    const int32_t* dbt = dst_bt + (int64_t)s * max_pages;
    const int pg0 = st0 / ps, pg1 = (st0 + len - 1) / ps;
    for (int pg = pg0; pg <= pg1; ++pg) {
        const int t0 = max(st0, pg * ps);
        const int nt = min(st0 + len, (pg + 1) * ps) - t0;
        const int64_t row = ((int64_t)h * ps + (t0 - pg * ps)) * vpr;
        const uint4* a = sc + (int64_t)__ldg(sbt + pg) * Hkv * ps * vpr + row;
        uint4* b = dc + (int64_t)__ldg(dbt + pg) * Hkv * ps * vpr + row;
        const int nv = nt * vpr;
        for (int e0 = threadIdx.x; e0 < nv; e0 += 4 * kThreads) {   // 4 loads in flight, then 4 stores
            uint4 x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (e0 + u * kThreads < nv) x[u] = __ldg(a + e0 + u * kThreads);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (e0 + u * kThreads < nv) b[e0 + u * kThreads] = x[u];
        }
    }
}

typedef int (*PFN_getAddressRange)(unsigned long long*, size_t*, unsigned long long);   // cuMemGetAddressRange_v2

PFN_getAddressRange get_range_fn() {
    static PFN_getAddressRange fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_getAddressRange>(ptr);
    }
    return fn;
}

// Serialised registration of one instance's store (host bytes, exchanged over the control plane).
struct BlobHeader {
    uint32_t magic, version;
    int32_t rank, pid;
    int32_t L_ssm, Hkv_ssm, d_ssm, L_llm, Hkv_llm, d_llm, page_size, n_ptrs;
    cudaIpcEventHandle_t ev[2];   // 0: push done, 1: SSM part landed
};
struct BlobEntry {
    cudaIpcMemHandle_t handle;    // of the allocation holding the pool
    uint64_t offset;              // pool pointer - allocation base
    uint64_t raw;                 // pool pointer in the exporting process (same-process imports)
};

struct Peer {
    bool present = false;
    bool local = false;           // same process: raw pointers, no IPC mapping
    std::vector<void*> ptrs;      // k_ssm[L_ssm], v_ssm[L_ssm], k_llm[L_llm], v_llm[L_llm]
    cudaEvent_t ev[2] = {nullptr, nullptr};
};

}  // namespace

struct rs_peer {
    int32_t rank = 0;
    int32_t L_ssm = 0, Hkv_ssm = 1, d_ssm = 8, L_llm = 0, Hkv_llm = 1, d_llm = 8, page_size = 64;
    std::vector<void*> ptrs;      // own pools, same order as Peer::ptrs
    cudaEvent_t ev[2] = {nullptr, nullptr};   // inter-process events this rank records
    Peer peers[kMaxPeers];
    std::map<std::string, void*> mapped;      // opened IPC allocations (handle bytes -> base), opened once
};

static int n_ptrs(const rs_peer* p) { return 2 * (p->L_ssm + p->L_llm); }

extern "C" rs_status rs_peer_create(const rs_kv_desc* kv, int32_t rank, rs_peer** out) {
    RS_REQUIRE(kv && out && rank >= 0 && rank < kMaxPeers, RS_ERR_INVALID_ARG, "rs_peer_create: bad args");
    RS_REQUIRE(kv->L_ssm >= 0 && kv->L_llm >= 0 && kv->L_ssm <= kMaxLayers && kv->L_llm <= kMaxLayers &&
                   kv->page_size > 0 && (kv->L_llm == 0 || (kv->Hkv_llm > 0 && kv->d_llm % 8 == 0)) &&
                   (kv->L_ssm == 0 || (kv->Hkv_ssm > 0 && kv->d_ssm % 8 == 0)),
               RS_ERR_INVALID_ARG, "rs_peer_create: bad KV description");
    auto* p = new rs_peer();
    p->rank = rank;
    p->L_ssm = kv->L_ssm; p->Hkv_ssm = kv->Hkv_ssm; p->d_ssm = kv->d_ssm;
    p->L_llm = kv->L_llm; p->Hkv_llm = kv->Hkv_llm; p->d_llm = kv->d_llm;
    p->page_size = kv->page_size;
    for (int i = 0; i < kv->L_ssm; ++i) p->ptrs.push_back(kv->k_ssm[i]);
    for (int i = 0; i < kv->L_ssm; ++i) p->ptrs.push_back(kv->v_ssm[i]);
    for (int i = 0; i < kv->L_llm; ++i) p->ptrs.push_back(kv->k_llm[i]);
    for (int i = 0; i < kv->L_llm; ++i) p->ptrs.push_back(kv->v_llm[i]);
    for (void* q : p->ptrs)
        if (!q || (reinterpret_cast<uintptr_t>(q) & 15)) {
            delete p;
            rs::set_error("rs_peer_create: null or unaligned pool pointer");
            return RS_ERR_INVALID_ARG;
        }
    rs::bind_device(p->ptrs.empty() ? nullptr : p->ptrs[0]);   // events on the pools' device
    for (int e = 0; e < 2; ++e)
        if (cudaEventCreateWithFlags(&p->ev[e], cudaEventDisableTiming | cudaEventInterprocess) != cudaSuccess) {
            rs::set_error("rs_peer_create: cudaEventCreate (interprocess) failed");
            delete p;
            return RS_ERR_CUDA;
        }
    *out = p;
    return RS_OK;
}

extern "C" size_t rs_peer_blob_bytes(const rs_peer* p) {
    return p ? sizeof(BlobHeader) + sizeof(BlobEntry) * n_ptrs(p) : 0;
}

extern "C" rs_status rs_peer_export(const rs_peer* p, uint8_t* blob, size_t bytes) {
    RS_REQUIRE(p && blob && bytes >= rs_peer_blob_bytes(p), RS_ERR_INVALID_ARG, "rs_peer_export: bad args");
    PFN_getAddressRange range = get_range_fn();
    RS_REQUIRE(range, RS_ERR_CUDA, "rs_peer_export: cuMemGetAddressRange unavailable");
    BlobHeader h;
    memset(&h, 0, sizeof(h));
    h.magic = kMagic;
    h.version = 1;
    h.rank = p->rank;
    h.pid = (int32_t)getpid();
    h.L_ssm = p->L_ssm; h.Hkv_ssm = p->Hkv_ssm; h.d_ssm = p->d_ssm;
    h.L_llm = p->L_llm; h.Hkv_llm = p->Hkv_llm; h.d_llm = p->d_llm;
    h.page_size = p->page_size;
    h.n_ptrs = n_ptrs(p);
    for (int e = 0; e < 2; ++e) RS_CUDA_CHECK(cudaIpcGetEventHandle(&h.ev[e], p->ev[e]));
    memcpy(blob, &h, sizeof(h));
    for (int i = 0; i < h.n_ptrs; ++i) {
        BlobEntry e;
        memset(&e, 0, sizeof(e));
        unsigned long long base = 0;
        size_t size = 0;
        const unsigned long long a = reinterpret_cast<unsigned long long>(p->ptrs[i]);
        RS_REQUIRE(range(&base, &size, a) == 0, RS_ERR_CUDA, "rs_peer_export: pool %d is not device memory", i);
        RS_CUDA_CHECK(cudaIpcGetMemHandle(&e.handle, reinterpret_cast<void*>(base)));
        e.offset = a - base;
        e.raw = a;
        memcpy(blob + sizeof(h) + i * sizeof(BlobEntry), &e, sizeof(e));
    }
    return RS_OK;
}

extern "C" rs_status rs_peer_import(rs_peer* p, const uint8_t* blob, size_t bytes) {
    RS_REQUIRE(p && blob && bytes >= sizeof(BlobHeader), RS_ERR_INVALID_ARG, "rs_peer_import: bad args");
    BlobHeader h;
    memcpy(&h, blob, sizeof(h));
    RS_REQUIRE(h.magic == kMagic && h.version == 1, RS_ERR_LAYOUT_MISMATCH, "rs_peer_import: not a peer blob");
    RS_REQUIRE(h.rank >= 0 && h.rank < kMaxPeers, RS_ERR_INVALID_ARG, "rs_peer_import: rank %d", h.rank);
    RS_REQUIRE(h.L_ssm == p->L_ssm && h.L_llm == p->L_llm && h.page_size == p->page_size &&
                   (h.L_ssm == 0 || (h.Hkv_ssm == p->Hkv_ssm && h.d_ssm == p->d_ssm)) &&
                   (h.L_llm == 0 || (h.Hkv_llm == p->Hkv_llm && h.d_llm == p->d_llm)) && h.n_ptrs == n_ptrs(p),
               RS_ERR_LAYOUT_MISMATCH, "rs_peer_import: rank %d's KV store has a different shape", h.rank);
    RS_REQUIRE(bytes >= sizeof(BlobHeader) + sizeof(BlobEntry) * h.n_ptrs, RS_ERR_INVALID_ARG,
               "rs_peer_import: blob truncated");
    Peer& q = p->peers[h.rank];
    RS_REQUIRE(!q.present, RS_ERR_INVALID_ARG, "rs_peer_import: rank %d already imported", h.rank);
    q.local = h.pid == (int32_t)getpid();
    q.ptrs.assign(h.n_ptrs, nullptr);
    for (int i = 0; i < h.n_ptrs; ++i) {
        BlobEntry e;
        memcpy(&e, blob + sizeof(h) + i * sizeof(BlobEntry), sizeof(e));
        if (q.local) {
            q.ptrs[i] = reinterpret_cast<void*>(e.raw);
            continue;
        }
        const std::string key(reinterpret_cast<const char*>(&e.handle), sizeof(e.handle));
        auto it = p->mapped.find(key);
        void* base = nullptr;
        if (it != p->mapped.end()) {
            base = it->second;
        } else {
            RS_CUDA_CHECK(cudaIpcOpenMemHandle(&base, e.handle, cudaIpcMemLazyEnablePeerAccess));
            p->mapped.emplace(key, base);
        }
        q.ptrs[i] = static_cast<uint8_t*>(base) + e.offset;
    }
    for (int k = 0; k < 2; ++k) {
        if (q.local) {
            q.ev[k] = nullptr;   // same process: the raw event is not exported; see rs_peer_wait
            continue;
        }
        RS_CUDA_CHECK(cudaIpcOpenEventHandle(&q.ev[k], h.ev[k]));
    }
    q.present = true;
    return RS_OK;
}

extern "C" rs_status rs_peer_push(rs_peer* p, int32_t dst_rank, const int32_t* src_block_table,
                                  const int32_t* dst_block_table, int32_t max_pages, const int32_t* starts,
                                  const int32_t* lens, int32_t n, int32_t parts, void* stream) {
    rs::bind_device(src_block_table);
    RS_REQUIRE(p && dst_rank >= 0 && dst_rank < kMaxPeers && n >= 0 && n <= 65535 && max_pages > 0 &&
                   parts >= 0 && parts <= 3,
               RS_ERR_INVALID_ARG, "rs_peer_push: bad args");
    if (n == 0 || parts == 0) return RS_OK;
    const Peer& q = p->peers[dst_rank];
    RS_REQUIRE(q.present, RS_ERR_INVALID_ARG, "rs_peer_push: rank %d not imported", dst_rank);
    RS_REQUIRE(src_block_table && dst_block_table && lens, RS_ERR_INVALID_ARG, "rs_peer_push: null pointer");
    cudaStream_t st = rs::as_stream(stream);
    // model order SSM then LLM (the SSM part first lets the destination draft)
    for (int m = 0; m < 2; ++m) {
        if (!(parts & (1 << m))) continue;
        const int L = m == 0 ? p->L_ssm : p->L_llm;
        if (L == 0) continue;
        const int Hkv = m == 0 ? p->Hkv_ssm : p->Hkv_llm, d = m == 0 ? p->d_ssm : p->d_llm;
        const int off = m == 0 ? 0 : 2 * p->L_ssm;
        LayerPtrs a, b;
        for (int l = 0; l < L; ++l) {
            a.k[l] = p->ptrs[off + l];
            a.v[l] = p->ptrs[off + L + l];
            b.k[l] = q.ptrs[off + l];
            b.v[l] = q.ptrs[off + L + l];
        }
        dim3 grid(n, L, 2 * Hkv);
        kv_push_kernel<<<grid, kThreads, 0, st>>>(a, b, Hkv, d, p->page_size, src_block_table, dst_block_table,
                                                  max_pages, starts, lens);
        RS_LAUNCH_CHECK();
    }
    return RS_OK;
}

extern "C" rs_status rs_peer_signal(rs_peer* p, int32_t which, void* stream) {
    RS_REQUIRE(p && (which == 0 || which == 1), RS_ERR_INVALID_ARG, "rs_peer_signal: bad args");
    RS_CUDA_CHECK(cudaEventRecord(p->ev[which], rs::as_stream(stream)));
    return RS_OK;
}

extern "C" rs_status rs_peer_wait(rs_peer* p, int32_t src_rank, int32_t which, void* stream) {
    RS_REQUIRE(p && src_rank >= 0 && src_rank < kMaxPeers && (which == 0 || which == 1), RS_ERR_INVALID_ARG,
               "rs_peer_wait: bad args");
    const Peer& q = p->peers[src_rank];
    RS_REQUIRE(q.present, RS_ERR_INVALID_ARG, "rs_peer_wait: rank %d not imported", src_rank);
    // same process (loopback): the source's own event object; it is this rs_peer's when
    // src_rank == p->rank, otherwise the caller runs both instances in one process and must
    // order the streams itself (no event is exported within a process)
    cudaEvent_t e = q.local ? (src_rank == p->rank ? p->ev[which] : nullptr) : q.ev[which];
    if (!e) return RS_OK;
    RS_CUDA_CHECK(cudaStreamWaitEvent(rs::as_stream(stream), e, 0));
    return RS_OK;
}

extern "C" void rs_peer_destroy(rs_peer* p) {
    if (!p) return;
    for (auto& q : p->peers)
        for (int k = 0; k < 2; ++k)
            if (q.ev[k]) cudaEventDestroy(q.ev[k]);
    for (auto& kv : p->mapped) cudaIpcCloseMemHandle(kv.second);
    for (int k = 0; k < 2; ++k)
        if (p->ev[k]) cudaEventDestroy(p->ev[k]);
    delete p;
}
