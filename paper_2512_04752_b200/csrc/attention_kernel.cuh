// a2 device code: tree-verification attention on sm_100a (tcgen05 / TMEM / TMA).
// P:76-80 (single-pass verification of the whole draft tree), P:213 (attention cost is
// "KVCache loading"); readings Z1-Z4. Host side (plan, launch): attention.cu.
//
// Work item = (sample b, kv head, M tile of 128 query rows, key-block range). Rows of a tile are
// the T_b*g (node, head-in-group) pairs, node-major, padded to 128 (UMMA M = 128); keys are the
// sample's logical slots in 64-key blocks = one KV page each.
//
// Persistent kernel, one CTA per SM, warp-specialised:
//   warp 0        TMA producer for Q tiles and K pages (ring of KS slots); in dynamic mode also
//                 takes items from the global queue
//   warp 3        TMA producer for V pages (ring of VS slots)
//   warp 1        S issuer: S_J = Q K_J^T (SS, M=128, N=64, K=D) into S[J&1]
//   warp 2        TMEM allocator + PV issuer: O[J&1] += P_J V_J (TS: P from TMEM, V MN-major)
//   warps 4..7    softmax warpgroup 0: blocks with even J      (rows of a tile: one per thread,
//   warps 8..11   softmax warpgroup 1: blocks with odd J        or two per thread when R = 16)
//   warps 12..15  (RM = 1 only) epilogue warpgroup: merge, normalise and store item i while the
//                 softmax warpgroups run item i+1 in the other 16-lane half of TMEM
// Each softmax warpgroup keeps its own running max/sum and its own O accumulator in TMEM, so
// the two run concurrently on alternate key blocks with no per-block synchronisation; the two
// partial states are merged in the epilogue. Online softmax in the exp2 domain with lazy
// rescaling (threshold 2^8) of O in TMEM.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include <type_traits>

#include "sm100_ptx.cuh"

namespace attn {

using namespace rs::ptx;

constexpr int kBlockN = 64;      // keys per KV block (= page_size)
constexpr int kM = 128;          // query rows per work item (UMMA M)
#ifndef RS_ATTN_KSLOTS
#define RS_ATTN_KSLOTS 4
#endif
#ifndef RS_ATTN_VSLOTS
#define RS_ATTN_VSLOTS 4
#endif
#ifndef RS_ATTN_EW_SLOTS
#define RS_ATTN_EW_SLOTS 4
#endif
#ifndef RS_ATTN_EW_KSLOTS
#define RS_ATTN_EW_KSLOTS RS_ATTN_EW_SLOTS
#endif
#ifndef RS_ATTN_EW_VSLOTS
#define RS_ATTN_EW_VSLOTS RS_ATTN_EW_SLOTS
#endif
constexpr int kMaxSlots = 8;
constexpr int kRing = 8;         // dynamic item queue ring depth (shared memory)
#ifndef RS_ATTN_STAGE
#define RS_ATTN_STAGE 0
#endif
constexpr int kKSlots = RS_ATTN_KSLOTS;
constexpr int kVSlots = RS_ATTN_VSLOTS;
constexpr bool kStageOut = RS_ATTN_STAGE != 0;   // epilogue output through smem + TMA store
#ifndef RS_ATTN_QBUFS
#define RS_ATTN_QBUFS 2
#endif
constexpr int kQBufs = RS_ATTN_QBUFS;   // Q tile buffers (RM 2/3; RM = 1 uses the two halves of one tile)
static_assert(kQBufs == 2, "the Q producer / S issuer handshake assumes two Q buffers (1 deadlocks)");
constexpr int kPF = 0;          // L2 prefetch distance in KV blocks (0 = off; measured: no gain)
#ifndef RS_ATTN_WARM
#define RS_ATTN_WARM 0
#endif
// Launch-time L2 warm-up: with early prefix streaming, each producer prefetches the prefix blocks
// [0, kWarm) of its CTA's first item into L2 before its ring wait, i.e. while the preceding
// layer's slowest CTAs still stream (PDL), so the first blocks of the launch come from L2.
constexpr int kWarm = RS_ATTN_WARM;
constexpr int kThreads = 384;    // 12 warps (RM 2/3)
// RM = 1 (every tile R = 16): 16 warps; warps 12-15 are an epilogue warpgroup, and consecutive
// items alternate between the two 16-lane halves of each TMEM sub-partition, so item i's O is
// normalised and stored while item i+1 already accumulates.
#ifndef RS_ATTN_DU_SPLIT
#define RS_ATTN_DU_SPLIT 0
#endif
// RM = 4 ("dual"): two warps per query row, each owning half of the 64 keys of a block (and half
// of the O columns in the epilogue): 8 softmax warps per tile, 20 warps in all
constexpr bool kDuSplit = RS_ATTN_DU_SPLIT != 0;
template <int RM> struct KT {
    static constexpr bool kEW = (RM == 1);
    static constexpr bool kCS = (RM == 4) && kDuSplit;
    static constexpr int kThreads = kEW ? 512 : (kCS ? 640 : 384);
    static constexpr int kSmWarps = kCS ? 8 : 4;   // softmax warps per warpgroup (tile)
};
// RM = 1: an item's 64 rows are half the TMEM lanes (16 per sub-partition), so its S and PV MMAs
// are issued with M = 64 at the item's lane half (tcgen05 M = 64 layout: A row m <-> lane
// (m % 16) + 32 (m / 16), + 16 for the odd half) instead of M = 128 over both items' halves: half
// the tensor-core work per key block (the M = 128 form computed the other item's rows too). Under
// the power cap that work sets the SM clock (c3s: no MMAs at all -> 1965 vs 1365 MHz).
#ifndef RS_ATTN_M64
#define RS_ATTN_M64 1
#endif
constexpr bool kM64 = RS_ATTN_M64 != 0;
constexpr int kTraceJ = 256;

// Row layout of a tile: logical query row r (node-major (node, head-in-group) pairs of the unit)
// lives in TMEM lane / UMMA row m = (r / R) * 32 + r % R, R = rstride in {16, 32}: each of the
// four TMEM sub-partitions (= softmax warps) holds R consecutive rows, so a short tile
// (T*g <= 64, R = 16) still spreads its work over all four SM sub-partitions.
struct alignas(16) WorkItem {
    int32_t b, kvh, mtile, blk_begin, blk_end, part;  // part: -1 = direct, else partial slot
    int32_t rstride;                                  // R (tile covers 4*R logical rows)
    int32_t unit;                                     // split-unit index, -1 if direct
    int32_t P, node0, T;                              // sample's prefix length, tree_off[b], tree size
    int32_t pad;                                      // (copied from the host lengths at plan time, so an
};                                                    //  item needs one 48-byte load and no dependent ones)
static_assert(sizeof(WorkItem) == 48, "WorkItem layout (rs_attn_plan_items)");

__device__ __forceinline__ WorkItem load_item(const WorkItem* items, int w) {
    const int4* src = reinterpret_cast<const int4*>(items + w);
    const int4 a = __ldg(src), b = __ldg(src + 1), c = __ldg(src + 2);
    WorkItem r;
    r.b = a.x; r.kvh = a.y; r.mtile = a.z; r.blk_begin = a.w;
    r.blk_end = b.x; r.part = b.y; r.rstride = b.z; r.unit = b.w;
    r.P = c.x; r.node0 = c.y; r.T = c.z; r.pad = c.w;
    return r;
}
struct SplitUnit {
    int32_t b, kvh, mtile, n_parts, part_base, rstride;
};

template <int D, int RM = 2>
struct Cfg {
    static constexpr bool kEW = (RM == 1);
    // RM = 1: the two logical Q buffers are the two 16-row halves of ONE 128-row tile (items
    // alternate lane halves), which frees 32 KB for deeper K/V rings.
    static constexpr int KS = kEW ? RS_ATTN_EW_KSLOTS : kKSlots;
    static constexpr int VS = kEW ? RS_ATTN_EW_VSLOTS : kVSlots;
    static_assert(KS <= kMaxSlots && VS <= kMaxSlots, "ring depth");
    static constexpr int kBoxes = D / 64;                    // 64-element (128 B) SW128 boxes
    static constexpr int kQBytes = kM * D * 2;
    static constexpr int kQStride = kEW ? 0 : kQBytes;       // smem offset between logical Q buffers
    static constexpr int kKVBytes = kBlockN * D * 2;         // one K or V page tile
    static constexpr int kOffQ = 0;
    static constexpr int kOffK = kOffQ + (kEW ? 1 : kQBufs) * kQBytes;
    static constexpr int kOffV = kOffK + KS * kKVBytes;
    static constexpr int kOffStage = kOffV + VS * kKVBytes;   // epilogue staging [2][128 rows][128 B]
    static constexpr int kOffBar = kOffStage + (kStageOut ? 2 * kM * 128 : 0);
    // column-split dual softmax: per (tile, slot, key half, row) a partial row max (two slots, by
    // the warpgroup's block parity), and per (tile, half, row) the partial row sum at the end
    static constexpr int kBarBytes = 1024;                    // the mbarrier block (struct Bars)
    static constexpr int kOffXch = kOffBar + kBarBytes;
    static constexpr int kXchBytes = KT<RM>::kCS ? (2 * 2 * 2 * kM + 2 * 2 * kM) * 4 : 0;
    static constexpr int kSmemBytes = kOffXch + kXchBytes + 1024;  // + exchange + alignment slack
    // TMEM columns: O0 [0,D) O1 [D,2D) | S0 S1 (64 fp32 each) | P0 P1 (32 bf16x2 each) | m,l x2
    static constexpr int kTmemCols = 512;
    static constexpr int kColS = 2 * D;
    static constexpr int kColP = 2 * D + 2 * kBlockN;
    static constexpr int kColML = 2 * D + 3 * kBlockN;
    static_assert(kColML + 8 <= kTmemCols, "TMEM budget");
};

struct Bars {
    uint64_t q_full[kQBufs], q_empty[kQBufs];
    uint64_t k_full[kMaxSlots], k_empty[kMaxSlots];
    uint64_t v_full[kMaxSlots], v_empty[kMaxSlots];
    uint64_t s_full[2], s_free[2];
    uint64_t p_full[2], pv_done[2];
    uint64_t o_free;
    uint64_t o_ready[2], ml_ready[2], o_free2[2];   // epilogue-warpgroup handshakes (RM = 1), by item parity
    uint64_t item_full[8], item_empty[8];             // dynamic item queue: ring of item indices
    int item_ring[8];
    uint32_t tmem_base;
    int merge_flag;
    int merge_flags[2];                               // RM = 4: one split-KV unit per warpgroup
};

struct Params {
    const int32_t* cta_off;
    const WorkItem* items;
    float* part_o;      // [n_parts][kM][D] fp32, normalised
    float* part_lse;    // [n_parts][kM] fp32 (log2 domain)
    const SplitUnit* units;
    int* unit_counter;  // [n_units], zero between launches (reset by the merging CTA)
    const int32_t* prefix_len;
    const int32_t* tree_off;
    const uint64_t* tree_mask;
    const int32_t* block_table;
    int max_pages;
    int Hq, Hkv, g;
    float scale_log2;   // sm_scale * log2(e)
    __nv_bfloat16* out;
    float* lse;
    unsigned long long* trace;   // optional per-block event timestamps (profiling)
    const int32_t* qorder;       // dynamic scheduling: queue position -> item index
    int* qctr;                   // dynamic scheduling: [0] next item, [1] CTAs done (zero between launches)
    int n_items;
    int dyn;                     // 1: CTAs take items from the global queue (atomicAdd), 0: static lists
    int early_prefix;            // 1: prefix K/V pages + block table may be read before griddepcontrol.wait
    int dbg;                     // ablation switches for profiling only (RS_ATTN_DBG; results wrong if != 0):
                                 // 1 skip epilogue O reads/stores, 2 skip softmax math, 4 skip PV MMA
};

// Profiling events (clock64 per CTA / block J): 0 K issued, 1 V issued, 2 S issued,
// 3 S ready (softmax), 4 P written, 5 PV issued, 6 epilogue start, 7 epilogue end, 8 K seen
// landed by the S issuer, 9 V seen landed by the PV issuer; globaltimer at J = kTraceJ-1, 14/15.
#define TRACE(J, ev)                                                                          \
    do {                                                                                      \
        if (p.trace && (J) < (uint32_t)kTraceJ)                                               \
            p.trace[((size_t)blockIdx.x * kTraceJ + (J)) * 16 + (ev)] = clock64();             \
    } while (0)

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 2^x on the FMA/ALU pipes (x <= 8): round-to-nearest split via the 1.5*2^23 magic constant,
// degree-3 Taylor polynomial on [-0.5, 0.5] (relative error < 7e-4, below bf16 rounding), exponent
// added to the float bits. Used for a quarter of the elements so the MUFU pipe (ex2.approx) is
// not the softmax bottleneck (every ex2 costs 8 issue cycles of MUFU per warp).
__device__ __forceinline__ float ex2_poly(float x) {
    x = fmaxf(x, -126.0f);
    const float t = x + 12582912.0f;
    const float f = x - (t - 12582912.0f);
    float p = fmaf(f, 0.0555041086648216f, 0.2402264923172690f);
    p = fmaf(p, f, 0.6931471805599453f);
    p = fmaf(p, f, 1.0f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
#ifndef RS_ATTN_EXP_EMU
#define RS_ATTN_EXP_EMU 0   // eighths of the exponentials on the FMA pipe (0: all on MUFU)
#endif
// Dual items (RM = 4, the tensor-bound config 5): two softmax warps per SM sub-partition each
// need 64 MUFU ex2 per row per key block, as many MUFU cycles as the block's MMAs take; putting
// RS_ATTN_EXP_EMU_DUAL of every 8 on the FMA pipe measured 312 -> 298 us per layer (c5g8).
#ifndef RS_ATTN_EXP_EMU_DUAL
#define RS_ATTN_EXP_EMU_DUAL 2
#endif
// element c of a row block: EMU of every 8 on the FMA pipe
template <int EMU = RS_ATTN_EXP_EMU>
__device__ __forceinline__ float ex2_mix(float x, int c) {
    if (EMU && (c & 7) >= 8 - EMU) return ex2_poly(x);
    return ex2(x);
}

// Packed fp32 pairs (sm_100 FFMA2 / FADD2): one instruction per two elements of a row.
#ifndef RS_ATTN_DU_EPI
#define RS_ATTN_DU_EPI 16   // dual-item epilogue: O columns read from TMEM per wait (16 | 32 | 64)
#endif
constexpr int kDuEpi = RS_ATTN_DU_EPI;

#ifndef RS_ATTN_F32X2
#define RS_ATTN_F32X2 0
#endif
__device__ __forceinline__ uint64_t f2_pack(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// RM: 1 = every tile has R = 16, 2 = every tile has R = 32, 3 = mixed (both paths compiled in),
// 4 = "dual": every item covers TWO query tiles (mtile, mtile + 1) of a (sample, kv head) and
// each softmax warpgroup owns one of them (O0/O1, S0/S1, P0/P1 indexed by the tile): every K/V
// tile brought into shared memory feeds both tiles' S and PV MMAs, halving the L2 -> SM bytes
// per FLOP (config 5). The issuers walk "virtual blocks" vb = 2 * key block + tile.
template <int D, int RM>
__global__ void __launch_bounds__(KT<RM>::kThreads, 1)
tree_attn_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                 const Params p) {
    using C = Cfg<D, RM>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Bars* bars = reinterpret_cast<Bars*>(smem + C::kOffBar);
    static_assert(sizeof(Bars) <= C::kBarBytes, "barrier block overlaps the exchange region");
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int item_begin = p.cta_off[blockIdx.x];
    const int item_end = p.cta_off[blockIdx.x + 1];
    // The CTA's item sequence: its static plan list, then (p.dyn) the dynamic tail: warp 0 takes
    // the next item of the global queue with atomicAdd; every position is published through a
    // shared-memory ring that every other warp reads once per position. -1 ends the sequence.
    auto seq_read = [&](int it) -> int {   // warp-collective, every warp except warp 0
        if (!p.dyn) return item_begin + it < item_end ? item_begin + it : -1;
        const int sl = it % kRing;
        mbar_wait(&bars->item_full[sl], (it / kRing) & 1);
        const int w = *reinterpret_cast<volatile int*>(&bars->item_ring[sl]);
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&bars->item_empty[sl]);
        return w;
    };
    auto seq_fetch = [&](int it) -> int {  // warp 0: produce position it of the sequence
        if (!p.dyn) return item_begin + it < item_end ? item_begin + it : -1;
        int w = item_begin + it;
        if (w >= item_end) {   // own list done: the next tail item of the global queue
            griddep_wait();    // (the counter is reset by the previous launch's last CTA)
            if ((threadIdx.x & 31) == 0) w = atomicAdd(p.qctr, 1);
            w = __shfl_sync(0xffffffffu, w, 0);
            w = (w < p.n_items) ? __ldg(p.qorder + w) : -1;
        }
        const int sl = it % kRing;
        mbar_wait(&bars->item_empty[sl], ((it / kRing) & 1) ^ 1);
        if ((threadIdx.x & 31) == 0) {
            bars->item_ring[sl] = w;
            mbar_arrive(&bars->item_full[sl]);   // release: the ring entry is visible to waiters
        }
        __syncwarp();
        return w;
    };
    if (p.trace && threadIdx.x == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        p.trace[((size_t)blockIdx.x * kTraceJ + kTraceJ - 1) * 16 + 13] = smid;
        p.trace[((size_t)blockIdx.x * kTraceJ + kTraceJ - 1) * 16 + 14] = globaltimer_ns();
    }

    if (threadIdx.x == 0) {
        for (int i = 0; i < kQBufs; ++i) { mbar_init(&bars->q_full[i], 1); mbar_init(&bars->q_empty[i], 1); }
        for (int i = 0; i < C::KS; ++i) { mbar_init(&bars->k_full[i], 1); mbar_init(&bars->k_empty[i], 1); }
        for (int i = 0; i < C::VS; ++i) { mbar_init(&bars->v_full[i], 1); mbar_init(&bars->v_empty[i], 1); }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->s_full[i], 1);
            mbar_init(&bars->s_free[i], KT<RM>::kSmWarps);
            mbar_init(&bars->p_full[i], KT<RM>::kSmWarps);
            mbar_init(&bars->pv_done[i], 1);
        }
        mbar_init(&bars->o_free, 2 * KT<RM>::kSmWarps);
        for (int i = 0; i < kRing; ++i) {
            mbar_init(&bars->item_full[i], 1);
            mbar_init(&bars->item_empty[i], KT<RM>::kThreads / 32 - 1);   // every warp but warp 0
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&bars->o_ready[i], 1);
            mbar_init(&bars->ml_ready[i], 8);
            mbar_init(&bars->o_free2[i], 4);
        }
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
    // Programmatic dependent launch: the next layer's grid may be scheduled now (its CTAs start
    // as this grid's CTAs exit). Before griddep_wait() returns, the preceding grid's writes are
    // not guaranteed visible. Only the item tables (uploaded by a copy, not a kernel) are read
    // before it unconditionally. With plan.early_prefix set (rs_attn_plan_set_early_prefix: the
    // caller guarantees no kernel that may still be running writes the prefix K/V or the block
    // table), the K and V producers also stream the PREFIX blocks (every slot < P_b) while the
    // previous grid drains; a block holding any tree slot (written upstream, e.g. by the QKV
    // projection right before this launch) is loaded only after the producer's own wait. Q, the
    // tree masks, outputs and the shared split-KV workspace are touched only after it.
    griddep_launch_dependents();
    if (warp >= 4 || ((warp == 0 || warp == 3) && !p.early_prefix)) griddep_wait();
    if (warp == 0 || warp == 3) {
        // ============================ TMA producers ============================
        // warp 0: Q tiles + K pages; warp 3: V pages (whole warp runs the loop; one elected lane
        // issues). Page ids come 32 at a time from one coalesced load, a chunk ahead of use; item
        // descriptors are read two items ahead. Each producer also prefetches its pages kPF blocks
        // ahead into L2 (cp.async.bulk.prefetch.tensor), so the smem ring only has to cover the
        // L2 -> SM latency while HBM keeps kPF blocks per SM in flight.
        const bool isK = warp == 0;
        const CUtensorMap* tm = isK ? &tmK : &tmV;
        const int kSlots = isK ? C::KS : C::VS;
        const int pf = ((p.dbg >> 8) & 63) ? ((p.dbg >> 8) & 63) : kPF;
        const bool do_pf = pf > 0;
        bool waited = !p.early_prefix;   // this warp has executed griddep_wait()
        uint32_t J = 0;
        auto issue_q = [&](const WorkItem& x, int slot_it) {
            if constexpr (RM == 4) {
                // both Q buffers: tile mtile -> buffer 0, mtile + 1 -> buffer 1 (used every item)
                mbar_wait(&bars->q_empty[0], (slot_it & 1) ^ 1);
                mbar_wait(&bars->q_empty[1], (slot_it & 1) ^ 1);
                const int R = x.rstride;
                if (elect_one()) {
                    for (int t = 0; t < 2; ++t) {
                        const int row0 = (x.mtile + t) * 4 * R;
                        uint8_t* qs = smem + C::kOffQ + t * C::kQStride;
                        mbar_arrive_expect_tx(&bars->q_full[t], 4 * R * 128 * C::kBoxes);
                        for (int q = 0; q < 4; ++q)
                            for (int s = 0; s < R; s += 16) {
                                const int node = x.node0 + (row0 + q * R + s) / p.g;
#pragma unroll
                                for (int bx = 0; bx < C::kBoxes; ++bx)
                                    tma_load_3d(qs + bx * (kM * 128) + (32 * q + s) * 128, &tmQ, &bars->q_full[t],
                                                bx * 64, x.kvh * p.g, node);
                            }
                    }
                }
                __syncwarp();
                return;
            }
            const int qb = slot_it % kQBufs;
            mbar_wait(&bars->q_empty[qb], ((slot_it / kQBufs) & 1) ^ 1);
            const int R = x.rstride;
            const int row0 = x.mtile * 4 * R;               // first logical row of the tile
            uint8_t* qs = smem + C::kOffQ + qb * C::kQStride;
            if (elect_one()) {
                mbar_arrive_expect_tx(&bars->q_full[qb], 4 * R * 128 * C::kBoxes);
                // boxes of 16 rows (16/g nodes x g heads x 64 d): logical rows q*R + 16*s of
                // quarter q go to UMMA rows 32*q + 16*s
                for (int q = 0; q < 4; ++q)
                    for (int s = 0; s < R; s += 16) {
                        const int node = x.node0 + (row0 + q * R + s) / p.g;
#pragma unroll
                        for (int bx = 0; bx < C::kBoxes; ++bx)
                            tma_load_3d(qs + bx * (kM * 128) +
                                            (KT<RM>::kEW ? (kM64 ? 64 * (slot_it & 1) + 16 * q + s : 32 * q + s + 16 * (slot_it & 1))
                                                          : 32 * q + s) * 128,
                                        &tmQ, &bars->q_full[qb], bx * 64, x.kvh * p.g, node);
                    }
            }
            __syncwarp();
        };
        auto page_chunk = [&](const WorkItem& x, int base) {
            const int j = base + lane;
            return (j < x.blk_end - x.blk_begin)
                       ? __ldg(p.block_table + (int64_t)x.b * p.max_pages + x.blk_begin + j) : 0;
        };
        auto seq = [&](int it) { return isK ? seq_fetch(it) : seq_read(it); };
        int w = seq(0);
        if (w >= 0) {
            int wnx = seq(1);
            WorkItem wi = load_item(p.items, w);
            WorkItem wn = wnx >= 0 ? load_item(p.items, wnx) : wi;
            const int q0_at = min(wi.blk_end - wi.blk_begin, C::KS) - 1;   // first Q after the first K ring fill
            int pg_cur = page_chunk(wi, 0);
            // launch-time warm-up (kWarm, early prefix only: prefix blocks, before the wait)
            if (kWarm > 0 && p.early_prefix) {
                const int nw = min(min(kWarm, 32), wi.blk_end - wi.blk_begin);
                for (int k = 0; k < nw; ++k) {
                    const int page = __shfl_sync(0xffffffffu, pg_cur, k);
                    if ((wi.blk_begin + k + 1) * kBlockN <= wi.P && elect_one())
#pragma unroll
                        for (int bx = 0; bx < C::kBoxes; ++bx) tma_prefetch_2d(tm, bx * 64, (page * p.Hkv + wi.kvh) * kBlockN);
                    __syncwarp();
                }
            }
            // warm L2 with the first blocks of this CTA
            for (int k = 0; k < pf && k < wi.blk_end - wi.blk_begin; ++k) {
                const int page = __shfl_sync(0xffffffffu, pg_cur, k & 31);
                if (k < 32 && elect_one())
#pragma unroll
                    for (int bx = 0; bx < C::kBoxes; ++bx) tma_prefetch_2d(tm, bx * 64, (page * p.Hkv + wi.kvh) * kBlockN);
                __syncwarp();
            }
            for (int it = 0; w >= 0; ++it) {
                const bool has_next = wnx >= 0;
                const int wnnx = has_next ? seq(it + 2) : -1;
                const WorkItem wnn = wnnx >= 0 ? load_item(p.items, wnnx) : wn;
                const int nb = wi.blk_end - wi.blk_begin;
                const int nbn = has_next ? wn.blk_end - wn.blk_begin : 0;
                const int pg_first_next = has_next ? page_chunk(wn, 0) : 0;
                const int q_next_at = nb > 6 ? nb - 6 : 0;
                int pg_nxt = nb > 32 ? page_chunk(wi, 32) : 0;
                for (int base = 0; base < nb; base += 32) {
                    const int cnt = min(32, nb - base);
                    for (int k = 0; k < cnt; ++k, ++J) {
                        const int j = base + k;
                        if (isK && it == 0 && j == q0_at) {
                            if (!waited) { griddep_wait(); waited = true; }
                            issue_q(wi, 0);
                        }
                        // a block with a tree slot (slot >= P_b) only after the wait
                        if (!waited && (wi.blk_begin + j + 1) * kBlockN > wi.P) { griddep_wait(); waited = true; }
                        // RM = 1 with static lists: Q(0) and Q(1) here, then the epilogue warpgroup
                        // issues Q(it + 2) once item it's epilogue is done (issuing Q here stalled
                        // the K stream ~2 000 cycles per item: eight small 3-D TMA boxes)
                        const bool ew_static = KT<RM>::kEW && !p.dyn;
                        if (RM != 4 && isK && has_next && (ew_static ? (it == 0 && j == q0_at) : j == q_next_at)) {
                            if (lane == 0) TRACE(J, 11);   // (profiling: next item's Q issued at block J)
                            issue_q(wn, it + 1);
                        }
                        if (RM == 4 && isK && it > 0 && j == 0) issue_q(wi, it);
                        // L2 prefetch of block j + pf (this item or the next one)
                        if (do_pf) {
                            const int f = j + pf;
                            int fpage = -1, fkvh = wi.kvh;
                            if (f < nb) {
                                const int fk = k + pf;
                                const int v0 = __shfl_sync(0xffffffffu, pg_cur, fk & 31);
                                const int v1 = __shfl_sync(0xffffffffu, pg_nxt, fk & 31);
                                fpage = fk < 32 ? v0 : v1;
                            } else if (f - nb < nbn && f - nb < 32) {
                                fpage = __shfl_sync(0xffffffffu, pg_first_next, (f - nb) & 31);
                                fkvh = wn.kvh;
                            }
                            if (fpage >= 0 && (f < nb ? (k + pf < 64) : true) && elect_one()) {
#pragma unroll
                                for (int bx = 0; bx < C::kBoxes; ++bx)
                                    tma_prefetch_2d(tm, bx * 64, (fpage * p.Hkv + fkvh) * kBlockN);
                            }
                            __syncwarp();
                        }
                        const int page = __shfl_sync(0xffffffffu, pg_cur, k);
                        const int s = J % kSlots;
                        uint64_t* empty = isK ? &bars->k_empty[s] : &bars->v_empty[s];
                        uint64_t* full = isK ? &bars->k_full[s] : &bars->v_full[s];
                        mbar_wait(empty, ((J / kSlots) & 1) ^ 1);
                        const int row = (page * p.Hkv + wi.kvh) * kBlockN;
                        uint8_t* dst = smem + (isK ? C::kOffK : C::kOffV) + s * C::kKVBytes;
                        if (elect_one()) {
                            TRACE(J, isK ? 0 : 1);
                            mbar_arrive_expect_tx(full, C::kKVBytes);
#pragma unroll
                            for (int bx = 0; bx < C::kBoxes; ++bx)
                                tma_load_2d(dst + bx * (kBlockN * 128), tm, full, bx * 64, row);
                        }
                        __syncwarp();
                    }
                    pg_cur = pg_nxt;
                    pg_nxt = (base + 64 < nb) ? page_chunk(wi, base + 64) : 0;
                }
                pg_cur = pg_first_next;
                wi = wn;
                wn = wnn;
                w = wnx;
                wnx = wnnx;
            }
        }
    } else if (warp == 1) {
        // ============================ MMA issuer: S = Q K^T ============================
        // Runs ahead as far as the S double buffer allows (S_J needs S_{J-2} consumed).
        constexpr bool S64 = KT<RM>::kEW && kM64;
        constexpr uint32_t idS = idesc_bf16_f32(S64 ? 64 : kM, kBlockN, 0);
        const uint32_t sbase = smem_u32(smem);
        uint32_t sJ = 0;
        int it = 0;
        int w = seq_read(0);
        int nblk = w >= 0 ? __ldg(&p.items[w].blk_end) - __ldg(&p.items[w].blk_begin) : 0;
        constexpr bool DU = RM == 4;
        for (; w >= 0; ++it) {
            const int wn = seq_read(it + 1);
            const int nblk_next = wn >= 0 ? __ldg(&p.items[wn].blk_end) - __ldg(&p.items[wn].blk_begin) : 0;
            const int qb = it % kQBufs;
            if (DU) {
                mbar_wait(&bars->q_full[0], it & 1);
                mbar_wait(&bars->q_full[1], it & 1);
            } else {
                mbar_wait(&bars->q_full[qb], (it / kQBufs) & 1);
            }
            if (lane == 0) TRACE(sJ, 10);   // (profiling: this item's Q seen landed)
            // dual: virtual block sJ = 2 * key block + tile; key block counter kJ = sJ >> 1
            const int nv = DU ? 2 * nblk : nblk;
            for (int j = 0; j < nv; ++j, ++sJ) {
                const uint32_t kJ = DU ? (sJ >> 1) : sJ;
                // (M = 64: the item's 64 Q rows are contiguous at half it & 1 of the tile)
                const uint32_t qa = sbase + C::kOffQ + (DU ? (sJ & 1) : qb) * C::kQStride + (S64 ? (it & 1) * 64 * 128 : 0);
                if (!DU || (sJ & 1) == 0) mbar_wait(&bars->k_full[kJ % C::KS], (kJ / C::KS) & 1);
                if (lane == 0) TRACE(sJ, 8);
                mbar_wait(&bars->s_free[sJ & 1], ((sJ >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t ka = sbase + C::kOffK + (kJ % C::KS) * C::kKVBytes;
                const uint32_t sd = tmem + C::kColS + (sJ & 1) * kBlockN + (S64 ? (uint32_t)(16 * (it & 1)) << 16 : 0u);
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < ((p.dbg & 16) ? 0 : D / 16); ++k) {
                        const int bx = k >> 2, within = (k & 3) * 32;
                        uint64_t ad = smem_desc_sw128(qa + bx * (kM * 128) + within, 16, 1024);
                        uint64_t bd = smem_desc_sw128(ka + bx * (kBlockN * 128) + within, 16, 1024);
                        umma_f16(sd, ad, bd, idS, k > 0 ? 1u : 0u);
                    }
                    TRACE(sJ, 2);
                    umma_commit(&bars->s_full[sJ & 1]);
                    if (!DU || (sJ & 1) == 1) umma_commit(&bars->k_empty[kJ % C::KS]);
                    if (j == nv - 1) {
                        if (DU) {
                            umma_commit(&bars->q_empty[0]);
                            umma_commit(&bars->q_empty[1]);
                        } else {
                            umma_commit(&bars->q_empty[qb]);
                        }
                    }
                }
                __syncwarp();
            }
            nblk = nblk_next;
            w = wn;
        }
    } else if (warp == 2) {
        // ============================ MMA issuer: O += P V ============================
        constexpr bool P64 = KT<RM>::kEW && kM64;
        constexpr uint32_t idPV = idesc_bf16_f32(P64 ? 64 : kM, D, 1);
        const uint32_t sbase = smem_u32(smem);
        uint32_t pJ = 0;
        int it = 0;
        int w = seq_read(0);
        int nblk = w >= 0 ? __ldg(&p.items[w].blk_end) - __ldg(&p.items[w].blk_begin) : 0;
        for (; w >= 0; ++it) {
            const int wn = seq_read(it + 1);
            const int nblk_next = wn >= 0 ? __ldg(&p.items[wn].blk_end) - __ldg(&p.items[wn].blk_begin) : 0;
            // keys [key_end, ...) of the sample's last page: their V rows are zeroed below
            const int key_end = __ldg(&p.items[w].P) + __ldg(&p.items[w].T);
            const int blk0 = __ldg(&p.items[w].blk_begin);
            constexpr bool DU = RM == 4;
            const int nv = DU ? 2 * nblk : nblk;   // dual: virtual block pJ = 2 * key block + tile
            for (int j = 0; j < nv; ++j, ++pJ) {
                // EW: O is pre-zeroed, so every PV accumulates; else the first block of each
                // warpgroup (dual: of each tile) in the item overwrites
                const bool first = !KT<RM>::kEW && j < 2;
                const uint32_t vJ = DU ? (pJ >> 1) : pJ;
                if (!DU || (pJ & 1) == 0) {
                    mbar_wait(&bars->v_full[vJ % C::VS], (vJ / C::VS) & 1);
                    // Keys past the end of the sample in its last page get P = 0, but their V
                    // rows hold whatever the page held (possibly NaN bytes, and 0 * NaN = NaN in
                    // the MMA): zero them here, where the V tile is awaited anyway, so the softmax
                    // never waits on a V load (a tail block's P used to wait for its V tile, which
                    // stalled the whole P -> PV -> V-slot chain at every item end).
                    const int nvalid = key_end - (blk0 + (DU ? (j >> 1) : j)) * kBlockN;
                    if (nvalid < kBlockN) {
                        uint8_t* vs = smem + C::kOffV + (vJ % C::VS) * C::kKVBytes;
                        const int nz = (kBlockN - nvalid) * C::kBoxes * 8;   // 16-byte chunks
                        for (int q = lane; q < nz; q += 32) {
                            const int row = nvalid + q / (C::kBoxes * 8), rem = q % (C::kBoxes * 8);
                            reinterpret_cast<uint4*>(vs + (rem >> 3) * (kBlockN * 128) + row * 128)[rem & 7] =
                                make_uint4(0, 0, 0, 0);
                        }
                        fence_proxy_async_smem();
                    }
                    __syncwarp();
                }
                mbar_wait(&bars->p_full[pJ & 1], (pJ >> 1) & 1);
                if (lane == 0) TRACE(pJ, 9);
                // (EW: the softmax warpgroup re-zeroes its O half before its first P of the item,
                // after the epilogue of item it-2 released it, so PV needs no wait here)
                if (!KT<RM>::kEW && j == 0) mbar_wait(&bars->o_free, (it & 1) ^ 1);
                tc_fence_after();
                const uint32_t lh = P64 ? (uint32_t)(16 * (it & 1)) << 16 : 0u;   // the item's lane half
                const uint32_t pa = tmem + C::kColP + (pJ & 1) * (kBlockN / 2) + lh;
                const uint32_t va = sbase + C::kOffV + (vJ % C::VS) * C::kKVBytes;
                const uint32_t od = tmem + (pJ & 1) * D + lh;
                if (elect_one()) {
                    TRACE(pJ, 5);
#pragma unroll
                    for (int kk = 0; kk < ((p.dbg & 16) ? 0 : (p.dbg & 4) ? 1 : kBlockN / 16); ++kk) {
                        uint64_t bd = smem_desc_sw128(va + kk * 2048, kBlockN * 128, 1024);
                        umma_f16_ts(od, pa + kk * 8, bd, idPV, (first && kk == 0) ? 0u : 1u);
                    }
                    umma_commit(&bars->pv_done[pJ & 1]);
                    if (!DU || (pJ & 1) == 1) umma_commit(&bars->v_empty[vJ % C::VS]);
                    if (KT<RM>::kEW && j == nblk - 1) umma_commit(&bars->o_ready[it & 1]);
                }
                __syncwarp();
            }
            nblk = nblk_next;
            w = wn;
        }
    } else if (KT<RM>::kEW && warp >= 12) {
        // ============================ epilogue warpgroup (RM = 1) ============================
        // Item it (TMEM lane half h = it & 1): wait for its last PV (o_ready) and both softmax
        // warpgroups' (m, l) (ml_ready), merge the two partial states, normalise, store bf16 (or
        // the split-KV partial), re-zero the O half for item it+2 and release it (o_free2).
        const int wq = warp & 3;
        const int hl = lane & 15;
        const int rr = wq * 32 + hl;
        const uint32_t qbase = (uint32_t)(wq * 32) << 16;
        uint32_t J = 0;
        int it = 0;
        int w = seq_read(0);
        WorkItem wi = w >= 0 ? load_item(p.items, w) : WorkItem{};
        for (; w >= 0; ++it) {
            const int wnx = seq_read(it + 1);
            const WorkItem wn = wnx >= 0 ? load_item(p.items, wnx) : wi;
            const int h = it & 1;
            const int off = wi.node0;
            const int rows = min(64, wi.T * p.g - wi.mtile * 64);
            const bool warp_active = wq * 16 < rows;
            const int rl = wq * 16 + hl;
            const bool row_valid = rl < rows;
            const int grow = wi.mtile * 64 + rl;
            const int node = grow / p.g;
            const int nblk = wi.blk_end - wi.blk_begin;
            const bool had0 = nblk >= 2 || (J & 1) == 0;
            const bool had1 = nblk >= 2 || (J & 1) == 1;
            const bool direct = wi.part < 0;
            mbar_wait(&bars->o_ready[h], (it >> 1) & 1);
            mbar_wait(&bars->ml_ready[h], (it >> 1) & 1);
            tc_fence_after();
            if (wq == 0 && lane == 0) TRACE(J + nblk - 1, 6);
            {   // only valid rows compute and store
                uint32_t m0u, l0u, m1u, l1u;
                tmem_ld2(tmem + qbase + C::kColML + 4 * h, m0u, l0u);
                tmem_ld2(tmem + qbase + C::kColML + 4 * h + 2, m1u, l1u);
                tmem_wait_ld();
                const float m0 = __uint_as_float(m0u), l0 = __uint_as_float(l0u);
                const float m1 = __uint_as_float(m1u), l1 = __uint_as_float(l1u);
                const float M = fmaxf(had0 ? m0 : -INFINITY, had1 ? m1 : -INFINITY);
                const float w0 = (had0 && l0 > 0.0f) ? ex2(m0 - M) : 0.0f;
                const float w1 = (had1 && l1 > 0.0f) ? ex2(m1 - M) : 0.0f;
                const float L = l0 * w0 + l1 * w1;
                const float invL = L > 0.0f ? 1.0f / L : 0.0f;
                const float f0 = w0 * invL, f1 = w1 * invL;
                const int hh = wi.kvh * p.g + (grow % p.g);
                __nv_bfloat16* orow = p.out + ((int64_t)(off + node) * p.Hq + hh) * D;
                // split parts keep their normalised partial O in bf16 (like the output): half the
                // partial traffic; one more bf16 rounding before the merge (< 2^-9 relative)
                __nv_bfloat16* dst_row = direct ? orow
                                                : reinterpret_cast<__nv_bfloat16*>(p.part_o) + ((int64_t)wi.part * kM + rr) * D;
                const uint32_t rowbase = tmem + ((uint32_t)(wq * 32 + 16 * h) << 16);
                const int cb = (lane & 16) ? D / 2 : 0;   // my columns [cb, cb + D/2)
#pragma unroll 1
                for (int cc = 0; cc < D / 2; cc += 16) {
                    uint32_t a[16], bb[16];
                    tmem_ld_hs16<D / 2>(rowbase + cc, a);
                    tmem_ld_hs16<D / 2>(rowbase + D + cc, bb);
                    tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < 16; ++c)
                        a[c] = __float_as_uint(__uint_as_float(a[c]) * f0 + __uint_as_float(bb[c]) * f1);
                    if (warp_active && row_valid && !(p.dbg & 32)) {   // (dbg 32: skip stores, measurement only)
#pragma unroll
                        for (int c = 0; c < 16; c += 8) {
                            uint4 u;
                            u.x = pack_bf16(__uint_as_float(a[c]), __uint_as_float(a[c + 1]));
                            u.y = pack_bf16(__uint_as_float(a[c + 2]), __uint_as_float(a[c + 3]));
                            u.z = pack_bf16(__uint_as_float(a[c + 4]), __uint_as_float(a[c + 5]));
                            u.w = pack_bf16(__uint_as_float(a[c + 6]), __uint_as_float(a[c + 7]));
                            *reinterpret_cast<uint4*>(dst_row + cb + cc + c) = u;
                        }
                    }
                }
                if (warp_active && row_valid && lane < 16) {
                    const float lse2 = L > 0.0f ? M + __log2f(L) : -INFINITY;
                    if (direct) {
                        if (p.lse) p.lse[(int64_t)(off + node) * p.Hq + hh] = lse2 * 0.6931471805599453f;
                    } else {
                        p.part_lse[(int64_t)wi.part * kM + rr] = lse2;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->o_free2[h]);
            if (wq == 0 && lane == 0) TRACE(J + nblk - 1, 7);
            if (wq == 0 && !p.dyn && item_begin + it + 2 < item_end) {
                // Q of item it + 2 into lane half h (item it's S MMAs are long done: q_empty[h])
                const WorkItem x = load_item(p.items, item_begin + it + 2);
                const int qs_it = it + 2;
                mbar_wait(&bars->q_empty[qs_it & 1], ((qs_it >> 1) & 1) ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&bars->q_full[qs_it & 1], 4 * x.rstride * 128 * C::kBoxes);
                    const int row0 = x.mtile * 4 * x.rstride;
                    for (int q = 0; q < 4; ++q)
                        for (int s2 = 0; s2 < x.rstride; s2 += 16) {
                            const int node = x.node0 + (row0 + q * x.rstride + s2) / p.g;
#pragma unroll
                            for (int bx = 0; bx < C::kBoxes; ++bx)
                                tma_load_3d(smem + C::kOffQ + bx * (kM * 128) +
                                                (kM64 ? 64 * (qs_it & 1) + 16 * q + s2 : 32 * q + s2 + 16 * (qs_it & 1)) * 128,
                                            &tmQ, &bars->q_full[qs_it & 1], bx * 64, x.kvh * p.g, node);
                        }
                }
                __syncwarp();
            }
            if (wi.part >= 0) {
                // split-KV unit: the CTA that completes its last part merges all parts
                __threadfence();
                named_bar_sync(3, 128);
                if (threadIdx.x == 12 * 32) {
                    const int old = atomicAdd(&p.unit_counter[wi.unit], 1);
                    const int last = (old == p.units[wi.unit].n_parts - 1) ? 1 : 0;
                    if (last) p.unit_counter[wi.unit] = 0;          // ready for the next launch
                    bars->merge_flag = last;
                }
                named_bar_sync(3, 128);
                if (bars->merge_flag && row_valid && warp_active) {
                    __threadfence();
                    const SplitUnit u = p.units[wi.unit];
                    float M = -INFINITY;
                    for (int q = 0; q < u.n_parts; ++q)
                        M = fmaxf(M, __ldcg(p.part_lse + (int64_t)(u.part_base + q) * kM + rr));
                    float wsum = 0.0f;
                    for (int q = 0; q < u.n_parts; ++q) {
                        const float lq = __ldcg(p.part_lse + (int64_t)(u.part_base + q) * kM + rr);
                        wsum += (lq == -INFINITY) ? 0.0f : ex2(lq - M);
                    }
                    const float inv = wsum > 0.0f ? 1.0f / wsum : 0.0f;
                    const int hh = wi.kvh * p.g + (grow % p.g);
                    __nv_bfloat16* orow = p.out + ((int64_t)(off + node) * p.Hq + hh) * D;
                    const int mcb = (lane & 16) ? D / 2 : 0;
#pragma unroll 1
                    for (int c0 = mcb; c0 < mcb + D / 2; c0 += 8) {
                        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                        for (int q = 0; q < u.n_parts; ++q) {
                            const float lq = __ldcg(p.part_lse + (int64_t)(u.part_base + q) * kM + rr);
                            const float wq2 = (lq == -INFINITY) ? 0.0f : ex2(lq - M) * inv;
                            const uint4 x = __ldcg(reinterpret_cast<const uint4*>(
                                reinterpret_cast<const __nv_bfloat16*>(p.part_o) + ((int64_t)(u.part_base + q) * kM + rr) * D + c0));
                            const uint32_t xw[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                acc[2 * e] += wq2 * __uint_as_float(xw[e] << 16);
                                acc[2 * e + 1] += wq2 * __uint_as_float(xw[e] & 0xFFFF0000u);
                            }
                        }
                        uint4 o;
                        o.x = pack_bf16(acc[0], acc[1]);
                        o.y = pack_bf16(acc[2], acc[3]);
                        o.z = pack_bf16(acc[4], acc[5]);
                        o.w = pack_bf16(acc[6], acc[7]);
                        *reinterpret_cast<uint4*>(orow + c0) = o;
                    }
                    if (p.lse && lane < 16)
                        p.lse[(int64_t)(off + node) * p.Hq + hh] = (M + __log2f(wsum)) * 0.6931471805599453f;
                }
            }
            J += nblk;
            wi = wn;
            w = wnx;
        }
    } else if (KT<RM>::kEW && warp >= 4) {
        // ============================ softmax (RM = 1, half-split rows) ============================
        const int grp = (warp - 4) >> 2;         // warpgroup: handles blocks with (J & 1) == grp
        const int wq = warp & 3;                 // TMEM sub-partition of this warp
        const int r = wq * 32 + lane;            // smem row for the V-tail zeroing
        const int hl = lane & 15;
        const uint32_t qbase = (uint32_t)(wq * 32) << 16;
        {
            // O (both lane halves) and P (both halves) of my warpgroup start at zero
            uint32_t z32[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) z32[c] = 0u;
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                const uint32_t lb = tmem + ((uint32_t)(wq * 32 + 16 * h2) << 16);
#pragma unroll
                for (int c0 = 0; c0 < D / 2; c0 += 32) tmem_st_hs32<D / 2>(lb + grp * D + c0, z32);
                tmem_st_hs16<16>(lb + C::kColP + grp * (kBlockN / 2), reinterpret_cast<const uint32_t(&)[16]>(z32[0]));
            }
            tmem_wait_st();
        }
        uint32_t J = 0;
        int it = 0;
        int w = seq_read(0);
        WorkItem wi = w >= 0 ? load_item(p.items, w) : WorkItem{};
        for (; w >= 0; ++it) {
            const int wnx = seq_read(it + 1);
            const WorkItem wn = wnx >= 0 ? load_item(p.items, wnx) : wi;   // prefetch
            const int h = it & 1;
            const uint32_t lane_base = (uint32_t)(wq * 32 + 16 * h) << 16;
            const uint32_t o_mine = tmem + lane_base + grp * D;
            const int P = wi.P;
            const int off = wi.node0;
            const int T = wi.T;
            const int rl = wq * 16 + hl;
            const int rows = min(64, T * p.g - wi.mtile * 64);
            const bool warp_active = wq * 16 < rows;
            const bool row_valid = rl < rows;
            const int grow = wi.mtile * 64 + rl;
            const int node = grow / p.g;
            const uint64_t mask = row_valid ? __ldg(p.tree_mask + off + node) : 0ull;
            const int key_end = P + T;
            const int nblk = wi.blk_end - wi.blk_begin;
            float m_run = -INFINITY, l_run = 0.0f;
            bool had = false;
            bool first_blk = true;
            for (int j = (int)((J & 1) != (uint32_t)grp); j < nblk; j += 2) {
                const uint32_t Jj = J + j;
                const int kbase = (wi.blk_begin + j) * kBlockN;
                mbar_wait(&bars->s_full[grp], (Jj >> 1) & 1);
                tc_fence_after();
                if (wq == 0 && lane == 0) TRACE(Jj, 3);
                bool pv_waited = Jj < 2;
                auto wait_prev_pv = [&]() {
                    if (!pv_waited) {
                        mbar_wait(&bars->pv_done[grp], ((Jj - 2) >> 1) & 1);
                        tc_fence_after();
                        pv_waited = true;
                    }
                };
                uint32_t sh[32];
                if (warp_active) {
                    tmem_ld_hs32<32>(tmem + lane_base + C::kColS + grp * kBlockN, sh);
                    tmem_wait_ld();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->s_free[grp]);
                if (warp_active && !(p.dbg & 16)) {   // (dbg 16: skip softmax math, measurement only)
                    const int kh = (lane & 16) ? 32 : 0;   // first key of my half
                    float mx8[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) mx8[k] = -INFINITY;
                    if (kbase + kBlockN <= P) {
#pragma unroll
                        for (int c = 0; c < 32; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(sh[c]));
                    } else {
                        const int dlt = P - kbase;
                        uint64_t vb = dlt >= 64 ? ~0ull : (dlt <= 0 ? 0ull : ((1ull << dlt) - 1ull));
                        if (dlt >= 0 && dlt < 64) vb |= mask << dlt;
                        else if (dlt < 0 && dlt > -64) vb |= mask >> (-dlt);
                        const uint32_t vh = (uint32_t)(vb >> kh);
#pragma unroll
                        for (int c = 0; c < 32; ++c) {
                            sh[c] = ((vh >> c) & 1u) ? sh[c] : 0xFF800000u;   // -inf
                            mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(sh[c]));
                        }
                    }
                    float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                     fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
                    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
                    const float m_blk = mx * p.scale_log2;
                    bool need_o = false;
                    float alpha = 1.0f;
                    if (m_blk > m_run + 8.0f) {
                        alpha = ex2(m_run - m_blk);
                        need_o = had && row_valid && (m_run != -INFINITY);
                        l_run *= alpha;
                        m_run = m_blk;
                    }
                    if (__any_sync(0xffffffffu, need_o)) {
                        wait_prev_pv();
                        const float f = need_o ? alpha : 1.0f;
#pragma unroll 1
                        for (int c0 = 0; c0 < D / 2; c0 += 32) {
                            uint32_t o[32];
                            tmem_ld_hs32<D / 2>(o_mine + c0, o);
                            tmem_wait_ld();
#pragma unroll
                            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
                            tmem_st_hs32<D / 2>(o_mine + c0, o);
                        }
                    }
                    const float mo = (m_run == -INFINITY) ? 0.0f : m_run;
                    float ls8[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) ls8[k] = 0.0f;
#pragma unroll
                    for (int c = 0; c < 32; c += 2) {
                        const float e0 = ex2_mix(fmaf(__uint_as_float(sh[c]), p.scale_log2, -mo), c);
                        const float e1 = ex2_mix(fmaf(__uint_as_float(sh[c + 1]), p.scale_log2, -mo), c + 1);
                        const uint32_t pk = pack_bf16(e0, e1);
                        sh[c >> 1] = pk;
                        ls8[(c >> 1) & 7] += e0 + e1;
                    }
                    l_run += ((ls8[0] + ls8[1]) + (ls8[2] + ls8[3])) + ((ls8[4] + ls8[5]) + (ls8[6] + ls8[7]));
                }
                wait_prev_pv();
                if (first_blk && it >= 2) {
                    // O half h last held item it-2: once its epilogue has read it, zero it. Only
                    // this warpgroup's MMAs touch these columns and its previous one is complete,
                    // so no MMA read-modify-write can race with the store.
                    mbar_wait(&bars->o_free2[h], ((it >> 1) & 1) ^ 1);
                    uint32_t z32[32];
#pragma unroll
                    for (int c = 0; c < 32; ++c) z32[c] = 0u;
#pragma unroll
                    for (int c0 = 0; c0 < D / 2; c0 += 32) tmem_st_hs32<D / 2>(o_mine + c0, z32);
                }
                if (warp_active)
                    tmem_st_hs16<16>(tmem + lane_base + C::kColP + grp * (kBlockN / 2),
                                     reinterpret_cast<const uint32_t(&)[16]>(sh[0]));
                if (first_blk) {
                    // the other lane half of my P buffer belongs to the previous item: zero it so
                    // this item's PV MMAs add nothing to that item's O
                    uint32_t z[16];
#pragma unroll
                    for (int c = 0; c < 16; ++c) z[c] = 0u;
                    tmem_st_hs16<16>(tmem + (lane_base ^ (16u << 16)) + C::kColP + grp * (kBlockN / 2), z);
                    if (!warp_active) {   // inactive warps: this item's half must hold zero P as well
                        tmem_st_hs16<16>(tmem + lane_base + C::kColP + grp * (kBlockN / 2), z);
                    }
                    first_blk = false;
                }
                tmem_wait_st();
                // (V rows past the sample's end are zeroed by the PV issuer)
                tc_fence_before();
                __syncwarp();
                if (wq == 0 && lane == 0) TRACE(Jj, 4);
                if (lane == 0) mbar_arrive(&bars->p_full[grp]);
                had = true;
            }
            // hand (m, l) of this warpgroup to the epilogue warps and move on
            l_run += __shfl_xor_sync(0xffffffffu, l_run, 16);
            if (it >= 2) mbar_wait(&bars->o_free2[h], ((it >> 1) & 1) ^ 1);   // ML[h] of item it-2 consumed
            tmem_st2(tmem + qbase + C::kColML + 4 * h + 2 * grp, __float_as_uint(m_run), __float_as_uint(l_run));
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->ml_ready[h]);
            J += nblk;
            wi = wn;
            w = wnx;
        }
    } else if (warp >= 4) {
        // ============================ softmax + epilogue ============================
        constexpr bool CS = KT<RM>::kCS;
        const int grp = CS ? (warp - 4) >> 3 : (warp - 4) >> 2;   // warpgroup: handles blocks with (J & 1) == grp
        const int hh = CS ? ((warp - 4) >> 2) & 1 : 0;             // CS: key / O-column half of this warp
        const int wq = warp & 3;                 // TMEM sub-partition of this warp
        const int r = wq * 32 + lane;            // UMMA row / TMEM lane of this thread
        const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
        const uint32_t o_mine = tmem + lane_base + grp * D;
        uint32_t J = 0;
        uint32_t bcnt = 0;   // CS: blocks this warpgroup has done (the max-exchange slot parity)
        int it = 0;
        int w = seq_read(0);
        WorkItem wi = w >= 0 ? load_item(p.items, w) : WorkItem{};
        for (; w >= 0; ++it) {
            const int wnx = seq_read(it + 1);
            const WorkItem wn = wnx >= 0 ? load_item(p.items, wnx) : wi;   // prefetch
            const int P = wi.P;
            const int off = wi.node0;
            const int T = wi.T;
            const int R = wi.rstride;
            // R = 16: the tile occupies TMEM lanes 0-15 of each sub-partition; two threads share a
            // row (16x32bx2 TMEM shapes), lanes 0-15 taking keys / columns of the low half and
            // lanes 16-31 those of the high half, so no lane idles.
            const bool hs = RM == 1 ? true : ((RM == 2 || RM == 4) ? false : (R == 16));
            constexpr bool DU = RM == 4;
            constexpr int kEmu = DU ? RS_ATTN_EXP_EMU_DUAL : RS_ATTN_EXP_EMU;
            const int mt = wi.mtile + (DU ? grp : 0);    // dual: this warpgroup's own tile
            const int hl = hs ? (lane & 15) : lane;      // row lane of this thread
            const int rr = wq * 32 + hl;                 // TMEM lane / UMMA row of my row
            const int rl = wq * R + hl;                  // logical row within the tile
            const int rows = min(4 * R, T * p.g - mt * 4 * R);
            const bool warp_active = wq * R < rows;
            const bool row_valid = hl < R && rl < rows;
            const int grow = mt * 4 * R + rl;            // row within the unit
            const int node = grow / p.g;
            const uint64_t mask = row_valid ? p.tree_mask[off + node] : 0ull;
            const int key_end = P + T;                   // keys >= key_end do not exist
            const int nblk = wi.blk_end - wi.blk_begin;
            const int nv = DU ? 2 * nblk : nblk;         // virtual blocks (dual: 2 * key block + tile)
            float m_run = -INFINITY, l_run = 0.0f;
            bool had = false;
            uint32_t Jlast = 0;
            // the block loop is instantiated per row mode so each path keeps only its own registers
            auto block_loop = [&](auto hs_tag) {
            constexpr bool HS = decltype(hs_tag)::value;
            for (int j = (int)((J & 1) != (uint32_t)grp); j < nv; j += 2) {
                const uint32_t Jj = J + j;
                const int kbase = (wi.blk_begin + (DU ? (j >> 1) : j)) * kBlockN;
                mbar_wait(&bars->s_full[grp], (Jj >> 1) & 1);
                tc_fence_after();
                if (wq == 0 && lane == 0 && hh == 0) TRACE(Jj, 3);
                // P buffer / O of this warpgroup were last used by its previous block (Jj - 2);
                // waited for only right before they are touched (rescale / P store)
                bool pv_waited = Jj < 2;
                auto wait_prev_pv = [&]() {
                    if (!pv_waited) {
                        mbar_wait(&bars->pv_done[grp], ((Jj - 2) >> 1) & 1);
                        tc_fence_after();
                        pv_waited = true;
                    }
                };
                if constexpr (HS) {
                    // ---- half-split row: 32 keys per thread ----
                    uint32_t sh[32];
                    if (warp_active) {
                        tmem_ld_hs32<32>(tmem + lane_base + C::kColS + grp * kBlockN, sh);
                        tmem_wait_ld();
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&bars->s_free[grp]);
                    if (p.dbg & 16) {
                        wait_prev_pv();
                    } else if (warp_active) {
                        const int kh = (lane & 16) ? 32 : 0;   // first key of my half
                        float mx8[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) mx8[k] = -INFINITY;
                        if (kbase + kBlockN <= P) {
#pragma unroll
                            for (int c = 0; c < 32; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(sh[c]));
                        } else {
                            const int dlt = P - kbase;
                            uint64_t vb = dlt >= 64 ? ~0ull : (dlt <= 0 ? 0ull : ((1ull << dlt) - 1ull));
                            if (dlt >= 0 && dlt < 64) vb |= mask << dlt;
                            else if (dlt < 0 && dlt > -64) vb |= mask >> (-dlt);
                            const uint32_t vh = (uint32_t)(vb >> kh);
#pragma unroll
                            for (int c = 0; c < 32; ++c) {
                                sh[c] = ((vh >> c) & 1u) ? sh[c] : 0xFF800000u;   // -inf
                                mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(sh[c]));
                            }
                        }
                        float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                         fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
                        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
                        const float m_blk = mx * p.scale_log2;
                        bool need_o = false;
                        float alpha = 1.0f;
                        if (m_blk > m_run + 8.0f) {
                            alpha = ex2(m_run - m_blk);
                            need_o = had && row_valid && (m_run != -INFINITY);
                            l_run *= alpha;
                            m_run = m_blk;
                        }
                        if (__any_sync(0xffffffffu, need_o)) {
                            wait_prev_pv();
                            const float f = need_o ? alpha : 1.0f;
#pragma unroll 1
                            for (int c0 = 0; c0 < D / 2; c0 += 32) {
                                uint32_t o[32];
                                tmem_ld_hs32<D / 2>(o_mine + c0, o);
                                tmem_wait_ld();
#pragma unroll
                                for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
                                tmem_st_hs32<D / 2>(o_mine + c0, o);
                            }
                        }
                        const float mo = (m_run == -INFINITY) ? 0.0f : m_run;
                        float ls8[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) ls8[k] = 0.0f;
#pragma unroll
                        for (int c = 0; c < 32; c += 2) {
                            const float e0 = ex2_mix(fmaf(__uint_as_float(sh[c]), p.scale_log2, -mo), c);
                            const float e1 = ex2_mix(fmaf(__uint_as_float(sh[c + 1]), p.scale_log2, -mo), c + 1);
                            const uint32_t pk = pack_bf16(e0, e1);
                            sh[c >> 1] = pk;
                            ls8[(c >> 1) & 7] += e0 + e1;
                        }
                        l_run += ((ls8[0] + ls8[1]) + (ls8[2] + ls8[3])) + ((ls8[4] + ls8[5]) + (ls8[6] + ls8[7]));
                        wait_prev_pv();
                        tmem_st_hs16<16>(tmem + lane_base + C::kColP + grp * (kBlockN / 2),
                                         reinterpret_cast<const uint32_t(&)[16]>(sh[0]));
                        tmem_wait_st();
                    } else {
                        wait_prev_pv();
                    }
                } else {
                if constexpr (CS) {
                // ---- column split (dual items): this warp owns keys [32 hh, 32 hh + 32) of the
                // block and O columns [D/2 hh, D/2 hh + D/2); the row max is combined with the
                // partner warp (same rows, other half) through shared memory and a 64-thread barrier
                uint32_t sr[32];
                if (warp_active) {
                    tmem_ld32(tmem + lane_base + C::kColS + grp * kBlockN + 32 * hh, sr);
                    tmem_wait_ld();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->s_free[grp]);
                float* xm = reinterpret_cast<float*>(smem + C::kOffXch) + (grp * 2 + (int)(bcnt & 1)) * 2 * kM;
                float mxh = -INFINITY;
                if (warp_active) {
                    float mx8[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) mx8[k] = -INFINITY;
                    if (kbase + kBlockN <= P) {
#pragma unroll
                        for (int c = 0; c < 32; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(sr[c]));
                    } else {
                        const int dlt = P - kbase;
                        uint64_t vb = dlt >= 64 ? ~0ull : (dlt <= 0 ? 0ull : ((1ull << dlt) - 1ull));
                        if (dlt >= 0 && dlt < 64) vb |= mask << dlt;
                        else if (dlt < 0 && dlt > -64) vb |= mask >> (-dlt);
                        const uint32_t vh = (uint32_t)(vb >> (32 * hh));
#pragma unroll
                        for (int c = 0; c < 32; ++c) {
                            sr[c] = ((vh >> c) & 1u) ? sr[c] : 0xFF800000u;   // -inf
                            mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(sr[c]));
                        }
                    }
                    mxh = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
                    xm[hh * kM + r] = mxh;
                }
                named_bar_sync(8 + grp * 4 + wq, 64);
                if (warp_active) {
                    const float m_blk = fmaxf(mxh, xm[(hh ^ 1) * kM + r]) * p.scale_log2;
                    bool need_o = false;
                    float alpha = 1.0f;
                    if (m_blk > m_run + 8.0f) {          // lazy rescale (both halves decide alike)
                        alpha = ex2(m_run - m_blk);
                        need_o = had && row_valid && (m_run != -INFINITY);
                        l_run *= alpha;
                        m_run = m_blk;
                    }
                    if (__any_sync(0xffffffffu, need_o)) {
                        wait_prev_pv();
                        const float f = need_o ? alpha : 1.0f;
#pragma unroll 1
                        for (int c0 = 0; c0 < D / 2; c0 += 32) {
                            uint32_t o[32];
                            tmem_ld32(o_mine + (D / 2) * hh + c0, o);
                            tmem_wait_ld();
#pragma unroll
                            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
                            tmem_st32(o_mine + (D / 2) * hh + c0, o);
                        }
                    }
                    const float mo = (m_run == -INFINITY) ? 0.0f : m_run;
                    float ls8[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) ls8[k] = 0.0f;
                    uint32_t pk16[16];
#pragma unroll
                    for (int c = 0; c < 32; c += 2) {
                        const float e0 = ex2_mix<kEmu>(fmaf(__uint_as_float(sr[c]), p.scale_log2, -mo), c);
                        const float e1 = ex2_mix<kEmu>(fmaf(__uint_as_float(sr[c + 1]), p.scale_log2, -mo), c + 1);
                        pk16[c >> 1] = pack_bf16(e0, e1);
                        ls8[(c >> 1) & 7] += e0 + e1;
                    }
                    l_run += ((ls8[0] + ls8[1]) + (ls8[2] + ls8[3])) + ((ls8[4] + ls8[5]) + (ls8[6] + ls8[7]));
                    wait_prev_pv();
                    tmem_st16(tmem + lane_base + C::kColP + grp * (kBlockN / 2) + 16 * hh, pk16);
                    tmem_wait_st();
                } else {
                    wait_prev_pv();
                }
                ++bcnt;
                } else {
                // sr: raw S bits -> masked S -> packed bf16 P in sr[0..31]
                uint32_t sr[64];
                if (warp_active) {
                    const uint32_t sa = tmem + lane_base + C::kColS + grp * kBlockN;
                    tmem_ld32(sa, reinterpret_cast<uint32_t(&)[32]>(sr[0]));
                    tmem_ld32(sa + 32, reinterpret_cast<uint32_t(&)[32]>(sr[32]));
                    tmem_wait_ld();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->s_free[grp]);
                if (warp_active && (p.dbg & 2)) {
                    wait_prev_pv();
                    tmem_st32(tmem + lane_base + C::kColP + grp * (kBlockN / 2),
                              reinterpret_cast<const uint32_t(&)[32]>(sr[0]));
                    tmem_wait_st();
                } else if (warp_active) {
                    // row max over the block: 8 independent partial maxima (short dependency chains)
                    float mx8[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) mx8[k] = -INFINITY;
                    if (kbase + kBlockN <= P) {
#pragma unroll
                        for (int c = 0; c < 64; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(sr[c]));
                    } else {
                        // visible-column bitmap of this block: prefix columns c < P - kbase,
                        // tree column c <-> node c - (P - kbase) (its ancestor bit)
                        const int dlt = P - kbase;
                        uint64_t vb = dlt >= 64 ? ~0ull : (dlt <= 0 ? 0ull : ((1ull << dlt) - 1ull));
                        if (dlt >= 0 && dlt < 64) vb |= mask << dlt;
                        else if (dlt < 0 && dlt > -64) vb |= mask >> (-dlt);
                        const uint32_t vlo = (uint32_t)vb, vhi = (uint32_t)(vb >> 32);
#pragma unroll
                        for (int c = 0; c < 64; ++c) {
                            const bool ok = ((c < 32 ? vlo >> c : vhi >> (c - 32)) & 1u) != 0u;
                            sr[c] = ok ? sr[c] : 0xFF800000u;   // -inf
                            mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(sr[c]));
                        }
                    }
                    const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                           fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
                    const float m_blk = mx * p.scale_log2;
                    bool need_o = false;
                    float alpha = 1.0f;
                    if (m_blk > m_run + 8.0f) {          // lazy rescale (values stay <= 2^8)
                        alpha = ex2(m_run - m_blk);      // m_run = -inf -> 0
                        need_o = had && row_valid && (m_run != -INFINITY);
                        l_run *= alpha;
                        m_run = m_blk;
                    }
                    if (__any_sync(0xffffffffu, need_o)) {
                        wait_prev_pv();
                        const float f = need_o ? alpha : 1.0f;
#pragma unroll 1
                        for (int c0 = 0; c0 < D; c0 += 32) {
                            uint32_t o[32];
                            tmem_ld32(o_mine + c0, o);
                            tmem_wait_ld();
#pragma unroll
                            for (int c = 0; c < 32; ++c) o[c] = __float_as_uint(__uint_as_float(o[c]) * f);
                            tmem_st32(o_mine + c0, o);
                        }
                    }
                    const float mo = (m_run == -INFINITY) ? 0.0f : m_run;
#if RS_ATTN_F32X2
                    {
                        const uint64_t sc2 = f2_pack(p.scale_log2, p.scale_log2), nm2 = f2_pack(-mo, -mo);
                        uint64_t ls2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
                        for (int c = 0; c < 64; c += 2) {
                            float x0, x1;
                            f2_unpack(f2_fma(f2_pack(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), sc2, nm2), x0, x1);
                            const float e0 = ex2_mix<kEmu>(x0, c), e1 = ex2_mix<kEmu>(x1, c + 1);
                            sr[c >> 1] = pack_bf16(e0, e1);
                            ls2[(c >> 1) & 3] = f2_add(ls2[(c >> 1) & 3], f2_pack(e0, e1));
                        }
                        float a0, a1, b0, b1;
                        f2_unpack(f2_add(f2_add(ls2[0], ls2[1]), f2_add(ls2[2], ls2[3])), a0, a1);
                        (void)b0; (void)b1;
                        l_run += a0 + a1;
                    }
#else
                    float ls8[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) ls8[k] = 0.0f;
#pragma unroll
                    for (int c = 0; c < 64; c += 2) {
                        const float e0 = ex2_mix<kEmu>(fmaf(__uint_as_float(sr[c]), p.scale_log2, -mo), c);
                        const float e1 = ex2_mix<kEmu>(fmaf(__uint_as_float(sr[c + 1]), p.scale_log2, -mo), c + 1);
                        const uint32_t pk = pack_bf16(e0, e1);
                        sr[c >> 1] = pk;
                        ls8[(c >> 1) & 7] += e0 + e1;
                    }
                    l_run += ((ls8[0] + ls8[1]) + (ls8[2] + ls8[3])) + ((ls8[4] + ls8[5]) + (ls8[6] + ls8[7]));
#endif
                    wait_prev_pv();
                    tmem_st32(tmem + lane_base + C::kColP + grp * (kBlockN / 2),
                              reinterpret_cast<const uint32_t(&)[32]>(sr[0]));
                    tmem_wait_st();
                } else {
                    wait_prev_pv();
                }
                }   // !CS
                }   // !hs
                // (V rows past the sample's end are zeroed by the PV issuer before the first MMA
                // that reads the tile — dual: tile 0's, which it issues before tile 1's)
                tc_fence_before();
                __syncwarp();
                if (wq == 0 && lane == 0 && hh == 0) TRACE(Jj, 4);
                if (lane == 0) mbar_arrive(&bars->p_full[grp]);
                had = true;
                Jlast = Jj;
            }
            };
            if (hs) block_loop(std::true_type{});
            else block_loop(std::false_type{});
            if constexpr (RM == 4) {
                // ---------------- dual epilogue: each warpgroup finishes its own tile ----------------
                if (had) {
                    mbar_wait(&bars->pv_done[grp], (Jlast >> 1) & 1);
                    tc_fence_after();
                }
                const bool direct = wi.part < 0;
                const int part = direct ? -1 : wi.part + grp * wi.pad;   // tile 1's parts follow tile 0's
                if constexpr (CS) {   // the row sum: both halves' partial sums
                    float* xl = reinterpret_cast<float*>(smem + C::kOffXch) + 2 * 2 * 2 * kM + grp * 2 * kM;
                    xl[hh * kM + r] = l_run;
                    named_bar_sync(8 + grp * 4 + wq, 64);
                    l_run += xl[(hh ^ 1) * kM + r];
                    named_bar_sync(8 + grp * 4 + wq, 64);   // (xl is rewritten at the next item end)
                }
                constexpr int kEpiCols = CS ? D / 2 : D;   // O columns of this warp
                if (warp_active) {
                    const float invL = (had && l_run > 0.0f) ? 1.0f / l_run : 0.0f;
                    const int h = wi.kvh * p.g + (grow % p.g);
                    __nv_bfloat16* orow = p.out + ((int64_t)(off + node) * p.Hq + h) * D;
                    float* prow = direct ? nullptr : p.part_o + ((int64_t)part * kM + rr) * D;
#pragma unroll 1
                    for (int cc = kEpiCols * hh; cc < ((p.dbg & 1) ? 0 : kEpiCols * (hh + 1)); cc += kDuEpi) {
                        uint32_t a[kDuEpi];                  // kDuEpi columns in flight per TMEM wait
#pragma unroll
                        for (int q = 0; q < kDuEpi / 16; ++q)
                            tmem_ld16(o_mine + cc + 16 * q, *reinterpret_cast<uint32_t(*)[16]>(a + 16 * q));
                        tmem_wait_ld();
#pragma unroll
                        for (int c = 0; c < kDuEpi; ++c) a[c] = __float_as_uint(__uint_as_float(a[c]) * invL);
                        if (row_valid) {
                            if (direct) {
#pragma unroll
                                for (int c = 0; c < kDuEpi; c += 8) {
                                    uint4 u;
                                    u.x = pack_bf16(__uint_as_float(a[c]), __uint_as_float(a[c + 1]));
                                    u.y = pack_bf16(__uint_as_float(a[c + 2]), __uint_as_float(a[c + 3]));
                                    u.z = pack_bf16(__uint_as_float(a[c + 4]), __uint_as_float(a[c + 5]));
                                    u.w = pack_bf16(__uint_as_float(a[c + 6]), __uint_as_float(a[c + 7]));
                                    *reinterpret_cast<uint4*>(orow + cc + c) = u;
                                }
                            } else {
#pragma unroll
                                for (int c = 0; c < kDuEpi; c += 4)
                                    *reinterpret_cast<uint4*>(prow + cc + c) = make_uint4(a[c], a[c + 1], a[c + 2], a[c + 3]);
                            }
                        }
                    }
                    if (row_valid && hh == 0) {
                        const float lse2 = (had && l_run > 0.0f) ? m_run + __log2f(l_run) : -INFINITY;
                        if (direct) {
                            if (p.lse) p.lse[(int64_t)(off + node) * p.Hq + h] = lse2 * 0.6931471805599453f;
                        } else {
                            p.part_lse[(int64_t)part * kM + rr] = lse2;
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bars->o_free);
                if (!direct) {
                    // this tile's split-KV unit (wi.unit + grp): the warpgroup that completes its
                    // last part merges all parts
                    __threadfence();
                    named_bar_sync(5 + grp, 32 * KT<RM>::kSmWarps);
                    if (wq == 0 && lane == 0 && hh == 0) {
                        const int unit = wi.unit + grp;
                        const int old = atomicAdd(&p.unit_counter[unit], 1);
                        const int last = (old == p.units[unit].n_parts - 1) ? 1 : 0;
                        if (last) p.unit_counter[unit] = 0;      // ready for the next launch
                        bars->merge_flags[grp] = last;
                    }
                    named_bar_sync(5 + grp, 32 * KT<RM>::kSmWarps);
                    if (bars->merge_flags[grp] && row_valid && warp_active) {
                        __threadfence();
                        const SplitUnit u = p.units[wi.unit + grp];
                        float M = -INFINITY;
                        for (int q = 0; q < u.n_parts; ++q)
                            M = fmaxf(M, __ldcg(p.part_lse + (int64_t)(u.part_base + q) * kM + rr));
                        float wsum = 0.0f;
                        for (int q = 0; q < u.n_parts; ++q) {
                            const float lq = __ldcg(p.part_lse + (int64_t)(u.part_base + q) * kM + rr);
                            wsum += (lq == -INFINITY) ? 0.0f : ex2(lq - M);
                        }
                        const float inv = wsum > 0.0f ? 1.0f / wsum : 0.0f;
                        const int h = wi.kvh * p.g + (grow % p.g);
                        __nv_bfloat16* orow = p.out + ((int64_t)(off + node) * p.Hq + h) * D;
#pragma unroll 1
                        for (int c0 = kEpiCols * hh; c0 < kEpiCols * (hh + 1); c0 += 8) {
                            float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                            for (int q = 0; q < u.n_parts; ++q) {
                                const float lq = __ldcg(p.part_lse + (int64_t)(u.part_base + q) * kM + rr);
                                const float wq2 = (lq == -INFINITY) ? 0.0f : ex2(lq - M) * inv;
                                const float4* src = reinterpret_cast<const float4*>(
                                    p.part_o + ((int64_t)(u.part_base + q) * kM + rr) * D + c0);
                                const float4 x0 = __ldcg(src), x1 = __ldcg(src + 1);
                                acc[0] += wq2 * x0.x; acc[1] += wq2 * x0.y; acc[2] += wq2 * x0.z; acc[3] += wq2 * x0.w;
                                acc[4] += wq2 * x1.x; acc[5] += wq2 * x1.y; acc[6] += wq2 * x1.z; acc[7] += wq2 * x1.w;
                            }
                            uint4 o;
                            o.x = pack_bf16(acc[0], acc[1]);
                            o.y = pack_bf16(acc[2], acc[3]);
                            o.z = pack_bf16(acc[4], acc[5]);
                            o.w = pack_bf16(acc[6], acc[7]);
                            *reinterpret_cast<uint4*>(orow + c0) = o;
                        }
                        if (p.lse && hh == 0) p.lse[(int64_t)(off + node) * p.Hq + h] = (M + __log2f(wsum)) * 0.6931471805599453f;
                    }
                }
                J += nv;
                wi = wn;
                w = wnx;
                continue;
            }
            // ---------------- epilogue: merge the two warpgroups' states ----------------
            if (wq == 0 && lane == 0) TRACE(J + nblk - 1, 6);
            const bool had0 = nblk >= 2 || (J & 1) == 0;
            const bool had1 = nblk >= 2 || (J & 1) == 1;
            if (had) {
                mbar_wait(&bars->pv_done[grp], (Jlast >> 1) & 1);
                tc_fence_after();
            }
            if (grp == 0 && wq == 0 && lane == 0) TRACE(J + nblk - 1, 10);
            // (m, l) exchange columns are double-buffered by item parity: a warpgroup can be at
            // most one epilogue ahead of the other (the named barrier needs both).
            const uint32_t ml_col = C::kColML + 4 * (it & 1);
            if (hs && warp_active) l_run += __shfl_xor_sync(0xffffffffu, l_run, 16);   // both key halves
            if (warp_active) {
                tmem_st2(tmem + lane_base + ml_col + 2 * grp, __float_as_uint(m_run), __float_as_uint(l_run));
                tmem_wait_st();
            }
            tc_fence_before();
            named_bar_sync(2, 256);
            if (grp == 0 && wq == 0 && lane == 0) TRACE(J + nblk - 1, 11);
            tc_fence_after();
            const bool direct = wi.part < 0;
            const int R_ = wi.rstride;
            // Direct items (D = 128): each warpgroup stages its 64-column half of the tile (bf16,
            // SW128 swizzle) and one thread stores every fully valid 16-row group with a TMA
            // store; rows of a partially valid group are stored by their threads.
            constexpr bool kStage = kStageOut && (D == 128);
            const bool staged = kStage && direct;
            uint8_t* stage = smem + C::kOffStage + grp * (kM * 128);
            const bool issuer = wq == 0 && lane == 0;
            if (staged) {
                if (issuer) bulk_wait_read_all();            // previous store done reading staging
                named_bar_sync(5 + grp, 128);
            }
            const int qgrp = hl < R_ ? (wq * R_ + (hl & ~15)) : 0;       // first logical row of my 16-row group
            const bool grp_full = staged && (qgrp + 16) <= rows;
            if (warp_active) {
                uint32_t mo_u, lo_u;
                tmem_ld2(tmem + lane_base + ml_col + 2 * (grp ^ 1), mo_u, lo_u);
                tmem_wait_ld();
                if (hs) {   // lanes 16-31 read unused TMEM lanes: take the row's values from lane - 16
                    mo_u = __shfl_sync(0xffffffffu, mo_u, hl);
                    lo_u = __shfl_sync(0xffffffffu, lo_u, hl);
                }
                const float m0 = grp == 0 ? m_run : __uint_as_float(mo_u);
                const float l0 = grp == 0 ? l_run : __uint_as_float(lo_u);
                const float m1 = grp == 1 ? m_run : __uint_as_float(mo_u);
                const float l1 = grp == 1 ? l_run : __uint_as_float(lo_u);
                const float M = fmaxf(had0 ? m0 : -INFINITY, had1 ? m1 : -INFINITY);
                const float w0 = (had0 && l0 > 0.0f) ? ex2(m0 - M) : 0.0f;
                const float w1 = (had1 && l1 > 0.0f) ? ex2(m1 - M) : 0.0f;
                const float L = l0 * w0 + l1 * w1;
                const float invL = L > 0.0f ? 1.0f / L : 0.0f;
                const float f0 = w0 * invL, f1 = w1 * invL;
                const int h = wi.kvh * p.g + (grow % p.g);
                __nv_bfloat16* orow = p.out + ((int64_t)(off + node) * p.Hq + h) * D;
                float* prow = direct ? nullptr : p.part_o + ((int64_t)wi.part * kM + rr) * D;
                const uint32_t rowbase = tmem + lane_base;
                if (grp == 0 && wq == 0 && lane == 0) TRACE(J + nblk - 1, 14);
                // my columns: [cb, cb + ncol) (half-split rows: each thread takes a quarter of D)
                const int cb = grp * (D / 2) + ((hs && (lane & 16)) ? D / 4 : 0);
                const int ncol = (p.dbg & 1) ? 0 : (hs ? D / 4 : D / 2);
#pragma unroll 1
                for (int cc = 0; cc < ncol; cc += 16) {
                    const int c0 = cb + cc;
                    uint32_t a[16], bb[16];
                    if (hs) {
                        if (had0) tmem_ld_hs16<D / 4>(rowbase + grp * (D / 2) + cc, a);
                        if (had1) tmem_ld_hs16<D / 4>(rowbase + D + grp * (D / 2) + cc, bb);
                    } else {
                        if (had0) tmem_ld16(rowbase + c0, a);
                        if (had1) tmem_ld16(rowbase + D + c0, bb);
                    }
                    tmem_wait_ld();
#pragma unroll
                    for (int c = 0; c < 16; ++c)
                        a[c] = __float_as_uint((had0 ? __uint_as_float(a[c]) * f0 : 0.0f) +
                                               (had1 ? __uint_as_float(bb[c]) * f1 : 0.0f));
                    if (grp == 0 && wq == 0 && lane == 0 && cc == 0) TRACE(J + nblk - 1, 15);
                    if (row_valid) {
                        if (direct) {
#pragma unroll
                            for (int c = 0; c < 16; c += 8) {
                                uint4 u;
                                u.x = pack_bf16(__uint_as_float(a[c]), __uint_as_float(a[c + 1]));
                                u.y = pack_bf16(__uint_as_float(a[c + 2]), __uint_as_float(a[c + 3]));
                                u.z = pack_bf16(__uint_as_float(a[c + 4]), __uint_as_float(a[c + 5]));
                                u.w = pack_bf16(__uint_as_float(a[c + 6]), __uint_as_float(a[c + 7]));
                                if (grp_full) {
                                    const int chunk = ((c0 + c) - grp * (D / 2)) >> 3;   // 16-byte chunk in the 128-byte row
                                    *reinterpret_cast<uint4*>(stage + rr * 128 + ((chunk ^ (rr & 7)) << 4)) = u;
                                } else {
                                    *reinterpret_cast<uint4*>(orow + c0 + c) = u;
                                }
                            }
                        } else {
#pragma unroll
                            for (int c = 0; c < 16; c += 4)
                                *reinterpret_cast<uint4*>(prow + c0 + c) = make_uint4(a[c], a[c + 1], a[c + 2], a[c + 3]);
                        }
                    }
                }
                if (row_valid && grp == 0 && hl == lane) {
                    const float lse2 = L > 0.0f ? M + __log2f(L) : -INFINITY;
                    if (direct) {
                        if (p.lse) p.lse[(int64_t)(off + node) * p.Hq + h] = lse2 * 0.6931471805599453f;
                    } else {
                        p.part_lse[(int64_t)wi.part * kM + rr] = lse2;
                    }
                }
            }
            tc_fence_before();
            if (grp == 0 && wq == 0 && lane == 0) TRACE(J + nblk - 1, 12);
            if (staged) {
                fence_proxy_async_smem();
                named_bar_sync(5 + grp, 128);
                if (issuer) {
                    const int row0 = wi.mtile * 4 * R_;
                    const int nodeb = off;
                    for (int q = 0; q < 4; ++q)
                        for (int t = 0; t < R_; t += 16)
                            if (q * R_ + t + 16 <= rows)
                                tma_store_3d(&tmO, stage + (32 * q + t) * 128, grp * (D / 2), wi.kvh * p.g,
                                             nodeb + (row0 + q * R_ + t) / p.g);
                    bulk_commit_group();
                    if (grp == 0) TRACE(J + nblk - 1, 13);
                }
            }
            __syncwarp();
            if (wq == 0 && lane == 0 && grp == 0) TRACE(J + nblk - 1, 7);
            if (lane == 0) mbar_arrive(&bars->o_free);
            if (wi.part >= 0) {
                // split-KV unit: the CTA that completes its last part merges all parts
                // o = sum_q 2^(lse_q - M) o_q / sum_q 2^(lse_q - M)  (threadfence-reduction pattern)
                __threadfence();
                named_bar_sync(3, 256);
                if (threadIdx.x == 128) {
                    const int old = atomicAdd(&p.unit_counter[wi.unit], 1);
                    const int last = (old == p.units[wi.unit].n_parts - 1) ? 1 : 0;
                    if (last) p.unit_counter[wi.unit] = 0;          // ready for the next launch
                    bars->merge_flag = last;
                }
                named_bar_sync(3, 256);
                if (bars->merge_flag && row_valid) {
                    __threadfence();
                    const SplitUnit u = p.units[wi.unit];
                    float M = -INFINITY;
                    for (int q = 0; q < u.n_parts; ++q)
                        M = fmaxf(M, __ldcg(p.part_lse + (int64_t)(u.part_base + q) * kM + rr));
                    float wsum = 0.0f;
                    for (int q = 0; q < u.n_parts; ++q) {
                        const float lq = __ldcg(p.part_lse + (int64_t)(u.part_base + q) * kM + rr);
                        wsum += (lq == -INFINITY) ? 0.0f : ex2(lq - M);
                    }
                    const float inv = wsum > 0.0f ? 1.0f / wsum : 0.0f;
                    const int h = wi.kvh * p.g + (grow % p.g);
                    __nv_bfloat16* orow = p.out + ((int64_t)(off + node) * p.Hq + h) * D;
#pragma unroll 1
                    const int mcb = grp * (D / 2) + ((hs && (lane & 16)) ? D / 4 : 0);
                    const int mce = mcb + (hs ? D / 4 : D / 2);
                    for (int c0 = mcb; c0 < mce; c0 += 8) {
                        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                        for (int q = 0; q < u.n_parts; ++q) {
                            const float lq = __ldcg(p.part_lse + (int64_t)(u.part_base + q) * kM + rr);
                            const float wq = (lq == -INFINITY) ? 0.0f : ex2(lq - M) * inv;
                            const float4* src = reinterpret_cast<const float4*>(
                                p.part_o + ((int64_t)(u.part_base + q) * kM + rr) * D + c0);
                            const float4 x0 = __ldcg(src), x1 = __ldcg(src + 1);
                            acc[0] += wq * x0.x; acc[1] += wq * x0.y; acc[2] += wq * x0.z; acc[3] += wq * x0.w;
                            acc[4] += wq * x1.x; acc[5] += wq * x1.y; acc[6] += wq * x1.z; acc[7] += wq * x1.w;
                        }
                        uint4 o;
                        o.x = pack_bf16(acc[0], acc[1]);
                        o.y = pack_bf16(acc[2], acc[3]);
                        o.z = pack_bf16(acc[4], acc[5]);
                        o.w = pack_bf16(acc[6], acc[7]);
                        *reinterpret_cast<uint4*>(orow + c0) = o;
                    }
                    if (grp == 0 && p.lse && hl == lane)
                        p.lse[(int64_t)(off + node) * p.Hq + h] = (M + __log2f(wsum)) * 0.6931471805599453f;
                }
            }
            J += nblk;
            wi = wn;
            w = wnx;
        }
        if (wq == 0 && lane == 0) bulk_wait_all();   // output TMA stores complete before exit
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) tmem_dealloc<C::kTmemCols>(tmem);
    if (p.dyn && threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(p.qctr + 1, 1) == (int)gridDim.x - 1) {   // last CTA out: ready for the next launch
            p.qctr[0] = 0;
            p.qctr[1] = 0;
            __threadfence();
        }
    }
    if (p.trace && threadIdx.x == 0) p.trace[((size_t)blockIdx.x * kTraceJ + kTraceJ - 1) * 16 + 15] = globaltimer_ns();
}

}  // namespace attn
