/* rlhfspec_core — C ABI of the RLHFSpec verification hot path on B200 (sm_100a).
 *
 * Paper: RLHFSpec (arXiv 2512.04752), /root/reference/PAPER.md, cited P:<line>.
 * Scope: DESIGN.md §1 / SURVEY.md §8. Readings Z1..Z27: DESIGN.md §2.
 *
 * Conventions (all entry points)
 *  - Every call returns rs_status (RS_OK = 0). No exception crosses the ABI. On error,
 *    rs_last_error() returns a thread-local, NUL-terminated message (valid until the next
 *    call on the same thread).
 *  - "device" pointers are caller-owned CUDA global-memory buffers on the current device;
 *    "host" pointers are caller-owned CPU memory. The library never frees caller memory and
 *    keeps no pointer past the call unless stated (rs_ctx registrations).
 *  - Kernels are enqueued on `stream` (a cudaStream_t passed as void*; NULL = legacy default
 *    stream) and are asynchronous: outputs are valid once the stream reaches that point.
 *    Host-only calls are synchronous.
 *  - No allocation happens on hot calls; workspace is caller-provided (size queries given).
 *  - Data errors found on the device (malformed tree, non-finite logits) do not become a
 *    return code: they set per-sample bits in `status_flags` (RS_FLAG_*).
 *  - Tensor layouts are row-major, innermost index last. bf16 = IEEE bfloat16 bit pattern.
 *  - Tree conventions (Z1): sample b owns flattened nodes tree_off[b] .. tree_off[b+1]-1
 *    (T_b = tree_off[b+1]-tree_off[b], 1 <= T_b <= 64); parent[] and path[] hold LOCAL node
 *    indices; node 0 is the root (the last committed token), parent[0] = -1, parent[i] < i.
 *  - KV cache (one tensor per layer): [num_pages, Hkv, page_size, head_dim] bf16; logical slot
 *    j of sample b is page block_table[b*max_pages + j/page_size], row j%page_size. Slots
 *    0..P_b-1 hold the committed prefix, slot P_b+i holds tree node i (written upstream).
 */
#ifndef RLHFSPEC_CORE_H
#define RLHFSPEC_CORE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RS_OK = 0,
    RS_ERR_INVALID_ARG = 1,        /* bad size / null pointer / out-of-range argument       */
    RS_ERR_MALFORMED_TREE = 2,     /* host-checked tree is not a topological tree    */
    RS_ERR_EMPTY_TREE = 3,         /* no candidate nodes                             */
    RS_ERR_INSUFFICIENT_NODES = 4, /* fewer candidates than n_min                     */
    RS_ERR_NONFINITE = 5,
    RS_ERR_NO_MEMORY = 6,          /* page reservation refused (migration handshake) */
    RS_ERR_LAYOUT_MISMATCH = 7,    /* migration header / buffer disagree            */
    RS_ERR_UNSUPPORTED = 8,        /* shape outside what the kernels implement              */
    RS_ERR_CUDA = 9,
    RS_ERR_NCCL = 10,
    RS_ERR_WORKSPACE = 11          /* workspace too small                                   */
} rs_status;

enum { RS_FLAG_MALFORMED = 1, RS_FLAG_NONFINITE = 2, RS_FLAG_INSUFFICIENT = 4 };
enum { RS_ACCEPT_GREEDY = 0, RS_ACCEPT_SAMPLE_DELTA = 1, RS_ACCEPT_SAMPLE_MSS = 2 };
enum { RS_DTYPE_BF16 = 0, RS_DTYPE_F32 = 1 };
#define RS_MAX_TREE 64

const char* rs_last_error(void);
const char* rs_version(void);

/* ===================================================================================== a1
 * rs_tree_build_mask — ancestor-or-self bitmask and depth per tree node ("each branch
 * represents a token sequence awaiting verification"; Z3).
 *   parent    device int32 [NT]   local parent index, -1 for the root
 *   tree_off  device int32 [B+1]
 *   tree_mask device uint64 [NT]  out: bit j set <=> local node j is on Path(root, i)
 *   depth     device int32 [NT]   out: root depth 0
 *   status_flags device int32 [B] out: RS_FLAG_MALFORMED if the tree is not topological or
 *             T_b outside [1, 64] (that sample's mask/depth are then zero)
 */
rs_status rs_tree_build_mask(const int32_t* parent, const int32_t* tree_off, int32_t B,
                             uint64_t* tree_mask, int32_t* depth, int32_t* status_flags,
                             void* stream);

/* ===================================================================================== f2
 * LM head fused with greedy acceptance. Verification scores every tree node
 * in one target pass; the LM head is one of its GEMMs; greedy acceptance
 * needs only each node's arg-max (DESIGN Z5, Z6). rs_lm_head_argmax computes
 *     argmax_token[r] = argmax_v  sum_k hidden[r,k] * weight[v,k]      (ties -> lowest v)
 * with fp32 accumulation on the tensor cores, reducing inside the GEMM epilogue, so the
 * [rows, V] logits are never written.
 *   hidden   device bf16 [rows, Dm] (final hidden state of each tree node, node-major as Q)
 *   weight   device bf16 [V, Dm] (nn.Linear layout); both 16-byte aligned; Dm % 64 == 0
 *   argmax_token device int32 [rows] out (-1 if any logit of the row is NaN or +-Inf: no arg-max, Z15)
 *   max_logit    device fp32 [rows] out (the fp32 maximum), or NULL
 *   ws, ws_bytes device workspace >= rs_lm_head_argmax_workspace_bytes(rows), 8-byte aligned
 * Launches a memset, the GEMM kernel and a finalize kernel on `stream`. */
/* rs_lm_head_logits — the same GEMM for the sampling modes (SAMPLE_DELTA / SAMPLE_MSS need
 * whole rows): logits[r, v] = bf16_RN( sum_k hidden[r,k] * weight[v,k] ), fp32 accumulation on the
 * tensor cores, the bf16 tile written by the epilogue (the input of rs_tree_accept_compact).
 *   hidden, weight as above; logits device bf16 [rows, V] out, 16-byte aligned; V % 8 == 0.
 * Errors: Dm not a positive multiple of 64, V % 8 != 0 or misaligned pointers -> RS_ERR_INVALID_ARG. */
rs_status rs_lm_head_logits(const void* hidden, const void* weight, int32_t rows, int32_t V, int32_t Dm,
                            void* logits, void* stream);
size_t rs_lm_head_argmax_workspace_bytes(int32_t rows);
rs_status rs_lm_head_argmax(const void* hidden, const void* weight, int32_t rows, int32_t V, int32_t Dm,
                            int32_t* argmax_token, float* max_logit, void* ws, size_t ws_bytes,
                            void* stream);

/* Greedy walk given the per-node arg-max: from the root, move to the
 * lowest-index child whose token equals argmax_token[current]; stop when none does.
 *   argmax_token, parent, token device int32 [NT]; tree_off device int32 [B+1]
 *   accepted_len [B], path [B,64] (-1 padded), bonus_token [B], status_flags [B]: as
 *   rs_tree_accept GREEDY. A malformed tree sets RS_FLAG_MALFORMED (accepted_len 0, bonus -1);
 *   a visited node with argmax_token < 0 sets RS_FLAG_NONFINITE (bonus -1). */
rs_status rs_tree_accept_greedy_tokens(const int32_t* argmax_token, const int32_t* parent,
                                       const int32_t* token, const int32_t* tree_off, int32_t B,
                                       int32_t* accepted_len, int32_t* path, int32_t* bonus_token,
                                       int32_t* status_flags, void* stream);
/* rs_tree_accept_greedy_tokens followed by rs_kv_compact in ONE launch (the f2 walk with the
 * KV commit, as rs_tree_accept_compact is for logits): a CTA per (sample, pair of layers) walks
 * the sample's tree on the per-node arg-max tokens and commits its layers' share of the path.
 * Outputs identical to the two calls in sequence; KV arguments as rs_kv_compact (L <= 256, else
 * RS_ERR_INVALID_ARG; head_dim % 8 != 0 -> RS_ERR_UNSUPPORTED). */
rs_status rs_tree_accept_greedy_tokens_compact(const int32_t* argmax_token, const int32_t* parent,
                                               const int32_t* token, const int32_t* tree_off, int32_t B,
                                               int32_t* accepted_len, int32_t* path, int32_t* bonus_token,
                                               int32_t* status_flags, void* const* k_layers_host,
                                               void* const* v_layers_host, int32_t L, int32_t Hkv,
                                               int32_t head_dim, int32_t page_size, const int32_t* block_table,
                                               int32_t max_pages, const int32_t* prefix_len, int32_t* new_len,
                                               int32_t* moves, void* stream);

/* ===================================================================================== f3
 * rs_tree_select — the verification trees of a batch, built on the GPU from the draft's
 * candidate trees for the n chosen by rs_select_strategy ("the selection of n";
 * P:217-227 layer-level search; readings Z1, Z6, Z9, Z11 in DESIGN.md):
 *   dl(u) = o(u) * dl(parent(u)); w(u) = F(dl(u)) (F: piecewise linear through the knots as
 *   np.interp, clamped to [0, 1]); S(n) = the first n pops of the search (queue order: w desc,
 *   depth asc, id asc); tree = root (node 0, token root_token[b]) + S(n) in ascending candidate
 *   index with re-indexed parents (a candidate with parent -1 hangs under node 0).
 *   cand_parent device int32 [NC]  parent candidate index (< i) or -1 (child of the root)
 *   cand_o      device f64 [NC]    draft acceptance estimates o(u)
 *   cand_token  device int32 [NC]; cand_off device int32 [B+1] (<= 256 candidates per sample)
 *   root_token  device int32 [B]   the last committed token of each sample
 *   n           1..63: every tree gets T = n + 1 nodes (tree_off[b] = b * (n + 1))
 *   knots_x, knots_y device f64 [n_knots], 2 <= n_knots <= 16, knots_x increasing
 *   parent_out, token_out, depth_out device int32 [B*(n+1)]; tree_mask_out device u64 [B*(n+1)]
 *               (exactly what rs_tree_build_mask would give for parent_out)
 *   status_flags device int32 [B]: RS_FLAG_MALFORMED (candidate parents not topological, an
 *               o(u) outside [0, 1] or NaN, > 256 candidates, knots not strictly increasing in x
 *               and non-decreasing in y (checked on the device: every sample flagged), or a
 *               selected node whose parent was not selected — its token is then -1) /
 *               RS_FLAG_INSUFFICIENT (the search ran out before n pops); such a sample's missing
 *               nodes are children of the root with token -1, which rs_tree_accept flags.
 * Errors: n outside [1, 63] -> RS_ERR_UNSUPPORTED; n_knots outside [2, 16] / null ->
 * RS_ERR_INVALID_ARG. */
rs_status rs_tree_select(const int32_t* cand_parent, const double* cand_o, const int32_t* cand_token,
                         const int32_t* cand_off, const int32_t* root_token, int32_t B, int32_t n,
                         const double* knots_x, const double* knots_y, int32_t n_knots,
                         int32_t* parent_out, int32_t* token_out, uint64_t* tree_mask_out,
                         int32_t* depth_out, int32_t* status_flags, void* stream);

/* ===================================================================================== a2
 * Tree-verification attention (P:76-80 single-pass verification of all tree tokens; P:213
 * "attention primarily incurs cost due to KVCache loading"). For sample b, q head h
 * (kv head h/g), node i:  o = softmax_j(q.k_j * sm_scale) v_j over
 *   j in {0..P_b-1} U {P_b + t : bit t of tree_mask[tree_off[b]+i]}.
 * Implemented for head_dim in {64, 128}, page_size = 64, Hq % Hkv == 0, T_b*g <= 512.
 *
 * Plan/run split: the plan is host metadata built from HOST copies of prefix_len and tree_off
 * (the lengths of this step; reused by every layer), uploaded once into device workspace.
 */
typedef struct rs_attn_plan rs_attn_plan;

/* prefix_len_host int32 [B], tree_off_host int32 [B+1]; num_ctas: persistent grid size,
 * 0 = number of SMs of the current device. */
rs_status rs_attn_plan_create(const int32_t* prefix_len_host, const int32_t* tree_off_host,
                              int32_t B, int32_t Hq, int32_t Hkv, int32_t head_dim,
                              int32_t page_size, int32_t num_ctas, rs_attn_plan** plan_out);
/* Device workspace bytes the plan needs (schedule + split-KV partials). */
size_t rs_attn_plan_workspace_bytes(const rs_attn_plan* plan);
/* Copy the schedule into `ws` (device, >= rs_attn_plan_workspace_bytes, 256-byte aligned). */
rs_status rs_attn_plan_upload(const rs_attn_plan* plan, void* ws, size_t ws_bytes, void* stream);
/* Number of work items / split units (for reporting). */
rs_status rs_attn_plan_info(const rs_attn_plan* plan, int32_t* num_ctas, int32_t* num_items,
                            int32_t* num_split_units);
/* Copy the schedule out (for inspection / tests): cta_off host int32 [num_ctas+1] (items of
 * CTA c are [cta_off[c], cta_off[c+1])), items host int32 [num_items, 12] =
 * (sample, kv_head, m_tile, first_block, end_block, partial_slot or -1, rows per TMEM
 * sub-partition R, split unit or -1, prefix_len, tree_off, tree size, 0). Either may be NULL. */
rs_status rs_attn_plan_items(const rs_attn_plan* plan, int32_t* cta_off, int32_t* items);
void rs_attn_plan_destroy(rs_attn_plan* plan);
/* Programmatic dependent launch (PDL). Every attention launch may begin while the previous
 * kernel on the stream drains; by default it reads NOTHING written by kernels (K/V, block
 * table, Q, masks) before that kernel has completed (griddepcontrol.wait). enable = 1 lets the
 * K/V producers stream the PREFIX blocks (every slot < P_b) and read the block table early: set
 * it only when no kernel that may still be running when the attention launch is enqueued writes
 * the prefix K/V pages or the block table (e.g. the previous step's rs_kv_compact is separated
 * from this launch by another kernel, as in a verify step: mask build, then the layers). Blocks
 * holding tree slots (P_b + i) are always read after the wait, so the tree K/V may be written by
 * the kernel immediately before (the QKV/RoPE projection). Applies to later launches with this
 * plan. */
rs_status rs_attn_plan_set_early_prefix(rs_attn_plan* plan, int32_t enable);
/* Profiling hook: when buf (device, >= num_ctas*256*8*8 bytes) is set, every attention launch
 * records clock64() per (CTA, block, event) — see csrc/attention.cu. NULL disables. */
rs_status rs_attn_set_trace(void* buf, size_t bytes);

/* q        device bf16 [NT, Hq, head_dim] (post-RoPE)
 * k_pages, v_pages device bf16 [num_pages, Hkv, page_size, head_dim] (one layer)
 * block_table device int32 [B, max_pages]; prefix_len device int32 [B]; tree_off device int32 [B+1]
 * tree_mask device uint64 [NT] (rs_tree_build_mask)
 * out      device bf16 [NT, Hq, head_dim]
 * lse      device fp32 [NT, Hq] natural-log log-sum-exp, or NULL
 * ws       the workspace the plan was uploaded into (the partials area is overwritten).
 * The plan must have been created for the same B/Hq/Hkv/head_dim/page_size and lengths. */
rs_status rs_tree_verify_attention(const rs_attn_plan* plan, const void* q, const void* k_pages,
                                   const void* v_pages, int64_t num_pages,
                                   const int32_t* block_table, int32_t max_pages,
                                   const int32_t* prefix_len, const int32_t* tree_off,
                                   const uint64_t* tree_mask, int32_t B, int32_t Hq, int32_t Hkv,
                                   int32_t head_dim, int32_t page_size, float sm_scale, void* out,
                                   float* lse, void* ws, size_t ws_bytes, void* stream);

/* All L layers of one verify step in one call (same plan, tree mask and workspace; per-layer
 * host arrays of device pointers q_layers/k_layers/v_layers/out_layers[L], lse_layers[L] or
 * NULL). Launches L kernels back to back on `stream`. */
rs_status rs_tree_verify_attention_layers(
    const rs_attn_plan* plan, int32_t L, const void* const* q_layers, const void* const* k_layers,
    const void* const* v_layers, int64_t num_pages, const int32_t* block_table, int32_t max_pages,
    const int32_t* prefix_len, const int32_t* tree_off, const uint64_t* tree_mask, int32_t B, int32_t Hq,
    int32_t Hkv, int32_t head_dim, int32_t page_size, float sm_scale, void* const* out_layers,
    float* const* lse_layers, void* ws, size_t ws_bytes, void* stream);

/* ===================================================================================== a3
 * rs_tree_accept — walk each sample's tree from the root and return its longest accepted
 * path and the bonus token (rule per mode in DESIGN.md §2 Z5-Z8, bit-exact
 * arithmetic in "Bit-exact sampling").
 *   mode        RS_ACCEPT_GREEDY | RS_ACCEPT_SAMPLE_DELTA | RS_ACCEPT_SAMPLE_MSS
 *   logits      device [NT, V], RS_DTYPE_BF16 or RS_DTYPE_F32 (target LLM row per node)
 *   draft_probs device fp32 [NT, V]: row c = the draft distribution the children of c were
 *               drawn from (MSS only; must be NULL otherwise); read only for nodes that have
 *               children (Z29)
 *   parent, token device int32 [NT]; tree_off device int32 [B+1]; gid device int64 [B]
 *               (global sample ids; the RNG is keyed by gid, so results do not depend on
 *               which GPU/slot holds the sample)
 *   temperature > 0 (sampling modes; ignored by GREEDY); seed, step: RNG key / counter
 *   accepted_len device int32 [B]  out: a_b (accepted drafts, bonus excluded)
 *   path         device int32 [B, 64] out: path[b][0..a_b] local node ids (path[b][0]=0), -1 padded
 *   bonus_token  device int32 [B]  out: the bonus token (-1 on a flagged sample)
 *   status_flags device int32 [B]  out: RS_FLAG_* bits. RS_FLAG_MALFORMED (accepted_len 0,
 *               bonus -1): T_b outside [1, 64], parent[0] != -1, parent[i] outside [0, i), or a
 *               draft node (i >= 1) whose token is outside [0, V) (e.g. rs_tree_select's -1 pad).
 *               RS_FLAG_NONFINITE: a visited row holds NaN/Inf logits, or (MSS) the draft row of
 *               a visited node with children holds a value outside [0, 1] or NaN (walk stops
 *               there, bonus -1).
 *   ws, ws_bytes: device workspace >= rs_tree_accept_workspace_bytes(mode, B, V) bytes, 16-byte
 *               aligned; currently 0 bytes for every mode (MSS keeps the visited row and its
 *               residual in the cluster's shared memory), so NULL is allowed; too small ->
 *               RS_ERR_WORKSPACE. */
size_t rs_tree_accept_workspace_bytes(int32_t mode, int32_t B, int32_t V);
/* As rs_tree_accept with the draft probabilities' dtype given: draft_dtype RS_DTYPE_F32 or
 * RS_DTYPE_BF16 (a bf16 value is used as the fp32 number it denotes, so the arithmetic of
 * "Bit-exact sampling" is unchanged; a bf16 row is 2/3 of the bytes). rs_tree_accept = the F32 form. */
rs_status rs_tree_accept_ex(int32_t mode, const void* logits, int32_t logits_dtype, const void* draft_probs,
                            int32_t draft_dtype, const int32_t* parent, const int32_t* token,
                            const int32_t* tree_off, const int64_t* gid, int32_t B, int32_t V,
                            float temperature, uint64_t seed, uint64_t step, int32_t* accepted_len,
                            int32_t* path, int32_t* bonus_token, int32_t* status_flags, void* ws,
                            size_t ws_bytes, void* stream);
rs_status rs_tree_accept(int32_t mode, const void* logits, int32_t logits_dtype,
                         const float* draft_probs, const int32_t* parent, const int32_t* token,
                         const int32_t* tree_off, const int64_t* gid, int32_t B, int32_t V,
                         float temperature, uint64_t seed, uint64_t step, int32_t* accepted_len,
                         int32_t* path, int32_t* bonus_token, int32_t* status_flags, void* ws,
                         size_t ws_bytes, void* stream);

/* Device-side Philox4x32-10 and exp_spec over arrays (conformance hooks for the parity
 * tests; the same device functions the acceptance kernel uses).
 *   ctr device uint32 [n,4], key uint32 [2] (host), out device uint32 [n,4]
 *   x device fp32 [n] (x <= 0), y device fp32 [n] */
rs_status rs_philox4x32_10(const uint32_t* ctr, int64_t n, const uint32_t* key_host, uint32_t* out,
                           void* stream);
rs_status rs_exp_spec(const float* x, int64_t n, float* y, void* stream);

/* ===================================================================================== a4
 * rs_kv_compact — commit the accepted path's K/V (only this step's KVCache changes):
 *   for k = 1..a_b:  K/V[b, slot P_b+k] <- K/V[b, slot P_b+path[b][k]]   (every layer, head)
 *   new_len[b] = P_b + 1 + a_b
 * with sequential ascending-k semantics (rows are gathered before any is written).
 *   k_layers_host, v_layers_host  host arrays of L device pointers (one bf16 cache per layer)
 *   accepted_len, path   device outputs of rs_tree_accept
 *   new_len  device int32 [B] out; moves device int32 [B, 64, 2] out (src_slot, dst_slot per
 *            k = 1..a_b, -1 padded) or NULL. Flagged samples (accepted_len 0) move nothing. */
rs_status rs_kv_compact(void* const* k_layers_host, void* const* v_layers_host, int32_t L,
                        int64_t num_pages, int32_t Hkv, int32_t head_dim, int32_t page_size,
                        const int32_t* block_table, int32_t max_pages, const int32_t* prefix_len,
                        const int32_t* accepted_len, const int32_t* path, int32_t B,
                        int32_t* new_len, int32_t* moves, void* stream);

/* rs_tree_accept_compact — rs_tree_accept_ex followed by rs_kv_compact in ONE launch (a3 + a4,
 * P:76-80 then P:303): the cluster that walks sample b's tree commits its path's K/V as soon as
 * its walk ends (the other samples are still walking), so no second launch or pass over the
 * path. Every output (accepted_len, path, bonus_token, status_flags, new_len, moves and the K/V
 * bytes) is identical to the two calls in sequence; arguments as in rs_tree_accept_ex and
 * rs_kv_compact (num_pages is not needed). L <= 256 (else RS_ERR_INVALID_ARG: use the two
 * calls); head_dim % 8 != 0 -> RS_ERR_UNSUPPORTED. The K/V pointers are read at launch (they are
 * kernel parameters, so a captured CUDA graph keeps the layer list it was captured with).
 *   draft_row  MSS only (else must be NULL): device int32 [NT] or NULL. NULL: node i's draft
 *              distribution is row i of draft_probs ([NT, V], as in rs_tree_accept_ex). Else
 *              draft_probs is [R, V] holding only the rows that are used, and draft_row[i] is the
 *              row of node i (-1 for a node without children; a non-negative entry must index a
 *              row of draft_probs: the caller's guarantee, not checked). Either way the draft row of a node
 *              WITHOUT children is never read (Z29: nothing was drawn from it; a visited
 *              leaf's bonus comes from the target weights), so a caller uploads only the rows of
 *              nodes with children; a node with children whose draft_row is negative sets
 *              RS_FLAG_MALFORMED (accepted_len 0, bonus -1). */
rs_status rs_tree_accept_compact(int32_t mode, const void* logits, int32_t logits_dtype, const void* draft_probs,
                                 int32_t draft_dtype, const int32_t* draft_row, const int32_t* parent,
                                 const int32_t* token,
                                 const int32_t* tree_off, const int64_t* gid, int32_t B, int32_t V,
                                 float temperature, uint64_t seed, uint64_t step, int32_t* accepted_len,
                                 int32_t* path, int32_t* bonus_token, int32_t* status_flags, void* ws,
                                 size_t ws_bytes, void* const* k_layers_host, void* const* v_layers_host,
                                 int32_t L, int32_t Hkv, int32_t head_dim, int32_t page_size,
                                 const int32_t* block_table, int32_t max_pages, const int32_t* prefix_len,
                                 int32_t* new_len, int32_t* moves, void* stream);

/* ===================================================================================== a0
 * Workload-aware drafting-strategy selection: n = argmax al(n)/t_sd(n) (Eq. 2)
 * by layer-level priority-queue search with early stop (Eq. 3). Host only. */
typedef struct {
    double c_draft, b0, b1, b2, b3, k_sat;   /* t_sd = c_draft+b0+b1*Nseq+b2*Nd+b3*relu(Nd-k)*Nd */
    int32_t seq_bucket, draft_bucket;        /* bucket widths of the prediction cache   */
} rs_cost_model;

typedef struct {
    int32_t n, depth, width;     /* chosen draft-token num and the depth/width of T = n+1 trees */
    int32_t n_stop;              /* n at which the early stop fired (or the last n searched)   */
    int32_t cache_hit;           /* 1 if t_sd(n) of the chosen n came from the bucket cache     */
    int32_t cache_entries;
    double al, t_sd, objective;  /* predicted al(n) (sum of w over S(n), all samples), t_sd, ratio */
} rs_strategy;

typedef struct rs_selector rs_selector;
/* knots_x/knots_y host double [n_knots]: the acceptance fit F (monotone piecewise linear,
 * clamped to [0,1]). */
rs_status rs_selector_create(const rs_cost_model* cost, const double* knots_x,
                             const double* knots_y, int32_t n_knots, rs_selector** out);
void rs_selector_destroy(rs_selector* sel);
/* cand_parent host int32 [N] (per sample, -1 = child of the committed root, parent < index),
 * cand_o host double [N] draft probabilities o(v) in (0,1], cand_off host int32 [B+1],
 * prefix_len host int32 [B]. selected: host int32 [B, n_max] candidate ids in selection order
 * (the first n of each row form S_b(n)) up to out->n_stop — the search runs step-major over the
 * batch and stops with the objective's early stop (Eq. 3) — then -1, or NULL. */
rs_status rs_select_strategy(rs_selector* sel, const int32_t* cand_parent, const double* cand_o,
                             const int32_t* cand_off, const int32_t* prefix_len, int32_t B,
                             int32_t n_min, int32_t n_max, int32_t patience, rs_strategy* out,
                             int32_t* selected);
/* dl(u) = o(u) * dl(parent(u)) of every candidate (Z9), host arrays as rs_select_strategy. */
rs_status rs_draft_logits(const int32_t* cand_parent, const double* cand_o, const int32_t* cand_off,
                          int32_t B, double* dl_out);
/* The acceptance fit F from observations ("fit a function ... between draft logits and token
 * acceptance probability based on offline profiling data"; reading Z24): dl, accepted
 * host double [n] (accepted in [0,1]: 0/1 outcomes or rates); n_buckets equal-width buckets of dl
 * over [0,1] (dl clipped); per non-empty bucket the mean dl and mean acceptance weighted by its
 * count; a weighted pool-adjacent-violators pass makes the rates non-decreasing. Writes
 * *n_knots <= n_buckets knots (x strictly increasing, y non-decreasing) into knots_x/knots_y
 * (capacity n_buckets). RS_ERR_INVALID_ARG ("InsufficientData") with < 2 distinct dl values. */
rs_status rs_acceptance_fit(const double* dl, const double* accepted, int64_t n, int32_t n_buckets,
                            double* knots_x, double* knots_y, int32_t* n_knots);
/* Least-squares fit of the cost model's b0..b3 (c_draft kept) to measured step times. */
rs_status rs_cost_model_fit(const double* n_seq, const double* n_draft, const double* t_sec,
                            int32_t n, rs_cost_model* inout);

/* ===================================================================================== ctx
 * rs_ctx — one generation instance (one process per GPU): non-owning registrations of its KV
 * pools (model 0 = SSM, 1 = LLM; [num_pages, Hkv, page_size, head_dim] bf16 per layer, kept until
 * rs_ctx_destroy) and its drafting-strategy state: the acceptance fit F and the t_sd cost model,
 * with the selector built from them (rs_ctx_selector; pass it to rs_select_strategy). Not
 * thread-safe; distinct ctxs are independent. */
typedef struct { int32_t rank, world, page_size; } rs_ctx_desc;
typedef struct rs_ctx rs_ctx;
rs_status rs_ctx_create(const rs_ctx_desc* desc, rs_ctx** out);
rs_status rs_ctx_destroy(rs_ctx* ctx);
rs_status rs_ctx_register_kv(rs_ctx* ctx, int32_t model, int32_t L, void* const* k_layers,
                             void* const* v_layers, int32_t num_pages, int32_t Hkv, int32_t head_dim);
/* Set the cost model (cost may be NULL: kept) and/or F's knots (knots NULL: kept); rebuilds the
 * selector (empty bucket cache). Invalid knots -> RS_ERR_INVALID_ARG and nothing changes. */
rs_status rs_ctx_set_strategy(rs_ctx* ctx, const rs_cost_model* cost, const double* knots_x,
                              const double* knots_y, int32_t n_knots);
/* *n_knots: in = capacity of knots_x/knots_y (may be NULL), out = number of knots. */
rs_status rs_ctx_get_strategy(const rs_ctx* ctx, rs_cost_model* cost, double* knots_x, double* knots_y,
                              int32_t* n_knots);
/* The ctx's selector (borrowed; NULL until F is set). Invalidated by the next set/fit/calibrate. */
rs_selector* rs_ctx_selector(rs_ctx* ctx);
/* Refit F from (dl, accepted) observations (rs_acceptance_fit) — offline profiling data, or the
 * online data P:192 collects to update the function. */
rs_status rs_ctx_fit_acceptance(rs_ctx* ctx, const double* dl, const double* accepted, int64_t n,
                                int32_t n_buckets);

/* rs_calibrate — the offline profiling of the t_sd regression on THIS box:
 * for every grid point (B[i], P[i], T[i]) a synthetic batch (every sample prefix P, a chain tree
 * of T nodes, consecutive pages of the registered LLM pools) runs the tree-mask build and the
 * verification attention of every registered LLM layer (the library's kernels, `reps` timed
 * repetitions after one warm-up, median, CUDA events on `stream`); the point's step time is
 *   c_draft + t_attention + dense_s_per_token * B*T
 * (dense_s_per_token: the verification FFN / projections per verified token, outside this
 * library — measure them, e.g. with rs_lm_head_argmax's GEMM rate, and pass them in), and
 * rs_cost_model_fit fits b0..b3 with N_seq = B*P, N_draft = B*T (c_draft, k_sat and the buckets
 * of the ctx's current cost model are kept). The ctx's selector is rebuilt with the fit. Reads
 * the registered pools, writes only the caller's q/out scratch and workspace.
 *   q, out   device bf16 scratch >= max_i B*T*Hq*head_dim elements each (qo_elems)
 *   ws       device, >= rs_calibrate_workspace_bytes(ctx, desc), 256-byte aligned
 *   t_attn_out host double [n_points] (measured attention + mask seconds per point) or NULL */
typedef struct {
    int32_t Hq;
    int32_t n_points;
    const int32_t* B;
    const int32_t* P;
    const int32_t* T;
    int32_t reps;
    void* q;
    void* out;
    size_t qo_elems;
    void* ws;
    size_t ws_bytes;
    double dense_s_per_token;
    void* stream;
} rs_calib_desc;
size_t rs_calibrate_workspace_bytes(const rs_ctx* ctx, const rs_calib_desc* desc);
rs_status rs_calibrate(rs_ctx* ctx, const rs_calib_desc* desc, double* t_attn_out);

/* ===================================================================================== a6
 * Sample reallocation policy. Host only. */
/* Knee of the throughput-vs-sample-count curve (Z13). counts strictly increasing. */
rs_status rs_knee_threshold(const double* counts, const double* tput, int32_t n, double frac,
                            int32_t* threshold);
/* Greedy plan for Eq. 6: transfers (src[i], dst[i], count[i]), i < *n_transfers
 * (arrays of capacity G). Every instance appears in at most one transfer. */
rs_status rs_plan_reallocation(const int32_t* loads, int32_t G, int32_t threshold, int32_t* src,
                               int32_t* dst, int32_t* count, int32_t* n_transfers);
/* The reallocation trigger: *trigger = 1 iff steps_since_last >= cooldown and some
 * instance's load is below threshold while another's is above it (loads: host int32 [G]). */
rs_status rs_realloc_should_trigger(const int32_t* loads, int32_t G, int32_t threshold, int32_t steps_since_last,
                                    int32_t cooldown, int32_t* trigger);
/* Samples to move: shortest sequence first, then lowest average accepted tokens, then gid. */
rs_status rs_choose_samples(const int64_t* gid, const int32_t* seq_len, const double* avg_accepted,
                            int32_t n, int32_t k, int64_t* chosen);

/* ===================================================================================== a5
 * KV migration: pack into one contiguous buffer ordered model -> layer -> sample
 * (Z18: per segment K then V, each [Hkv][len][head_dim]), transfer, unpack. */
/* Elements (bf16) of one model's part of the buffer: L * 2 * Hkv * head_dim * sum(lens). */
int64_t rs_kv_pack_elems(int32_t L, int32_t Hkv, int32_t head_dim, const int32_t* lens_host,
                         int32_t n);
/* Gather n samples (rows sample_rows[i] of block_table, lens[i] tokens) of one model into
 * buf + buf_offset_elems. sample_rows, lens: device int32 [n]. */
rs_status rs_kv_pack(void* const* k_layers_host, void* const* v_layers_host, int32_t L, int32_t Hkv,
                     int32_t head_dim, int32_t page_size, const int32_t* block_table,
                     int32_t max_pages, const int32_t* sample_rows, const int32_t* lens, int32_t n,
                     void* buf, int64_t buf_offset_elems, void* stream);
/* Inverse: scatter from the buffer into the pages of block_table rows sample_rows[i]. */
rs_status rs_kv_unpack(void* const* k_layers_host, void* const* v_layers_host, int32_t L,
                       int32_t Hkv, int32_t head_dim, int32_t page_size, const int32_t* block_table,
                       int32_t max_pages, const int32_t* sample_rows, const int32_t* lens,
                       int32_t n, const void* buf, int64_t buf_offset_elems, void* stream);
/* Token-range variants (f1): sample i contributes tokens starts[i] .. starts[i]+lens[i]-1
 * (starts device int32 [n]); the buffer layout is the one above with len = lens[i]. */
rs_status rs_kv_pack_range(void* const* k_layers_host, void* const* v_layers_host, int32_t L,
                           int32_t Hkv, int32_t head_dim, int32_t page_size, const int32_t* block_table,
                           int32_t max_pages, const int32_t* sample_rows, const int32_t* starts,
                           const int32_t* lens, int32_t n, void* buf, int64_t buf_offset_elems,
                           void* stream);
rs_status rs_kv_unpack_range(void* const* k_layers_host, void* const* v_layers_host, int32_t L,
                             int32_t Hkv, int32_t head_dim, int32_t page_size, const int32_t* block_table,
                             int32_t max_pages, const int32_t* sample_rows, const int32_t* starts,
                             const int32_t* lens, int32_t n, const void* buf, int64_t buf_offset_elems,
                             void* stream);

/* Host page allocator of one instance's paged KV store (same page ids in every layer/model).
 * Allocation is all-or-nothing: RS_ERR_NO_MEMORY and nothing reserved if too few pages are
 * free. Freeing a page that is not allocated is RS_ERR_INVALID_ARG. */
typedef struct rs_page_pool rs_page_pool;
rs_status rs_page_pool_create(int32_t num_pages, rs_page_pool** out);
void rs_page_pool_destroy(rs_page_pool* pool);
int32_t rs_page_pool_free_count(const rs_page_pool* pool);
rs_status rs_page_pool_alloc(rs_page_pool* pool, int32_t n, int32_t* pages_out);
rs_status rs_page_pool_free(rs_page_pool* pool, const int32_t* pages, int32_t n);
/* Destination side of the handshake: reserve ceil(lens[i]/page_size) pages per sample
 * (all-or-nothing) and write host block-table rows [n, max_pages] (tail padded with the last
 * page). */
rs_status rs_migrate_reserve(rs_page_pool* pool, const int32_t* lens_host, int32_t n,
                             int32_t page_size, int32_t max_pages, int32_t* block_table_rows_out);

/* NCCL communicator between generation instances (one process per GPU). The unique id is
 * made on one rank and distributed by the caller (e.g. torch.distributed broadcast). */
typedef struct rs_comm rs_comm;
rs_status rs_comm_unique_id(uint8_t* id_out_128);
rs_status rs_comm_create(const uint8_t* id_128, int32_t rank, int32_t world, rs_comm** out);
rs_status rs_comm_destroy(rs_comm* comm);

/* One instance's KV store: per model (SSM then LLM; L_ssm may be 0) host arrays of per-layer
 * device page pools [pages, Hkv, page_size, head_dim] bf16. */
typedef struct {
    void* const* k_ssm;
    void* const* v_ssm;
    int32_t L_ssm, Hkv_ssm, d_ssm;
    void* const* k_llm;
    void* const* v_llm;
    int32_t L_llm, Hkv_llm, d_llm;
    int32_t page_size;
} rs_kv_desc;

/* Move n samples from src_rank to dst_rank, called collectively by both ranks
 * (other ranks return at once). src: gids_host/lens_host [n], src_block_table device int32
 * [n, max_pages] (row i = sample i). dst: pool reserves the pages; dst_block_table_host
 * [n, max_pages] receives the new rows. Both: staging device buffer >= 2*(elems SSM + LLM)
 * bytes; device_scratch device int32 >= 2n + n*max_pages. Blocking (returns after the
 * stream is synchronised). On refusal both ranks return RS_ERR_NO_MEMORY and the source
 * keeps its samples (nothing was sent). */
rs_status rs_migrate_samples(rs_comm* comm, int32_t src_rank, int32_t dst_rank,
                             const rs_kv_desc* kv, rs_page_pool* pool, const int64_t* gids_host,
                             const int32_t* lens_host, int32_t n, const int32_t* src_block_table,
                             int32_t max_pages, int32_t* dst_block_table_host, void* staging,
                             size_t staging_bytes, int32_t* device_scratch, void* stream);

/* ===================================================================================== f1
 * Two-stage sample migration. Both ranks of the pair call each
 * stage with identical n (other ranks return at once); arguments marked src / dst are read on
 * that side only. Each stage starts with a small blocking handshake (request, all-or-nothing
 * page reservation on the destination, answer; refusal -> RS_ERR_NO_MEMORY on both ranks and
 * nothing is sent), then ENQUEUES pack -> NCCL send/recv -> unpack on `stream` and
 * returns without waiting: staging, device_scratch and the host block-table rows must stay
 * valid until `stream` has passed this work.
 *
 * Stage 1 — the verified prefix, while both instances keep computing on other streams (later
 * verification steps write only slots >= lens[i], the Markov property of verification):
 *   src: gids_host, lens_host [n] (tokens verified at the trigger), reserve_lens_host [n]
 *        (>= lens: tokens the destination reserves pages for), src_block_table device [n, max_pages]
 *   dst: pool, dst_block_table_host [n, max_pages] out (reserved rows)
 *   staging >= 2 * rs_kv_pack_elems(all models, lens) bytes; device_scratch int32 >= 2n + n*max_pages.
 * Stage 2 — the tokens verified on the source since stage 1 (the sample is paused on the
 * source from the call): tokens starts[i] .. starts[i]+lens[i]-1. The SSM part is sent and
 * unpacked first and `ssm_ready_event` (cudaEvent_t, may be NULL) is recorded on the
 * destination's `stream` once it has landed — drafting may resume there — then the
 * LLM part follows; the samples may be verified on the destination after `stream` completes.
 *   src: starts_host, lens_host [n], src_block_table
 *   dst: pool; dst_block_table_host (in: stage-1 rows, out: extended when a sample outgrew its
 *        reservation); dst_capacity_host int32 [n] (in/out: tokens the row's pages hold)
 *   device_scratch int32 >= 3n + n*max_pages. */
rs_status rs_migrate_stage1(rs_comm* comm, int32_t src_rank, int32_t dst_rank, const rs_kv_desc* kv,
                            rs_page_pool* pool, const int64_t* gids_host, const int32_t* lens_host,
                            const int32_t* reserve_lens_host, int32_t n, const int32_t* src_block_table,
                            int32_t max_pages, int32_t* dst_block_table_host, void* staging,
                            size_t staging_bytes, int32_t* device_scratch, void* stream);
rs_status rs_migrate_stage2(rs_comm* comm, int32_t src_rank, int32_t dst_rank, const rs_kv_desc* kv,
                            rs_page_pool* pool, const int32_t* starts_host, const int32_t* lens_host,
                            int32_t n, const int32_t* src_block_table, int32_t max_pages,
                            int32_t* dst_block_table_host, int32_t* dst_capacity_host, void* staging,
                            size_t staging_bytes, int32_t* device_scratch, void* ssm_ready_event,
                            void* stream);

/* ===================================================================================== a5 (peer memory)
 * KV migration over peer memory (P:302-327 on B200): the instances' KV stores are registered
 * once (rs_peer_create on each rank, the host blob of rs_peer_export sent to every other rank
 * over the caller's control plane, rs_peer_import there: CUDA IPC mappings of the peer's page
 * pools, NVLink P2P when the instances are on different GPUs). A migration is then ONE kernel
 * on the source: every (page, kv head) run of the samples' token range is read from the local
 * pools and stored straight into the destination's reserved pages — pack, transfer and unpack
 * of P:321-327 in one pass, with no staging buffer. The allocation handshake of P:325 is the
 * caller's: the destination reserves pages (rs_migrate_reserve, all-or-nothing; refusal ->
 * nothing is pushed and the source keeps its samples) and sends its block-table rows back.
 * Completion: the source records its inter-process event after the push (rs_peer_signal), tells
 * the destination over the control plane, and the destination's stream waits on it
 * (rs_peer_wait) before anything reads the new pages. The pools must outlive the rs_peer objects
 * of every rank that imported them. */
typedef struct rs_peer rs_peer;
/* Register this rank's store (pointers kept until rs_peer_destroy; 16-byte aligned pools). */
rs_status rs_peer_create(const rs_kv_desc* kv, int32_t rank, rs_peer** out);
/* Size of the registration blob (host bytes): header + one IPC handle / offset per layer pool. */
size_t rs_peer_blob_bytes(const rs_peer* peer);
rs_status rs_peer_export(const rs_peer* peer, uint8_t* blob, size_t bytes);
/* Map the store of the rank named in `blob` (same KV shapes, else RS_ERR_LAYOUT_MISMATCH; a
 * blob from this process is used by raw pointer). Each rank may be imported once. */
rs_status rs_peer_import(rs_peer* peer, const uint8_t* blob, size_t bytes);
/* Source side: copy tokens starts[i] .. starts[i]+lens[i]-1 (starts NULL = from 0) of sample i
 * from this rank's pages (row i of src_block_table) into dst_rank's pages (row i of
 * dst_block_table, the rows the destination reserved), every layer of the models selected by
 * `parts` (bit 0 = SSM, bit 1 = LLM; SSM launched first). src/dst block tables: device int32
 * [n, max_pages]; starts, lens: device int32 [n]. Enqueued on `stream`. Device data is not
 * validated (the kernel trusts it, like the attention kernel trusts its block table): the caller
 * guarantees starts[i] + lens[i] <= max_pages * page_size and page ids inside both pools. */
rs_status rs_peer_push(rs_peer* peer, int32_t dst_rank, const int32_t* src_block_table,
                       const int32_t* dst_block_table, int32_t max_pages, const int32_t* starts,
                       const int32_t* lens, int32_t n, int32_t parts, void* stream);
/* Record this rank's event `which` (0 = push done, 1 = SSM part landed) on `stream`. */
rs_status rs_peer_signal(rs_peer* peer, int32_t which, void* stream);
/* Make `stream` wait for src_rank's most recent rs_peer_signal(which) — call it only after the
 * source has told you (control plane) that the signal is enqueued. */
rs_status rs_peer_wait(rs_peer* peer, int32_t src_rank, int32_t which, void* stream);
void rs_peer_destroy(rs_peer* peer);

#ifdef __cplusplus
}
#endif
#endif /* RLHFSPEC_CORE_H */
