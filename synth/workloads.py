"""Seeded synthetic workloads for the batched tree-verification step.

Recipe:
  * prefix lengths: fixed, or LogNormal(ln median, sigma) clipped (long tail, Fig. 2 quantiles);
  * draft trees: BFS-ordered random trees (parent[i] < i), per-depth branching limits,
    T nodes including the root (node 0 = last committed token);
  * Q/K/V: N(0,1) rounded to bf16 (optionally q scaled);
  * paged KV: page_size-token pages, page ids drawn as a random permutation of the pool;
  * greedy logits: N(0,1) noise plus a +12 spike either on one child's token (prob p_accept)
    or on a non-child token;
  * sampling logits: draft q_c = softmax(3 N(0,1)); children i.i.d. from q_c (MSS) or the
    top-K of q_c (DELTA); target logits = log q_c + N(0, sigma^2).

Nothing here implements the method (no attention, acceptance rule, dl products, compaction).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np
import torch

__all__ = [
    "VerifyConfig", "CONFIGS", "TINY_PARENT", "random_tree_parents", "draw_prefix_lengths",
    "make_verify_batch", "make_candidate_tree", "lmsys_response_lengths", "planted_targets",
    "make_lm_head_inputs", "make_lm_head_sampling_inputs",
]

# Tiny config tree: paths [0,1,3,6], [0,1,4,7], [0,2,5].
TINY_PARENT = [-1, 0, 0, 1, 1, 2, 3, 4]


@dataclasses.dataclass
class VerifyConfig:
    name: str
    B: int
    Hq: int
    Hkv: int
    d: int
    V: int
    L: int
    page_size: int = 64
    prefix: tuple = ("fixed", 1024)          # ("fixed", P) | ("lognormal", median, sigma, lo, hi)
    tree: tuple = ("fixed", 16)              # ("fixed", T) | ("range", lo, hi) | ("tiny",) | ("strategy", n_cand)
    mode: str = "greedy"                     # greedy | delta | mss
    p_accept: float = 0.8                    # greedy: probability a node's argmax is a child's token
    temperature: float = 1.0
    q_scale: float = 1.0
    target_noise: float = 1.0                # sampling: sigma of target-vs-draft logit noise
    draft_dtype: str = "f32"                 # MSS draft probabilities: "f32" | "bf16" (the SSM's dtype)
    seed: int = 0

    @property
    def g(self) -> int:
        return self.Hq // self.Hkv


CONFIGS = {
    # BASELINE.json configs[0]
    "tiny": VerifyConfig("tiny", B=1, Hq=1, Hkv=1, d=64, V=1000, L=1, prefix=("fixed", 32),
                         tree=("tiny",), mode="greedy"),
    # configs[1]: Llama-3-8B shapes, batch 64, prefix 1K, 16-node tree, greedy
    "c2": VerifyConfig("c2", B=64, Hq=32, Hkv=8, d=128, V=128256, L=32, prefix=("fixed", 1024),
                       tree=("fixed", 16), mode="greedy"),
    # configs[2]: long-tail batch 256, prefixes 512-16K heavy tailed, trees 4-64, sampling
    "c3": VerifyConfig("c3", B=256, Hq=32, Hkv=8, d=128, V=128256, L=32,
                       prefix=("lognormal", 2048, 0.784, 512, 16384), tree=("range", 4, 64),
                       mode="mss"),
    # configs[4] per-GPU shard at G=8: 70B shapes, 128/8 samples, prefix 8K, 64-node trees
    # configs[2] as the method runs it: every sample's verification tree is its S(n) for the ONE n
    # select_strategy picks for the batch (Z20), from a candidate draft tree of n_cand nodes
    # (trees given to make_verify_batch by the caller, which runs the selector)
    "c3s": VerifyConfig("c3s", B=256, Hq=32, Hkv=8, d=128, V=128256, L=32,
                        prefix=("lognormal", 2048, 0.784, 512, 16384), tree=("strategy", 96),
                        mode="mss", draft_dtype="bf16"),
    "c5g8": VerifyConfig("c5g8", B=16, Hq=64, Hkv=8, d=128, V=128256, L=80, prefix=("fixed", 8192),
                         tree=("fixed", 64), mode="greedy"),
}


def random_tree_parents(rng: np.random.Generator, T: int, branching=(4, 3, 2, 2, 1),
                        p_skip: float = 0.25) -> np.ndarray:
    """BFS-ordered random tree with T nodes (node 0 = root, parent[0] = -1, parent[i] < i).

    Children attach to the current frontier node until its per-depth branching limit is
    reached (or a random skip), then the frontier advances — the parent array is
    non-decreasing, i.e. nodes are in BFS order.
    """
    parent = np.full(T, -1, dtype=np.int32)
    depth = np.zeros(T, dtype=np.int32)
    nchild = np.zeros(T, dtype=np.int32)
    cur = 0
    for i in range(1, T):
        while True:
            lim = branching[min(depth[cur], len(branching) - 1)]
            full = nchild[cur] >= lim
            skip = nchild[cur] > 0 and cur + 1 < i and rng.random() < p_skip
            if (full or skip) and cur + 1 < i:
                cur += 1
                continue
            break
        parent[i] = cur
        depth[i] = depth[cur] + 1
        nchild[cur] += 1
    return parent


def draw_prefix_lengths(rng: np.random.Generator, cfg: VerifyConfig) -> np.ndarray:
    kind = cfg.prefix[0]
    if kind == "fixed":
        return np.full(cfg.B, int(cfg.prefix[1]), dtype=np.int32)
    if kind == "lognormal":
        _, median, sigma, lo, hi = cfg.prefix
        x = rng.lognormal(mean=math.log(median), sigma=sigma, size=cfg.B)
        return np.clip(np.rint(x), lo, hi).astype(np.int32)
    if kind == "list":
        return np.asarray(cfg.prefix[1], dtype=np.int32)
    raise ValueError(kind)


def lmsys_response_lengths(rng: np.random.Generator, n: int, cap: int = 2048) -> np.ndarray:
    """Response lengths shaped like LMSYS-Chat-1M (median 378, p95 1373), capped."""
    mu = math.log(378.0)
    sigma = math.log(1373.0 / 378.0) / 1.6448536269514722
    return np.clip(np.rint(rng.lognormal(mu, sigma, size=n)), 1, cap).astype(np.int32)


def _tree_sizes(rng, cfg: VerifyConfig) -> np.ndarray:
    kind = cfg.tree[0]
    if kind == "tiny":
        return np.full(cfg.B, len(TINY_PARENT), dtype=np.int32)
    if kind == "fixed":
        return np.full(cfg.B, int(cfg.tree[1]), dtype=np.int32)
    if kind == "range":
        return rng.integers(cfg.tree[1], cfg.tree[2] + 1, size=cfg.B).astype(np.int32)
    if kind == "list":
        return np.asarray(cfg.tree[1], dtype=np.int32)
    raise ValueError(kind)


def _children_lists(parent: np.ndarray):
    ch = [[] for _ in range(len(parent))]
    for i in range(1, len(parent)):
        ch[parent[i]].append(i)
    return ch


def make_verify_batch(cfg: VerifyConfig, device="cpu", gen_device: Optional[str] = None,
                      layers: Optional[int] = None, spare_pages: int = 0,
                      with_logits: bool = True, parents: Optional[list] = None) -> dict:
    """Draw one verify-step batch. All tensors live on `device`; large random tensors are
    drawn with a torch generator on `gen_device` (default: `device`) seeded by cfg.seed."""
    rng = np.random.default_rng(cfg.seed)
    gen_device = gen_device or device
    gen = torch.Generator(device=gen_device)
    gen.manual_seed(cfg.seed + 12345)
    L = cfg.L if layers is None else layers
    B, Hq, Hkv, d, ps, V = cfg.B, cfg.Hq, cfg.Hkv, cfg.d, cfg.page_size, cfg.V

    P = draw_prefix_lengths(rng, cfg)
    if parents is not None:      # verification trees given by the caller (e.g. from select_strategy)
        parents = [np.asarray(x, dtype=np.int32) for x in parents]
        Tn = np.array([len(x) for x in parents], dtype=np.int32)
    else:
        Tn = _tree_sizes(rng, cfg)
    tree_off = np.zeros(B + 1, dtype=np.int32)
    tree_off[1:] = np.cumsum(Tn)
    NT = int(tree_off[-1])
    given = parents is not None
    parents = parents if given else []
    for b in range(B if not given else 0):
        if cfg.tree[0] == "tiny":
            parents.append(np.asarray(TINY_PARENT, dtype=np.int32))
        else:
            parents.append(random_tree_parents(rng, int(Tn[b])))
    parent = np.concatenate(parents).astype(np.int32)

    # node tokens: siblings distinct (greedy / delta); MSS overwrites with i.i.d. draws below
    token = np.zeros(NT, dtype=np.int32)
    for b in range(B):
        off = tree_off[b]
        ch = _children_lists(parents[b])
        token[off] = rng.integers(V)
        for c, kids in enumerate(ch):
            if kids:
                toks = rng.choice(V, size=len(kids), replace=False)
                token[off + np.asarray(kids)] = toks

    # paged KV cache: pages for slots [0, P_b + T_b)
    npg = (P + Tn + ps - 1) // ps
    max_pages = int(npg.max())
    num_pages = int(npg.sum()) + spare_pages
    perm = rng.permutation(num_pages).astype(np.int32)
    block_table = np.zeros((B, max_pages), dtype=np.int32)
    o = 0
    for b in range(B):
        block_table[b, :npg[b]] = perm[o:o + npg[b]]
        block_table[b, npg[b]:] = perm[o + npg[b] - 1]   # padding repeats a valid page (never read)
        o += npg[b]

    gid = (np.arange(B, dtype=np.int64) * 7919 + 1000003 * (cfg.seed + 1))

    out = dict(cfg=cfg, B=B, Hq=Hq, Hkv=Hkv, d=d, page_size=ps, V=V, L=L, NT=NT,
               prefix_len=P, T=Tn, tree_off=tree_off, parent=parent, token=token,
               block_table=block_table, max_pages=max_pages, num_pages=num_pages, gid=gid,
               sm_scale=1.0 / math.sqrt(d))

    def randn(shape):
        return torch.randn(shape, generator=gen, device=gen_device, dtype=torch.float32)

    kv_shape = (L, num_pages, Hkv, ps, d)
    k = torch.empty(kv_shape, dtype=torch.bfloat16, device=device)
    v = torch.empty(kv_shape, dtype=torch.bfloat16, device=device)
    for l in range(L):   # per layer to bound the fp32 temporary
        k[l].copy_(randn(kv_shape[1:]).to(torch.bfloat16))
        v[l].copy_(randn(kv_shape[1:]).to(torch.bfloat16))
    q = torch.empty((L, NT, Hq, d), dtype=torch.bfloat16, device=device)
    for l in range(L):
        q[l].copy_((randn((NT, Hq, d)) * cfg.q_scale).to(torch.bfloat16))
    out.update(k_cache=k, v_cache=v, q=q)

    if with_logits:
        out.update(_make_logits(cfg, rng, gen, gen_device, device, parents, tree_off, token, NT, V))
    return out


def _make_logits(cfg, rng, gen, gen_device, device, parents, tree_off, token, NT, V):
    res = {}
    if cfg.mode == "greedy":
        noise = torch.randn((NT, V), generator=gen, device=gen_device, dtype=torch.float32)
        spike_tok = np.zeros(NT, dtype=np.int64)
        for b in range(cfg.B):
            off = int(tree_off[b])
            ch = _children_lists(parents[b])
            for c, kids in enumerate(ch):
                kid_toks = set(int(token[off + x]) for x in kids)
                if kids and rng.random() < cfg.p_accept:
                    spike_tok[off + c] = token[off + kids[rng.integers(len(kids))]]
                else:
                    t = int(rng.integers(V))
                    while t in kid_toks:
                        t = int(rng.integers(V))
                    spike_tok[off + c] = t
        st = torch.from_numpy(spike_tok).to(gen_device)
        noise[torch.arange(NT, device=gen_device), st] += 12.0
        res["logits"] = noise.to(torch.bfloat16).to(device)
        res["draft_probs"] = None
    else:
        # draft distribution q_c per row (the SSM's output at node c)
        z = torch.randn((NT, V), generator=gen, device=gen_device, dtype=torch.float32) * 3.0
        q = torch.softmax(z, dim=-1)
        if cfg.mode == "mss" and cfg.draft_dtype == "bf16":
            q = q.to(torch.bfloat16).float()   # the distribution the children are drawn from and tested with
        tok = torch.from_numpy(token.astype(np.int64)).to(gen_device)
        for b in range(cfg.B):
            off = int(tree_off[b])
            ch = _children_lists(parents[b])
            for c, kids in enumerate(ch):
                if not kids:
                    continue
                if cfg.mode == "mss":   # children i.i.d. from q_c, in node-index order
                    draws = torch.multinomial(q[off + c], len(kids), replacement=True, generator=gen)
                else:                   # delta: deterministic top-K of q_c
                    draws = torch.topk(q[off + c], len(kids)).indices
                tok[off + torch.as_tensor(kids, device=gen_device)] = draws
        token[:] = tok.cpu().numpy().astype(np.int32)
        target = torch.log(q) + cfg.target_noise * torch.randn(
            (NT, V), generator=gen, device=gen_device, dtype=torch.float32)
        res["logits"] = target.to(torch.bfloat16).to(device)
        if cfg.mode == "mss":
            res["draft_probs"] = (q.to(torch.bfloat16) if cfg.draft_dtype == "bf16" else q).to(device)
        else:
            res["draft_probs"] = None
    return res


def make_candidate_tree(rng: np.random.Generator, n_nodes: int, branching=(4, 3, 2, 2, 1),
                        beta=(4.0, 2.0), decay: float = 0.9):
    """Draft candidate tree for select_strategy (SPEC S:304 shape): BFS parents over draft
    tokens (index 0 = first draft token under the implicit committed root; parent -1 means
    "child of the committed root") and per-node SSM probabilities o(v) ~ Beta * decay^depth.
    Returns (parent, o) with parent[i] < i."""
    # root-level nodes are children of the virtual root: build a tree with a virtual node 0
    par = random_tree_parents(rng, n_nodes + 1, branching=branching)
    parent = par[1:] - 1                      # virtual root (0) -> -1
    depth = np.zeros(n_nodes, dtype=np.int32)
    for i in range(n_nodes):
        depth[i] = 0 if parent[i] < 0 else depth[parent[i]] + 1
    o = rng.beta(beta[0], beta[1], size=n_nodes) * (decay ** depth)
    o = np.clip(o, 1e-6, 1.0)
    return parent.astype(np.int32), o.astype(np.float64)


def planted_targets(rng: np.random.Generator, parent: np.ndarray, tree_off: np.ndarray, token: np.ndarray,
                    V: int, p_accept: float) -> np.ndarray:
    """Per tree node, the token the target model is made to prefer: with probability p_accept
    one child's token (so the greedy walk can advance), else a token no child carries."""
    NT = int(tree_off[-1])
    tgt = np.zeros(NT, dtype=np.int64)
    for b in range(len(tree_off) - 1):
        off = int(tree_off[b])
        ch = _children_lists(np.asarray(parent[off:int(tree_off[b + 1])]))
        for c, kids in enumerate(ch):
            kid_toks = set(int(token[off + x]) for x in kids)
            if kids and rng.random() < p_accept:
                tgt[off + c] = token[off + kids[rng.integers(len(kids))]]
            else:
                t = int(rng.integers(V))
                while t in kid_toks:
                    t = int(rng.integers(V))
                tgt[off + c] = t
    return tgt


def make_lm_head_inputs(batch: dict, Dm: int, seed: int = 7, device="cpu", gen_device: Optional[str] = None,
                        p_accept: Optional[float] = None, plant: float = 0.1, noise: float = 0.25) -> dict:
    """Final hidden states [NT, Dm] and an LM-head weight [V, Dm] (bf16) for the tree nodes of
    `batch`. W ~ N(0, 1); hidden[r] = plant * W[tgt_r] + noise * N(0, 1), so
    the target's preferred token at node r is tgt_r (planted_targets) by a wide margin
    (plant*Dm against a noise sd of ~noise*sqrt(Dm)). The planted token is an input property
    used to steer acceptance; tests never take it as the expected arg-max."""
    cfg = batch["cfg"]
    rng = np.random.default_rng(seed)
    gen_device = gen_device or device
    gen = torch.Generator(device=gen_device)
    gen.manual_seed(seed + 777)
    V, NT = batch["V"], batch["NT"]
    pa = cfg.p_accept if p_accept is None else p_accept
    tgt = planted_targets(rng, batch["parent"], batch["tree_off"], batch["token"], V, pa)
    w = torch.empty((V, Dm), dtype=torch.bfloat16, device=device)
    step = 8192
    for v0 in range(0, V, step):      # bounded fp32 temporaries
        v1 = min(V, v0 + step)
        w[v0:v1].copy_(torch.randn((v1 - v0, Dm), generator=gen, device=gen_device).to(torch.bfloat16))
    t = torch.from_numpy(tgt).to(w.device)
    h = plant * w[t].float() + noise * torch.randn((NT, Dm), generator=gen, device=gen_device).to(w.device)
    return dict(hidden=h.to(torch.bfloat16), weight=w, planted=tgt, Dm=Dm)


def make_lm_head_sampling_inputs(batch: dict, Dm: int, seed: int = 7, device="cpu", gen_device: Optional[str] = None,
                                 hidden_sd: float = 0.05, draft_noise: float = 1.0,
                                 draft_dtype: Optional[str] = None) -> dict:
    """f2 for the sampling modes: final hidden states [NT, Dm] ~ N(0, hidden_sd) and an LM-head
    weight [V, Dm] ~ N(0, 1) (bf16), so the target logits H W^T have sd ~ hidden_sd * sqrt(Dm)
    (3.2 at Dm = 4096, the spread of the default recipe's log q + N(0, 1)); the draft
    distribution of node c is q_c = softmax(target logits of c + draft_noise * N(0, 1)) (the
    reverse of the default recipe: the draft is a noisy target) and the children of c are drawn
    i.i.d. from q_c. Returns hidden, weight, draft_probs [NT, V] and the node tokens (root tokens
    kept). The target logits here are the generator's own fp32 GEMM, an input property only."""
    cfg = batch["cfg"]
    gen_device = gen_device or device
    gen = torch.Generator(device=gen_device)
    gen.manual_seed(seed + 991)
    V, NT = batch["V"], batch["NT"]
    w = torch.empty((V, Dm), dtype=torch.bfloat16, device=device)
    step = 8192
    for v0 in range(0, V, step):
        v1 = min(V, v0 + step)
        w[v0:v1].copy_(torch.randn((v1 - v0, Dm), generator=gen, device=gen_device).to(torch.bfloat16))
    h = (hidden_sd * torch.randn((NT, Dm), generator=gen, device=gen_device)).to(torch.bfloat16).to(device)
    ddt = draft_dtype or cfg.draft_dtype
    q = torch.empty((NT, V), dtype=torch.bfloat16 if ddt == "bf16" else torch.float32, device=device)
    tok = np.array(batch["token"], dtype=np.int32, copy=True)
    par, off = np.asarray(batch["parent"]), np.asarray(batch["tree_off"])
    rows_per = 256
    wf = w.float()
    for r0 in range(0, NT, rows_per):   # bounded fp32 temporaries
        r1 = min(NT, r0 + rows_per)
        lg = h[r0:r1].float() @ wf.T
        z = lg + draft_noise * torch.randn(lg.shape, generator=gen, device=gen_device).to(lg.device)
        q[r0:r1].copy_(torch.softmax(z, dim=-1).to(q.dtype))
    # children of c drawn i.i.d. from q_c (as the drafted tokens are), one multinomial per parent row
    kids_of = {}
    for s_ in range(batch["B"]):
        o = int(off[s_])
        for i in range(1, int(off[s_ + 1]) - o):
            kids_of.setdefault(o + int(par[o + i]), []).append(o + i)
    if kids_of:
        prow = torch.as_tensor(sorted(kids_of), device=q.device)
        pq = q.index_select(0, prow).float()
        nk = max(len(v) for v in kids_of.values())
        draws = torch.multinomial(pq.to(gen_device), nk, replacement=True, generator=gen).cpu().numpy()
        for j, c in enumerate(sorted(kids_of)):
            for k, x in enumerate(kids_of[c]):
                tok[x] = int(draws[j, k])
    return dict(hidden=h, weight=w, draft_probs=q, token=tok, Dm=Dm)
