"""Oracle: workload-aware drafting-strategy selection (test infrastructure only).

Follows PAPER.md section 5 step by step:
  * draft logit dl(u) = prod_{v in Path(root,u)} o(v)
    reading Z9: the product includes u itself (the Fig. 1 sentence "dl(u6) = o(u0) x o(u2)"
    contradicts the definition; the definition wins);
  * node weight w(u) = F(dl(u)), F a monotone piecewise-linear acceptance fit
  * al(n) = sum_{u in S(n)} w(u)
  * t_sd(n) from a regression on N_seq (KVCache loading) and N_draft (FFN), plus a
    constant draft cost, behind a bucket cache
  * layer-level search: on reaching layer m push that layer's nodes into a max priority
    queue and pop u_max to form S(m) = S(m-1) U {u_max}
  * objective al(n)/t_sd(n) (Eq. 2); early stop after a continuous decrease
    (Eq. 3) — reading Z12: `patience` consecutive strict decreases.
Batch reading: one shared n per batch; every sample pops its own u_max per n,
so al sums over samples and N_draft = B * (n + 1) verified tokens (root included, Z1).
"""
from __future__ import annotations

import heapq

import numpy as np


def draft_logits(parent, o):
    """dl per node; parent[i] = -1 means child of the (virtual) committed root; parent[i] < i."""
    dl = np.zeros(len(parent))
    for i in range(len(parent)):
        dl[i] = o[i] * (1.0 if parent[i] < 0 else dl[parent[i]])
    return dl


def cand_depths(parent):
    dep = np.zeros(len(parent), dtype=np.int64)
    for i in range(len(parent)):
        dep[i] = 0 if parent[i] < 0 else dep[parent[i]] + 1
    return dep


def acceptance_fit(knots_x, knots_y, x):
    """F: piecewise-linear through (knots_x, knots_y), constant outside, clipped to [0, 1]."""
    return float(np.clip(np.interp(x, knots_x, knots_y), 0.0, 1.0))


def layer_search_order(parent, weights, n_max):
    """Sequence of u_max popped by the layer-level search: at step m push the nodes of
    layer m (depth m-1) and pop the max (ties: lower depth, then lower id). Returns the popped
    node list (length <= n_max); S(n) = first n entries."""
    dep = cand_depths(parent)
    pq = []
    order = []
    for m in range(1, n_max + 1):
        for u in np.nonzero(dep == m - 1)[0]:
            heapq.heappush(pq, (-weights[u], int(dep[u]), int(u)))
        if not pq:
            break
        order.append(heapq.heappop(pq)[2])
    return order


def fit_acceptance(dl, accepted, n_buckets=20):
    """F from (dl, accepted) observations ("we fit a function (i.e., F: X->Y) between draft
    logits and token acceptance probability based on offline profiling data"; SPEC S:128-131:
    "monotone piecewise-linear F minimizing squared error over bucketed empirical acceptance
    rates; isotonic-regression pass enforces monotonicity"). Reading Z24, step by step:
      1. bucket k = min(K-1, floor(dl*K)) over [0, 1] (dl clipped to [0, 1]), K = n_buckets;
      2. per non-empty bucket: x_k = mean dl, r_k = mean accepted, weight n_k = count
         (sums accumulated in observation order);
      3. pool-adjacent-violators over the buckets in ascending k with weights n_k (the
         weighted least-squares non-decreasing fit of r_k): a new block is appended, then while
         the previous block's value exceeds the last one's they merge into one block with value
         (sum of n*y) / (sum of n);
      4. knots (x_k, y_k), y_k = value of k's block; F interpolates them, constant outside.
    Returns (knots_x, knots_y). Raises ValueError("InsufficientData") with < 2 distinct dl."""
    dl = np.asarray(dl, dtype=np.float64)
    acc = np.asarray(accepted, dtype=np.float64)
    if len(dl) != len(acc) or len(np.unique(dl)) < 2:
        raise ValueError("InsufficientData")
    K = int(n_buckets)
    sx, sy, cnt = [0.0] * K, [0.0] * K, [0] * K
    for x, a in zip(dl, acc):
        xc = min(max(x, 0.0), 1.0)
        k = min(K - 1, int(np.floor(xc * K)))
        sx[k] += xc
        sy[k] += a
        cnt[k] += 1
    xs, rs, ws = [], [], []
    for k in range(K):
        if cnt[k]:
            xs.append(sx[k] / cnt[k])
            rs.append(sy[k] / cnt[k])
            ws.append(float(cnt[k]))
    # pool adjacent violators: blocks of (sum n*y, sum n, number of buckets)
    blocks = []
    for r, w in zip(rs, ws):
        blocks.append([r * w, w, 1])
        while len(blocks) > 1 and blocks[-2][0] / blocks[-2][1] > blocks[-1][0] / blocks[-1][1]:
            a = blocks.pop()
            blocks[-1][0] += a[0]
            blocks[-1][1] += a[1]
            blocks[-1][2] += a[2]
    ys = []
    for sy_, sw, m in blocks:
        ys.extend([sy_ / sw] * m)
    return np.array(xs), np.array(ys)


class CostModel:
    """t_sd = c_draft + b0 + b1*N_seq + b2*N_draft + b3*relu(N_draft - k_sat)*N_draft,
    evaluated at the lower corner of its (N_seq, N_draft) bucket (reading Z12)."""

    def __init__(self, c_draft, b0, b1, b2, b3, k_sat, seq_bucket=256, draft_bucket=4):
        self.c_draft, self.b0, self.b1, self.b2, self.b3, self.k_sat = c_draft, b0, b1, b2, b3, k_sat
        self.seq_bucket, self.draft_bucket = seq_bucket, draft_bucket

    def regression(self, n_seq, n_draft):
        return (self.c_draft + self.b0 + self.b1 * n_seq + self.b2 * n_draft
                + self.b3 * max(0.0, n_draft - self.k_sat) * n_draft)

    def t_sd(self, n_seq, n_draft):
        bs = (n_seq // self.seq_bucket) * self.seq_bucket
        bd = (n_draft // self.draft_bucket) * self.draft_bucket
        return self.regression(bs, bd)


def search_profile(al, t, n_min=1, patience=2):
    """The search loop on a given profile al[n-1], t[n-1] for n = 1..len(al): returns
    (argmax n, n at which the search stopped). Eq. 2 objective, Eq. 3 early stop."""
    best_n, best_obj, prev, dec, last = None, -np.inf, None, 0, None
    for n in range(1, len(al) + 1):
        last = n
        if n < n_min:
            continue
        obj = al[n - 1] / t[n - 1]
        if obj > best_obj:
            best_obj, best_n = obj, n
        if prev is not None and obj < prev:
            dec += 1
        else:
            dec = 0
        prev = obj
        if dec >= patience:
            break
    return best_n, last


def select_strategy(trees, prefix_len, knots_x, knots_y, cost: CostModel, n_min=2, n_max=48,
                    patience=2):
    """trees: per sample (parent, o) of candidate draft nodes. Returns a dict with the chosen n,
    the depth/width of the verification tree T = n + 1 (root at depth 0), predicted al, t_sd,
    objective and the evaluated profile."""
    B = len(trees)
    if B == 0:
        raise ValueError("EmptyTree")
    orders, weights, deps = [], [], []
    for parent, o in trees:
        if len(parent) == 0 or not np.any(np.asarray(parent) < 0):
            raise ValueError("EmptyTree")
        dl = draft_logits(parent, o)
        w = np.array([acceptance_fit(knots_x, knots_y, x) for x in dl])
        orders.append(layer_search_order(parent, w, n_max))
        weights.append(w)
        deps.append(cand_depths(parent))
    feasible = min(len(od) for od in orders)
    n_seq = int(np.sum(prefix_len))
    al_prof, t_prof = [], []
    al = 0.0
    for n in range(1, min(n_max, feasible) + 1):
        al += sum(weights[b][orders[b][n - 1]] for b in range(B))
        al_prof.append(al)
        t_prof.append(cost.t_sd(n_seq, B * (n + 1)))
    if not al_prof or len(al_prof) < n_min:
        raise ValueError("InsufficientNodes")
    n_best, n_stop = search_profile(al_prof, t_prof, n_min=n_min, patience=patience)
    depth, width = 0, 0
    for b in range(B):
        sel = orders[b][:n_best]
        d = deps[b][sel] + 1                 # verification-tree depth (root = 0)
        depth = max(depth, int(d.max()))
        width = max(width, int(np.bincount(d).max()))
    return dict(n=n_best, depth=depth, width=width, al=al_prof[n_best - 1], t_sd=t_prof[n_best - 1],
                objective=al_prof[n_best - 1] / t_prof[n_best - 1], n_stop=n_stop,
                al_profile=al_prof[:n_stop], t_profile=t_prof[:n_stop])


def verification_tree(parent, o, token, root_token, n, knots_x, knots_y):
    """The verification tree of one sample for a chosen n (the n selected draft nodes are
    verified in one pass as a tree under the last committed token): node 0 = root (token
    root_token), then S(n) (the first n nodes of the layer-level search) in ascending
    candidate index; a candidate whose parent is the virtual root (-1) hangs under node 0.
    S(n) is closed under parents (a node is popped only after its parent), so the result is
    topologically ordered. Returns (parent_v, token_v) int32 of length n + 1; raises
    ValueError("InsufficientNodes") when the search yields fewer than n nodes and
    ValueError("MalformedTree") when F's knots are not monotone (x strictly increasing, y
    non-decreasing), an o(u) is outside [0, 1], or S(n) is not closed under parents."""
    kx, ky = np.asarray(knots_x, float), np.asarray(knots_y, float)
    if not (np.all(np.isfinite(kx)) and np.all(np.isfinite(ky)) and np.all(np.diff(kx) > 0)
            and np.all(np.diff(ky) >= 0)):
        raise ValueError("MalformedTree")      # F must be monotone piecewise linear
    if not all(0.0 <= float(x) <= 1.0 for x in o):
        raise ValueError("MalformedTree")      # o(u) is a probability
    dl = draft_logits(parent, o)
    w = np.array([acceptance_fit(knots_x, knots_y, x) for x in dl])
    order = layer_search_order(parent, w, n)
    if len(order) < n:
        raise ValueError("InsufficientNodes")
    chosen = sorted(order)
    pos = {c: i + 1 for i, c in enumerate(chosen)}
    if any(parent[c] >= 0 and int(parent[c]) not in pos for c in chosen):
        raise ValueError("MalformedTree")      # S(n) not closed under parents
    par = [-1] + [0 if parent[c] < 0 else pos[int(parent[c])] for c in chosen]
    tok = [int(root_token)] + [int(token[c]) for c in chosen]
    return np.array(par, np.int32), np.array(tok, np.int32)
