"""Oracle: exact tree-verification attention in fp64 (test infrastructure only).

Definition (readings Z1-Z4, Z16). Tree-based verification runs
all tree tokens through the LLM "in a single decoding step"; attention's cost is
"KVCache loading" over the cumulative sequence lengths. For sample b, q-head h
(kv-head kappa = floor(h / g)), tree node i:

    A(b, i) = {0 .. P_b-1}  U  {P_b + j : j on Path(root, i)}           (prefix + ancestors-or-self)
    s_j     = (q[b,i,h] . k[b,j,kappa]) / sqrt(d)        for j in A(b, i)
    o       = sum_j exp(s_j - max s) v[b,j,kappa] / sum_j exp(s_j - max s)
    lse     = max s + log sum_j exp(s_j - max s)

Logical slot j of sample b lives at page block_table[b, j // page_size], row j % page_size,
of a cache laid out [num_pages, Hkv, page_size, d]. The tree mask is an input (bit j of
tree_mask[i] <=> slot P_b + j visible to node i), exactly as on the CUDA side.
"""
from __future__ import annotations

import numpy as np


def gather_slots(cache, block_table_row, n_slots, page_size):
    """[n_slots, Hkv, d] view of a sample's logical KV slots 0..n_slots-1."""
    s = np.arange(n_slots)
    return cache[block_table_row[s // page_size], :, s % page_size, :]


def allowed_matrix(P, T, mask_row_bits):
    """[T, P+T] boolean: key j visible to node i."""
    A = np.zeros((T, P + T), dtype=bool)
    A[:, :P] = True
    for i in range(T):
        bits = int(mask_row_bits[i])
        for j in range(T):
            if (bits >> j) & 1:
                A[i, P + j] = True
    return A


def tree_verify_attention(q, k_cache, v_cache, block_table, prefix_len, tree_off, tree_mask,
                          Hkv, page_size, sm_scale, samples=None):
    """q: [NT, Hq, d]; caches: [num_pages, Hkv, page_size, d] (any float dtype; computed in fp64).
    Returns (o [NT, Hq, d] fp64, lse [NT, Hq] fp64). `samples` restricts the computed samples
    (other rows are NaN)."""
    q = np.asarray(q, dtype=np.float64)
    NT, Hq, d = q.shape
    g = Hq // Hkv
    o = np.full((NT, Hq, d), np.nan)
    lse = np.full((NT, Hq), np.nan)
    B = len(prefix_len)
    for b in (range(B) if samples is None else samples):
        P = int(prefix_len[b])
        s0, s1 = int(tree_off[b]), int(tree_off[b + 1])
        T = s1 - s0
        K = gather_slots(k_cache, block_table[b], P + T, page_size).astype(np.float64)
        V = gather_slots(v_cache, block_table[b], P + T, page_size).astype(np.float64)
        A = allowed_matrix(P, T, tree_mask[s0:s1])
        qb = q[s0:s1].reshape(T, Hkv, g, d)
        # s[i, kappa, hh, j] = q[i, kappa*g+hh] . k[j, kappa] * scale
        s = np.einsum("ikhd,jkd->ikhj", qb, K) * sm_scale
        s = np.where(A[:, None, None, :], s, -np.inf)
        m = s.max(axis=-1, keepdims=True)
        p = np.exp(s - m)
        z = p.sum(axis=-1, keepdims=True)
        ob = np.einsum("ikhj,jkd->ikhd", p, V) / z
        o[s0:s1] = ob.reshape(T, Hq, d)
        lse[s0:s1] = (m[..., 0] + np.log(z[..., 0])).reshape(T, Hq)
    return o, lse
