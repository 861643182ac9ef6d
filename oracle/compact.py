"""Oracle: post-verification KV commit of the accepted path (test infrastructure only).

Paper: "each step of the LLM verification only targets the newly generated speculative
tokens ... only the KVCache generated in this step will be updated after verification,
leaving the KVCache verified by previous steps unchanged" (Markov property). The
verify pass wrote node i's K/V at logical slot P_b + i; after acceptance the committed
sequence is root, path[1], ..., path[a]. Reading (Z2): RoPE is applied upstream at
position P_b + depth(i) = P_b + k for path[k], so committing is a plain byte move:

    for k = 1 .. a_b (ascending):  K/V[b, slot P_b + k] <- K/V[b, slot P_b + path[k]]
    new_len[b] = P_b + 1 + a_b

applied to every layer and every kv head. Sequential ascending-k copies ARE the definition.
"""
from __future__ import annotations

import numpy as np

MAX_TREE = 64


def kv_compact(caches, block_table, prefix_len, accepted_len, path, page_size):
    """caches: list of arrays [num_pages, Hkv, page_size, d] (modified in place; any dtype).
    Returns (new_len[B], moves[B, 64, 2]) with moves[b, k-1] = (src_slot, dst_slot), -1 padded."""
    B = len(prefix_len)
    new_len = np.zeros(B, dtype=np.int32)
    moves = np.full((B, MAX_TREE, 2), -1, dtype=np.int32)
    for b in range(B):
        P = int(prefix_len[b])
        a = int(accepted_len[b])
        for k in range(1, a + 1):
            src = P + int(path[b, k])
            dst = P + k
            moves[b, k - 1] = (src, dst)
            sp, so = block_table[b, src // page_size], src % page_size
            dp, do = block_table[b, dst // page_size], dst % page_size
            for cache in caches:
                cache[dp, :, do, :] = cache[sp, :, so, :]
        new_len[b] = P + 1 + a
    return new_len, moves
