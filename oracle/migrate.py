"""Oracle: KV migration buffer layout, pack and unpack (test infrastructure only).

Paper, three-phase transmission: "(1) copying the KVCache from the KVCache store
into a buffer; (2) transferring ... ; (3) copying the KVCache from the buffer back to the
KVCache store", with the buffer organised hierarchically "according to the order of model
(SSM & LLM)-layer-sample" and pre-allocated contiguously so it moves "in a single copy
operation". Reading (Z18): within one (model, layer, sample) segment the
sample's K comes first, then its V, each laid out [Hkv][len][d] (head-major, token, dim).
"""
from __future__ import annotations

import numpy as np


def segment_table(models, lens):
    """models: list of (L, Hkv, d) in buffer order (SSM first, then LLM).
    lens: per-sample token counts in request order. Returns a list of
    (model, layer, sample, offset_elems, n_elems) with offsets in elements."""
    segs = []
    off = 0
    for mi, (L, Hkv, d) in enumerate(models):
        for l in range(L):
            for s, n in enumerate(lens):
                size = 2 * Hkv * int(n) * d
                segs.append((mi, l, s, off, size))
                off += size
    return segs, off


def pack(model_caches, block_tables, lens, page_size, starts=None):
    """model_caches: per model a list over layers of (K, V) arrays [pages, Hkv, ps, d].
    block_tables: per sample a page list (same page ids in every layer/model).
    starts: optional per-sample first token (default 0): the segment then holds tokens
    starts[s] .. starts[s]+lens[s]-1 — the two-stage migration sends the verified
    prefix first and the tokens verified meanwhile second, each in this same layout.
    Returns the 1-D buffer (dtype of the caches)."""
    parts = []
    for layers in model_caches:
        for (K, V) in layers:
            for s, n in enumerate(lens):
                t0 = 0 if starts is None else int(starts[s])
                slots = np.arange(t0, t0 + int(n))
                pages = np.asarray(block_tables[s])[slots // page_size]
                rows = slots % page_size
                for cache in (K, V):
                    seg = cache[pages, :, rows, :]          # [n, Hkv, d]
                    parts.append(np.transpose(seg, (1, 0, 2)).reshape(-1))   # [Hkv][n][d]
    if not parts:
        return np.zeros(0, dtype=np.uint16)
    return np.concatenate(parts)


def unpack(buf, model_caches, block_tables, lens, page_size, starts=None):
    """Inverse of pack into the destination caches (modified in place) using the
    destination's block tables."""
    off = 0
    for layers in model_caches:
        for (K, V) in layers:
            Hkv, d = K.shape[1], K.shape[3]
            for s, n in enumerate(lens):
                n = int(n)
                t0 = 0 if starts is None else int(starts[s])
                slots = np.arange(t0, t0 + n)
                pages = np.asarray(block_tables[s])[slots // page_size]
                rows = slots % page_size
                for cache in (K, V):
                    size = Hkv * n * d
                    seg = buf[off:off + size].reshape(Hkv, n, d)
                    cache[pages, :, rows, :] = np.transpose(seg, (1, 0, 2))
                    off += size
    return off
