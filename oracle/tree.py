"""Oracle: tree metadata (test infrastructure only; see oracle/__init__.py).

A speculative token tree ("multiple draft tokens are selected at each step to form a
tree, where each node represents a token and each branch represents a token sequence
awaiting verification"). Reading Z1/Z3: node 0 is the root (last committed
token), parent[i] < i, and node i attends to its ancestors-or-self.
"""
from __future__ import annotations

import numpy as np

MAX_TREE = 64


def validate(parent) -> bool:
    """True iff parent[] is a well-formed topologically ordered tree of 1..64 nodes."""
    T = len(parent)
    if T < 1 or T > MAX_TREE or parent[0] != -1:
        return False
    return all(0 <= parent[i] < i for i in range(1, T))


def ancestors_or_self(parent, i: int) -> list:
    """Nodes on Path(root, i), root first (P:80 'Path(root, u)')."""
    path = []
    i = int(i)
    while i >= 0:
        path.append(i)
        i = int(parent[i])
    return path[::-1]


def ancestor_mask(parent) -> np.ndarray:
    """uint64 per node: bit j set iff node j lies on Path(root, i) (ancestor-or-self)."""
    T = len(parent)
    m = np.zeros(T, dtype=np.uint64)
    for i in range(T):
        bits = 0
        for j in ancestors_or_self(parent, i):
            bits |= 1 << j
        m[i] = np.uint64(bits)
    return m


def depths(parent) -> np.ndarray:
    return np.array([len(ancestors_or_self(parent, i)) - 1 for i in range(len(parent))],
                    dtype=np.int32)


def batch_masks(parent_all, tree_off):
    """Per-sample masks for a flattened batch (local node indices in parent_all)."""
    B = len(tree_off) - 1
    masks = np.zeros(len(parent_all), dtype=np.uint64)
    dep = np.zeros(len(parent_all), dtype=np.int32)
    ok = np.zeros(B, dtype=bool)
    for b in range(B):
        s, e = tree_off[b], tree_off[b + 1]
        par = [int(x) for x in parent_all[s:e]]
        ok[b] = validate(par)
        if ok[b]:
            masks[s:e] = ancestor_mask(par)
            dep[s:e] = depths(par)
    return masks, dep, ok
