"""Oracle (test infrastructure only; never imported by the product path): the LM head feeding
greedy tree acceptance, SURVEY §8(f) row f2.

Verification scores every tree node with the target model in one pass ("the LLM
verifies the n draft tokens ... in a single forward pass"); the greedy rule then walks the tree
from the root and accepts the child whose token is the target's arg-max at the current node
(SURVEY §8(c) c-2). Row f2 moves the arg-max in front of the logits: the vocabulary projection
logits[r, v] = sum_k hidden[r, k] * W[v, k] (P:213 names the LM head among the verification
GEMMs) is reduced to its per-row arg-max without materialising the [rows, V] logits.

What this module computes, written out plainly (fp64 as the task's oracle rule fixes):
  * lm_head_logits  — the definition: H @ W^T in float64 (numpy matmul as a library step).
  * argmax_rows     — arg-max per row, ties -> lowest vocabulary id (DESIGN Z6).
  * greedy_walk     — c-2's walk with the per-node arg-max given: from the root, move to the
                      lowest-index child whose token equals argmax[c]; stop when none does;
                      bonus = argmax at the last node.
Pins: tests/test_oracle_lm_head.py (brute-force dot products, planted arg-max, tie rule,
brute-force enumeration of root-to-leaf paths, equality with the C walk of oracle/accept_ref.c
on logits whose arg-max is planted).
"""
from __future__ import annotations

import numpy as np

MAX_TREE = 64


def lm_head_logits(hidden, weight):
    """hidden [R, Dm], weight [V, Dm] (any float dtype; bf16 callers pass float32/64 copies of
    the exact bf16 values) -> logits [R, V] float64."""
    h = np.asarray(hidden, dtype=np.float64)
    w = np.asarray(weight, dtype=np.float64)
    return h @ w.T


def argmax_rows(logits):
    """Per-row arg-max (np.argmax returns the first maximal index = lowest vocab id) and max. A
    row holding any non-finite logit has no arg-max: -1 and NaN (reading Z15: such a row stops
    the greedy walk with RS_FLAG_NONFINITE, whichever path computed the logits)."""
    lg = np.asarray(logits)
    idx = np.argmax(lg, axis=1).astype(np.int32)
    mx = lg[np.arange(lg.shape[0]), idx].astype(np.float64)
    bad = ~np.all(np.isfinite(lg), axis=1)
    idx[bad] = -1
    mx[bad] = np.nan
    return idx, mx


def lm_head_argmax(hidden, weight):
    return argmax_rows(lm_head_logits(hidden, weight))


def greedy_walk(argmax_tok, parent, token, tree_off):
    """c-2 walk given argmax_tok[node] (global node index). Returns accepted_len [B], path [B, 64]
    (node indices local to the sample, -1 padded) and bonus [B]."""
    tree_off = np.asarray(tree_off)
    B = len(tree_off) - 1
    acc = np.zeros(B, dtype=np.int32)
    path = np.full((B, MAX_TREE), -1, dtype=np.int32)
    bonus = np.zeros(B, dtype=np.int32)
    for b in range(B):
        s, e = int(tree_off[b]), int(tree_off[b + 1])
        c = 0
        path[b, 0] = 0
        n = 0
        while True:
            t = int(argmax_tok[s + c])
            nxt = -1
            for x in range(c + 1, e - s):            # children in ascending node index
                if int(parent[s + x]) == c and int(token[s + x]) == t:
                    nxt = x
                    break
            if nxt < 0:
                break
            c = nxt
            n += 1
            path[b, n] = c
        acc[b] = n
        bonus[b] = int(argmax_tok[s + c])
    return acc, path, bonus
