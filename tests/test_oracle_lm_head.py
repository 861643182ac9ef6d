"""Pins for oracle.lm_head: the LM-head arg-max and the greedy walk given the
per-node arg-max. Each pin is something other than the oracle's own formula: a projection
whose logits are known in closed form (permutation rows), ties by duplicated rows, the planted
margin of the synthetic generator, sign/scale invariances, brute-force enumeration of
root-to-leaf paths, and equality with the independent C walk of oracle/accept_ref.c."""
import numpy as np
import pytest

from oracle import accept as A
from oracle import lm_head as LH
from oracle import tree as OT
from synth import CONFIGS, make_lm_head_inputs, make_verify_batch, random_tree_parents
from tests.helpers import bf16_bits


def test_permutation_rows_closed_form():
    """W = rows of a permutation matrix: logits[r, v] = H[r, perm[v]] exactly, so the arg-max
    is perm^-1 of the row's arg-max coordinate."""
    rng = np.random.default_rng(0)
    Dm = 37
    perm = rng.permutation(Dm)
    W = np.eye(Dm)[perm]                     # W[v] = e_{perm[v]}
    H = rng.standard_normal((11, Dm))
    lg = LH.lm_head_logits(H, W)
    for r in range(11):
        for v in range(Dm):
            assert lg[r, v] == H[r, perm[v]]
    idx, mx = LH.lm_head_argmax(H, W)
    inv = np.argsort(perm)
    assert np.array_equal(idx, inv[np.argmax(H, axis=1)])
    assert np.array_equal(mx, H.max(axis=1))


def test_ties_lowest_vocab_id():
    """Duplicated weight rows give exactly equal logits; the lowest vocabulary id wins (Z6)."""
    rng = np.random.default_rng(1)
    Dm, V = 16, 40
    W = rng.standard_normal((V, Dm))
    H = rng.standard_normal((8, Dm))
    idx0, _ = LH.lm_head_argmax(H, W)
    lo = 3
    for r in range(8):
        t = int(idx0[r])
        Wt = W.copy()
        j = min(t, lo)
        Wt[j] = W[t]                        # row j (<= t) now ties with row t
        idx, _ = LH.lm_head_argmax(H[r:r + 1], Wt)
        assert idx[0] == j


def test_sign_and_scale():
    rng = np.random.default_rng(2)
    H = rng.standard_normal((9, 24))
    W = rng.standard_normal((30, 24))
    idx, mx = LH.lm_head_argmax(H, W)
    idx2, mx2 = LH.lm_head_argmax(4.0 * H, W)      # exact power-of-two scaling
    assert np.array_equal(idx, idx2) and np.array_equal(4.0 * mx, mx2)
    idx3, mx3 = LH.lm_head_argmax(-H, W)           # arg-max of -x is the arg-min of x
    lg = H @ W.T
    assert np.array_equal(idx3, np.argmin(lg, axis=1))


def test_planted_margin():
    """The synthetic generator plants the preferred token; on real shapes it must be the arg-max."""
    b = make_verify_batch(CONFIGS["tiny"], device="cpu")
    inp = make_lm_head_inputs(b, Dm=512, seed=3)
    idx, _ = LH.lm_head_argmax(inp["hidden"].float().numpy(), inp["weight"].float().numpy())
    assert np.array_equal(idx, inp["planted"].astype(np.int32))


def _bruteforce_walk(parent, token, amax):
    """Longest prefix over all root-to-leaf paths whose every token equals the arg-max at its
    parent (EAGLE's candidate-path formulation); distinct sibling tokens make it unique."""
    T = len(parent)
    kids = [[x for x in range(T) if parent[x] == c] for c in range(T)]
    best = [0]
    for leaf in [i for i in range(T) if not kids[i]]:
        path = OT.ancestors_or_self(parent, leaf)
        acc = [0]
        for x in path[1:]:
            if token[x] == amax[parent[x]]:
                acc.append(x)
            else:
                break
        if len(acc) > len(best):
            best = acc
    return best


@pytest.mark.parametrize("seed", range(3))
def test_walk_bruteforce_and_c_oracle(seed):
    rng = np.random.default_rng(seed)
    V = 30
    parents, tokens, amaxs = [], [], []
    for _ in range(25):
        T = int(rng.integers(1, 64))
        par = random_tree_parents(rng, T)
        tok = np.zeros(T, dtype=np.int32)
        kids = [[x for x in range(T) if par[x] == c] for c in range(T)]
        for c in range(T):
            if kids[c]:
                tok[kids[c]] = rng.choice(V, size=len(kids[c]), replace=False)
        am = rng.integers(0, V, size=T).astype(np.int32)
        for c in range(T):
            if kids[c] and rng.random() < 0.75:
                am[c] = tok[rng.choice(kids[c])]
        parents.append(par), tokens.append(tok), amaxs.append(am)
    tree_off = np.concatenate([[0], np.cumsum([len(p) for p in parents])]).astype(np.int32)
    parent, token, amax = (np.concatenate(x).astype(np.int32) for x in (parents, tokens, amaxs))
    acc, path, bonus = LH.greedy_walk(amax, parent, token, tree_off)
    for b in range(len(parents)):
        bf = _bruteforce_walk(parents[b], tokens[b], amaxs[b])
        assert acc[b] == len(bf) - 1
        assert path[b, :acc[b] + 1].tolist() == bf and np.all(path[b, acc[b] + 1:] == -1)
        assert bonus[b] == amaxs[b][bf[-1]]
    # the C oracle's greedy rule on logits whose arg-max is amax (one +8 spike over N(0,1)
    # noise in bf16) reaches the same walk
    NT = len(parent)
    lg = rng.standard_normal((NT, V)).astype(np.float32)
    lg[np.arange(NT), amax] += 8.0
    gid = np.arange(len(parents), dtype=np.int64)
    acc2, path2, bonus2, flags = A.tree_accept(A.GREEDY, bf16_bits(lg), parent, token, tree_off, gid, V)
    assert np.array_equal(acc, acc2) and np.array_equal(path, path2) and np.array_equal(bonus, bonus2)


def test_walk_special_cases():
    # T = 1: nothing to accept, bonus = arg-max of the root
    acc, path, bonus = LH.greedy_walk(np.array([5]), np.array([-1]), np.array([9]), np.array([0, 1]))
    assert acc[0] == 0 and bonus[0] == 5 and path[0, 0] == 0
    # chain whose tokens follow the arg-max: everything accepted
    par = np.array([-1, 0, 1, 2]); tok = np.array([0, 4, 5, 6]); am = np.array([4, 5, 6, 7])
    acc, path, bonus = LH.greedy_walk(am, par, tok, np.array([0, 4]))
    assert acc[0] == 3 and path[0, :4].tolist() == [0, 1, 2, 3] and bonus[0] == 7
    # duplicate sibling tokens: the lowest node index is taken (Z6), even if the other goes deeper
    par = np.array([-1, 0, 0, 2]); tok = np.array([0, 4, 4, 5]); am = np.array([4, 9, 5, 1])
    acc, path, bonus = LH.greedy_walk(am, par, tok, np.array([0, 4]))
    assert acc[0] == 1 and path[0, :2].tolist() == [0, 1] and bonus[0] == 9


def test_nonfinite_rows_have_no_argmax():
    """Z15 on the fused path: a row with any NaN or +-Inf logit has no arg-max (-1, NaN), so the
    walk stops there with RS_FLAG_NONFINITE exactly as rs_tree_accept does on logits; finite
    rows are untouched (a +Inf would otherwise win, a NaN would be skipped)."""
    lg = np.array([[0.0, 3.0, 1.0], [0.0, np.inf, 1.0], [np.nan, 3.0, 5.0], [-np.inf, -1.0, -2.0]])
    idx, mx = LH.argmax_rows(lg)
    assert idx.tolist() == [1, -1, -1, -1]
    assert mx[0] == 3.0 and np.isnan(mx[1:]).all()
    acc, path, bonus = LH.greedy_walk(np.array([-1, 5], np.int32), np.array([-1, 0], np.int32),
                                       np.array([0, 5], np.int32), np.array([0, 2], np.int32))
    assert acc[0] == 0 and bonus[0] == -1
