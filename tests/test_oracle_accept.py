"""Pins for oracle.accept: greedy by brute force, sampling by distribution (chi-square on 1e6
trials), closed forms, special cases, and negative controls proving the tests have power."""
import numpy as np
import pytest

from oracle import accept as A
from oracle import tree as OT
from synth import random_tree_parents
from tests.helpers import bf16_bits, bits_to_f32, chi2_pvalue, softmax64

V_SMALL = 8


# ---------------------------------------------------------------- greedy
def _root_to_leaf_paths(parent):
    T = len(parent)
    kids = [[x for x in range(T) if parent[x] == c] for c in range(T)]
    leaves = [i for i in range(T) if not kids[i]]
    return [OT.ancestors_or_self(parent, l) for l in leaves]


def _greedy_bruteforce(parent, token, logits_f32):
    """EAGLE-style: for each root-to-leaf path, the accepted prefix is the longest prefix whose
    every token equals the argmax of its parent's row; the answer is the longest over paths."""
    amax = logits_f32.argmax(axis=1)     # numpy: first occurrence = lowest id on ties
    best = [0]
    for path in _root_to_leaf_paths(parent):
        acc = [0]
        for x in path[1:]:
            if token[x] == amax[parent[x]]:
                acc.append(x)
            else:
                break
        if len(acc) > len(best):
            best = acc
    return best, int(amax[best[-1]])


def _greedy_case(rng, T, V, p_hit):
    parent = random_tree_parents(rng, T)
    token = np.zeros(T, dtype=np.int32)
    kids = [[x for x in range(T) if parent[x] == c] for c in range(T)]
    for c in range(T):
        if kids[c]:
            token[kids[c]] = rng.choice(V, size=len(kids[c]), replace=False)
    logits = rng.standard_normal((T, V)).astype(np.float32)
    for c in range(T):
        if kids[c] and rng.random() < p_hit:
            logits[c, token[rng.choice(kids[c])]] += 6.0
    return parent, token, logits


@pytest.mark.parametrize("seed", range(4))
def test_greedy_equals_bruteforce(seed):
    rng = np.random.default_rng(seed)
    B, V = 40, 50
    cases = [_greedy_case(rng, int(rng.integers(1, 40)), V, 0.7) for _ in range(B)]
    tree_off = np.concatenate([[0], np.cumsum([len(c[0]) for c in cases])]).astype(np.int32)
    parent = np.concatenate([c[0] for c in cases])
    token = np.concatenate([c[1] for c in cases])
    logits = bf16_bits(np.concatenate([c[2] for c in cases]))
    acc, path, bonus, flags = A.tree_accept(A.GREEDY, logits, parent, token, tree_off,
                                            np.arange(B), V)
    lf = bits_to_f32(logits)
    for b, (par, tok, _) in enumerate(cases):
        s = tree_off[b]
        best, bon = _greedy_bruteforce(list(par), tok, lf[s:s + len(par)])
        assert flags[b] == 0
        assert acc[b] == len(best) - 1
        assert list(path[b, :len(best)]) == best and np.all(path[b, len(best):] == -1)
        assert bonus[b] == bon


def test_greedy_special_cases():
    V = 16
    # T = 1: nothing accepted, bonus = argmax of row 0
    l = np.zeros((1, V), np.float32)
    l[0, 9] = 2.0
    acc, path, bonus, _ = A.tree_accept(A.GREEDY, bf16_bits(l), [-1], [3], [0, 1], [0], V)
    assert acc[0] == 0 and bonus[0] == 9 and path[0, 0] == 0 and path[0, 1] == -1
    # chain whose tokens equal the parent argmax -> all T-1 accepted
    T = 10
    par = np.arange(-1, T - 1)
    tok = np.arange(T) + 1
    l = np.zeros((T, V), np.float32)
    for c in range(T - 1):
        l[c, tok[c + 1]] = 1.0
    l[T - 1, 0] = 1.0
    acc, path, bonus, _ = A.tree_accept(A.GREEDY, bf16_bits(l), par, tok, [0, T], [0], V)
    assert acc[0] == T - 1 and list(path[0, :T]) == list(range(T)) and bonus[0] == 0
    # no child matches -> a = 0
    l2 = l.copy()
    l2[0, :] = 0
    l2[0, 15] = 1.0
    acc, _, bonus, _ = A.tree_accept(A.GREEDY, bf16_bits(l2), par, tok, [0, T], [0], V)
    assert acc[0] == 0 and bonus[0] == 15
    # ties -> lowest vocab id; duplicate sibling tokens -> lowest node index
    par3 = [-1, 0, 0]
    tok3 = [0, 5, 5]
    l3 = np.zeros((3, V), np.float32)
    l3[0, 5] = 1.0
    l3[0, 7] = 1.0       # tie between 5 and 7 -> 5
    acc, path, _, _ = A.tree_accept(A.GREEDY, bf16_bits(l3), par3, tok3, [0, 3], [0], V)
    assert acc[0] == 1 and path[0, 1] == 1


def test_flags_malformed_and_nonfinite():
    V = 8
    l = np.zeros((4, V), np.float32)
    acc, path, bonus, flags = A.tree_accept(A.GREEDY, bf16_bits(l), [-1, 0, 3, 1], [0] * 4,
                                            [0, 4], [0], V)
    assert flags[0] == A.FLAG_MALFORMED and acc[0] == 0 and bonus[0] == -1 and path[0, 0] == -1
    l[0, 3] = np.nan
    for mode in (A.GREEDY, A.DELTA):
        acc, path, bonus, flags = A.tree_accept(mode, bf16_bits(l), [-1, 0, 0, 1], [0, 1, 2, 3],
                                                [0, 4], [0], V)
        assert flags[0] == A.FLAG_NONFINITE and bonus[0] == -1 and acc[0] == 0


# ---------------------------------------------------------------- sampling
def _replicate(parent, token_rows, logits, n, draft=None):
    """n independent trials of the same tree (token_rows: [n, T] per-trial tokens)."""
    T = len(parent)
    tree_off = (np.arange(n + 1) * T).astype(np.int32)
    par = np.tile(np.asarray(parent, np.int32), n)
    tok = np.asarray(token_rows, np.int32).reshape(-1)
    lg = np.tile(logits, (n, 1))
    dp = None if draft is None else np.tile(draft.astype(np.float32), (n, 1))
    return tree_off, par, tok, lg, dp


def _emitted(acc, path, bonus, tok, T, k):
    """k-th emitted token per trial (1-based); -1 if fewer emitted."""
    n = len(acc)
    out = np.full(n, -1)
    for b in range(n):
        toks = [tok[b * T + x] for x in path[b, 1:acc[b] + 1]] + [bonus[b]]
        if len(toks) >= k:
            out[b] = toks[k - 1]
    return out


def _two_level_case(seed, K):
    rng = np.random.default_rng(seed)
    # root with K children, each with 2 children (BFS order)
    parent = [-1] + [0] * K
    for c in range(1, K + 1):
        parent += [c, c]
    T = len(parent)
    logits = bf16_bits(rng.standard_normal((T, V_SMALL)) * 1.5)
    q = softmax64(rng.standard_normal((T, V_SMALL)) * 1.2)
    return parent, logits, q


def _draw_children_tokens(rng, parent, q, n, how):
    T = len(parent)
    toks = np.zeros((n, T), dtype=np.int32)
    kids = [[x for x in range(T) if parent[x] == c] for c in range(T)]
    for c in range(T):
        if not kids[c]:
            continue
        K = len(kids[c])
        if how == "iid":
            toks[:, kids[c]] = rng.choice(V_SMALL, size=(n, K), p=q[c])
        elif how == "iid_sorted":          # negative control: reorder draws by descending q
            d = rng.choice(V_SMALL, size=(n, K), p=q[c])
            order = np.argsort(-q[c][d], axis=1, kind="stable")
            toks[:, kids[c]] = np.take_along_axis(d, order, axis=1)
        elif how == "topk":
            toks[:, kids[c]] = np.argsort(-q[c], kind="stable")[:K]
    return toks


N_TRIALS = 1_000_000


@pytest.mark.parametrize("mode,how,K", [(A.MSS, "iid", 1), (A.MSS, "iid", 2), (A.MSS, "iid", 3),
                                        (A.DELTA, "topk", 1), (A.DELTA, "topk", 3)])
def test_sampling_preserves_target_distribution(mode, how, K):
    """chi-square on 1e6 trials: first emitted token ~ p_root; second ~ p_x given first = x."""
    parent, logits, q = _two_level_case(100 + K, K)
    rng = np.random.default_rng(7 + K)
    toks = _draw_children_tokens(rng, parent, q, N_TRIALS, how)
    tree_off, par, tok, lg, dp = _replicate(parent, toks, logits, N_TRIALS,
                                            q if mode == A.MSS else None)
    acc, path, bonus, flags = A.tree_accept(mode, lg, par, tok, tree_off,
                                            np.arange(N_TRIALS) * 3 + 1, V_SMALL, draft_probs=dp,
                                            seed=1234, step=5)
    assert not flags.any()
    p = softmax64(bits_to_f32(logits))
    T = len(parent)
    first = _emitted(acc, path, bonus, tok, T, 1)
    pv, _ = chi2_pvalue(np.bincount(first, minlength=V_SMALL), p[0])
    assert pv > 1e-4, pv
    # conditional second token given the first came from accepting child x (a tree node)
    for b_node in range(1, K + 1):
        sel = (acc >= 1) & (path[:, 1] == b_node)
        if sel.sum() < 5000:
            continue
        second = _emitted(acc[sel], path[sel], bonus[sel], tok[np.repeat(sel, T)], T, 2)
        pv2, _ = chi2_pvalue(np.bincount(second, minlength=V_SMALL), p[b_node])
        assert pv2 > 1e-4, (b_node, pv2)


@pytest.mark.parametrize("how,mode", [("iid_sorted", A.MSS), ("topk", A.MSS)])
def test_chi2_has_power_negative_controls(how, mode):
    """Known-biased pairings must be rejected (SURVEY 8(c) c-3 TV table)."""
    parent, logits, q = _two_level_case(202, 2)
    rng = np.random.default_rng(9)
    n = 300_000
    toks = _draw_children_tokens(rng, parent, q, n, how)
    tree_off, par, tok, lg, dp = _replicate(parent, toks, logits, n, q)
    acc, path, bonus, _ = A.tree_accept(mode, lg, par, tok, tree_off, np.arange(n), V_SMALL,
                                        draft_probs=dp, seed=99, step=1)
    p = softmax64(bits_to_f32(logits))
    first = _emitted(acc, path, bonus, tok, len(parent), 1)
    pv, _ = chi2_pvalue(np.bincount(first, minlength=V_SMALL), p[0])
    assert pv < 1e-6, pv


def test_single_child_acceptance_closed_forms():
    """MSS: P(accept) = sum_v min(p_v, q_v) = 1 - TV(p, q); DELTA: P(accept x) = p(x)."""
    rng = np.random.default_rng(3)
    parent = [-1, 0]
    logits = bf16_bits(rng.standard_normal((2, V_SMALL)))
    q = softmax64(rng.standard_normal((2, V_SMALL)))
    p = softmax64(bits_to_f32(logits))
    n = 400_000
    toks = _draw_children_tokens(rng, parent, q, n, "iid")
    tree_off, par, tok, lg, dp = _replicate(parent, toks, logits, n, q)
    acc, *_ = A.tree_accept(A.MSS, lg, par, tok, tree_off, np.arange(n), V_SMALL, draft_probs=dp,
                            seed=5, step=0)
    expect = np.minimum(p[0], q[0]).sum()
    assert abs(acc.mean() - expect) < 5 * np.sqrt(expect * (1 - expect) / n)
    for x in range(V_SMALL):
        toks = np.tile(np.array([[0, x]], np.int32), (n // 8, 1))
        tree_off, par, tok, lg, _ = _replicate(parent, toks, logits, n // 8)
        acc, *_ = A.tree_accept(A.DELTA, lg, par, tok, tree_off, np.arange(n // 8), V_SMALL,
                                seed=6, step=x)
        e = p[0, x]
        assert abs(acc.mean() - e) < 5 * np.sqrt(e * (1 - e) / (n // 8)) + 1e-9


def test_sampling_special_cases():
    # p one-hot on a non-child token -> always rejected, bonus is that token
    l = np.full((3, V_SMALL), -60.0, np.float32)
    l[0, 6] = 0.0
    q = softmax64(np.zeros((3, V_SMALL)))
    n = 2000
    toks = np.tile(np.array([[0, 1, 2]], np.int32), (n, 1))
    for mode in (A.DELTA, A.MSS):
        tree_off, par, tok, lg, dp = _replicate([-1, 0, 0], toks, bf16_bits(l), n, q)
        acc, _, bonus, _ = A.tree_accept(mode, lg, par, tok, tree_off, np.arange(n), V_SMALL,
                                         draft_probs=dp)
        assert np.all(acc == 0) and np.all(bonus == 6)
    # T = 1 -> bonus ~ p_root (chi-square)
    rng = np.random.default_rng(4)
    l1 = bf16_bits(rng.standard_normal((1, V_SMALL)))
    n = 200_000
    tree_off, par, tok, lg, _ = _replicate([-1], np.zeros((n, 1), np.int32), l1, n)
    acc, _, bonus, _ = A.tree_accept(A.DELTA, lg, par, tok, tree_off, np.arange(n), V_SMALL)
    pv, _ = chi2_pvalue(np.bincount(bonus, minlength=V_SMALL), softmax64(bits_to_f32(l1))[0])
    assert pv > 1e-4 and np.all(acc == 0)


def test_temperature_scales_target():
    """Bonus distribution at temperature tau follows softmax(l / tau)."""
    rng = np.random.default_rng(8)
    l1 = bf16_bits(rng.standard_normal((1, V_SMALL)) * 2)
    n = 200_000
    tree_off, par, tok, lg, _ = _replicate([-1], np.zeros((n, 1), np.int32), l1, n)
    for tau in (0.5, 2.0):
        _, _, bonus, _ = A.tree_accept(A.DELTA, lg, par, tok, tree_off, np.arange(n), V_SMALL,
                                       temperature=tau)
        pv, _ = chi2_pvalue(np.bincount(bonus, minlength=V_SMALL),
                            softmax64(bits_to_f32(l1), tau)[0])
        assert pv > 1e-4, (tau, pv)


def test_rng_keyed_by_gid_not_position():
    """Results depend on (seed, step, gid) only: permuting samples permutes outputs."""
    parent, logits, q = _two_level_case(31, 3)
    rng = np.random.default_rng(1)
    n = 500
    toks = _draw_children_tokens(rng, parent, q, n, "iid")
    gid = rng.permutation(10 * n)[:n]
    tree_off, par, tok, lg, dp = _replicate(parent, toks, logits, n, q)
    r1 = A.tree_accept(A.MSS, lg, par, tok, tree_off, gid, V_SMALL, draft_probs=dp, seed=3, step=9)
    perm = rng.permutation(n)
    T = len(parent)
    tree_off2, par2, tok2, lg2, dp2 = _replicate(parent, toks[perm], logits, n, q)
    r2 = A.tree_accept(A.MSS, lg2, par2, tok2, tree_off2, gid[perm], V_SMALL, draft_probs=dp2,
                       seed=3, step=9)
    for a, b in zip(r1, r2):
        np.testing.assert_array_equal(a[perm], b)
    r3 = A.tree_accept(A.MSS, lg, par, tok, tree_off, gid, V_SMALL, draft_probs=dp, seed=3, step=10)
    assert not all(np.array_equal(a, b) for a, b in zip(r1, r3))


# ---------------------------------------------------------------- malformed tokens, degenerate residual
def test_out_of_vocabulary_token_is_malformed():
    """A draft node whose token is outside [0, V) (rs_tree_select pads with -1) makes the tree
    malformed in every mode (reading Z5: rows are indexed by the child's token); the root's
    token is never tested, so -1 there is fine."""
    V = 8
    l = np.zeros((3, V), np.float32)
    q = softmax64(np.zeros((3, V)))
    for bad in (-1, V, V + 100):
        for mode in (A.GREEDY, A.DELTA, A.MSS):
            acc, path, bonus, flags = A.tree_accept(mode, bf16_bits(l), [-1, 0, 0], [0, 2, bad], [0, 3],
                                                    [0], V, draft_probs=q if mode == A.MSS else None)
            assert flags[0] == A.FLAG_MALFORMED and acc[0] == 0 and bonus[0] == -1, (bad, mode)
    acc, _, bonus, flags = A.tree_accept(A.GREEDY, bf16_bits(l), [-1, 0], [-1, 3], [0, 2], [0], V)
    assert flags[0] == 0 and bonus[0] == 0


def _uniform_support_logits(V, support, rows):
    l = np.full((rows, V), -100.0, np.float32)     # exp(-100) underflows exp_spec -> weight 0
    l[:, support] = 0.0                              # weight exactly 2^32 each
    return l


def test_mss_degenerate_residual_zero_draft_mass():
    """Degenerate residual (DESIGN "Bit-exact sampling": an all-zero residual keeps the
    pre-rejection weights). A draft row whose mass quantises to 0 (Zq = 0) rejects every child
    of zero target weight (qw_x = 0 -> accept iff w_x > 0) and leaves r = max(w*0 - 0*Z, 0) = 0.
    The bonus is then drawn from the ORIGINAL target p: with p uniform on k = 4 tokens of
    weight 2^32 each (Z = 4*2^32), t = U'*Z >> 32 = 4*U' and the bonus is support[4*U' >> 32]
    (closed form; U' = Philox word 0 at counter (0xFFFFFFFF, 0, step, gid), key = seed, pinned
    by the Random123 vectors)."""
    V, support = 16, [1, 3, 4, 6]
    l = bf16_bits(_uniform_support_logits(V, support, 3))
    q = np.zeros((3, V), np.float32)                 # Zq = 0
    for gid in range(40):
        acc, path, bonus, flags = A.tree_accept(A.MSS, l, [-1, 0, 0], [0, 9, 11], [0, 3], [gid], V,
                                                draft_probs=q, seed=77, step=5)
        u2 = int(A.philox4x32_10([0xFFFFFFFF, 0, 5, gid], [77, 0])[0])
        assert flags[0] == 0 and acc[0] == 0
        assert bonus[0] == support[(4 * u2) >> 32], gid


def test_mss_degenerate_residual_proportional_draft():
    """q exactly proportional to p (p uniform on 4 tokens, q = 1/4 on them): rejecting a child
    outside the support leaves r_v = w_v*Zq - qw_v*Z = 2^32*2^32 - 2^30*2^34 = 0 for every v, so
    the pre-rejection weights are kept and the next child (in the support) is accepted with
    certainty (U*(qw*Z) = U*2^64 < 2^32*(w*Zq) = 2^96). Had the residual been taken as the
    all-zero vector, Z = 0 and that child would be rejected."""
    V, support = 16, [1, 3, 4, 6]
    l = _uniform_support_logits(V, support, 4)
    l[3] = -100.0
    l[3, 5] = 0.0                                    # leaf row: bonus deterministic (token 5)
    q = np.zeros((4, V), np.float32)
    q[:, support] = 0.25
    for gid in range(20):
        acc, path, bonus, flags = A.tree_accept(A.MSS, bf16_bits(l), [-1, 0, 0, 0], [0, 9, 11, 3], [0, 4],
                                                [gid], V, draft_probs=q, seed=3, step=gid)
        assert flags[0] == 0 and acc[0] == 1 and list(path[0, :2]) == [0, 3] and bonus[0] == 5


def test_mss_draft_row_must_be_probabilities():
    """MSS: a visited node whose draft row holds a value outside [0, 1] (or NaN) is flagged like
    a non-finite row (walk stops there, bonus -1); rows never visited are not checked."""
    V = 8
    l = np.zeros((3, V), np.float32)
    l[0, 2] = 30.0                                     # child token 2 is (almost) certain at the root
    q = softmax64(np.zeros((3, V))).astype(np.float32)
    q[0, 2] = 1.0
    for bad in (1.5, -0.25, np.nan):
        qb = q.copy()
        qb[1, 5] = bad                                 # row of node 1 (visited after accepting it)
        acc, path, bonus, flags = A.tree_accept(A.MSS, bf16_bits(l), [-1, 0, 1], [0, 2, 3], [0, 3], [0], V,
                                                draft_probs=qb)
        assert flags[0] == A.FLAG_NONFINITE and acc[0] == 1 and bonus[0] == -1, bad
        qb = q.copy()
        qb[2, 5] = bad                                 # never visited when node 2 is rejected
        l2 = l.copy()
        l2[1, :] = 0.0
        l2[1, 0] = 30.0                                # node 1's row: child token 3 rejected
        acc, path, bonus, flags = A.tree_accept(A.MSS, bf16_bits(l2), [-1, 0, 1], [0, 2, 3], [0, 3], [0], V,
                                                draft_probs=qb)
        assert flags[0] == 0 and acc[0] == 1


def test_mss_leaf_draft_row_is_not_read():
    """Reading Z29 (children are drawn from q_c): the draft row of a node WITHOUT children
    is not a distribution anything was drawn from, so a visited leaf's row is never read — a
    NaN / out-of-range row there changes nothing, while the same row on a node with children
    flags the sample (test_mss_draft_row_must_be_probabilities)."""
    V = 8
    l = np.zeros((2, V), np.float32)
    l[0, 2] = 30.0                                     # child token 2 is (almost) certain at the root
    l[1, 6] = 3.0                                      # the leaf's target row (bonus drawn from it)
    q = softmax64(np.zeros((2, V))).astype(np.float32)
    q[0, :] = 0.0
    q[0, 2] = 1.0
    ref = A.tree_accept(A.MSS, bf16_bits(l), [-1, 0], [0, 2], [0, 2], [5], V, draft_probs=q, seed=1, step=2)
    assert ref[3][0] == 0 and ref[0][0] == 1 and list(ref[1][0, :2]) == [0, 1]
    for bad in (1.5, -0.25, np.nan):
        qb = q.copy()
        qb[1, :] = bad                                 # the leaf's row: garbage
        got = A.tree_accept(A.MSS, bf16_bits(l), [-1, 0], [0, 2], [0, 2], [5], V, draft_probs=qb, seed=1, step=2)
        for x, y in zip(got, ref):
            np.testing.assert_array_equal(x, y)


def test_mss_draft_row_map():
    """draft_row (row of node i's q, -1 = none) is a pure relayout: the rows of the nodes with
    children packed into a smaller array give the results of the full [NT, V] array; a node with
    children but no row makes its tree malformed (other samples unaffected)."""
    V, n = 32, 40
    rng = np.random.default_rng(13)
    par = np.tile(np.array([-1, 0, 0, 1, 1, 2], np.int32), n)   # internal: 0, 1, 2; leaves: 3, 4, 5
    q = rng.dirichlet(np.ones(V) * 0.3, size=6 * n).astype(np.float32)
    tok = np.zeros(6 * n, np.int32)
    for i in range(6 * n):
        if par[i] >= 0:
            pr = q[(i // 6) * 6 + par[i]].astype(np.float64)
            tok[i] = rng.choice(V, p=pr / pr.sum())
    lg = (np.log(q + 1e-12) + rng.standard_normal((6 * n, V))).astype(np.float32)
    off = (np.arange(n + 1) * 6).astype(np.int32)
    gid = np.arange(n) * 3 + 7
    full = A.tree_accept(A.MSS, lg, par, tok, off, gid, V, draft_probs=q, seed=4, step=1)
    internal = np.array([i for i in range(6 * n) if (i % 6) in (0, 1, 2)])
    row = np.full(6 * n, -1, np.int32)
    row[internal] = np.arange(len(internal))
    qc = q[internal].copy()
    packed = A.tree_accept(A.MSS, lg, par, tok, off, gid, V, draft_probs=qc, seed=4, step=1, draft_row=row)
    for x, y in zip(packed, full):
        np.testing.assert_array_equal(x, y)
    assert full[0].sum() > 0 and (full[3] == 0).all()
    row2 = row.copy()
    row2[6 * 3 + 1] = -1                               # sample 3: node 1 has children but no row
    bad = A.tree_accept(A.MSS, lg, par, tok, off, gid, V, draft_probs=qc, seed=4, step=1, draft_row=row2)
    assert bad[3][3] == A.FLAG_MALFORMED and bad[0][3] == 0 and bad[2][3] == -1
    keep = np.arange(n) != 3
    for x, y in zip(bad, full):
        np.testing.assert_array_equal(x[keep], y[keep])
