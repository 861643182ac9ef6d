"""Pins for oracle.strategy (select_strategy) and oracle.realloc (Eq. 6 planner) from the
paper's / SPEC's worked numbers (tests/golden/paper_worked_examples.txt) and brute force."""
import itertools
import math
import os

import numpy as np
import pytest

from oracle import realloc as OR
from oracle import strategy as OS
from synth import lmsys_response_lengths, make_candidate_tree

GOLD = os.path.join(os.path.dirname(__file__), "golden", "paper_worked_examples.txt")


def _golden(kind):
    for line in open(GOLD):
        if line.startswith(kind + " "):
            return line.strip()
    raise KeyError(kind)


def _kv(tok):
    k, v = tok.split("=")
    return k, v


# ----------------------------------------------------------------- selection search
def test_profile_argmax_and_early_stop_spec_example():
    line = _golden("profile").split()
    al = [float(x) for x in _kv(line[1])[1].split(",")]
    t = [float(x) for x in _kv(line[2])[1].split(",")]
    n_exp, stop_exp = int(_kv(line[4])[1]), int(_kv(line[5])[1])
    n, stop = OS.search_profile(al, t, n_min=1, patience=2)
    assert (n, stop) == (n_exp, stop_exp)


def test_sugar_water_inequality():
    line = _golden("sugar").split()
    a, b, c, d = (float(_kv(x)[1]) for x in line[1:5])
    nxt = float(line[-1])
    assert (a + c) / (b + d) == pytest.approx(nxt)
    assert c / d < a / b and c / d < (a + c) / (b + d) < a / b      # Eq. 3


def test_early_stop_equals_full_scan_when_increments_decrease():
    """When dal/dt is non-increasing the early-stopped argmax equals the full scan (Eq. 3)."""
    rng = np.random.default_rng(0)
    for _ in range(1000):
        n = int(rng.integers(3, 40))
        dal = np.sort(rng.random(n))[::-1] + 1e-3           # decreasing gains
        dt = np.sort(rng.random(n)) + 0.05                   # increasing costs
        al, t = np.cumsum(dal), 0.5 + np.cumsum(dt)
        n_es, _ = OS.search_profile(al, t, n_min=1, patience=2)
        assert n_es == int(np.argmax(al / t)) + 1


def test_argmax_invariant_to_t_ar():
    rng = np.random.default_rng(1)
    al = np.cumsum(np.sort(rng.random(20))[::-1])
    t = 1 + np.cumsum(np.sort(rng.random(20)))
    for t_ar in (0.1, 1.0, 37.0):
        assert OS.search_profile(al * t_ar, t, 1, 2)[0] == OS.search_profile(al, t, 1, 2)[0]


def test_draft_logit_chain_example():
    line = _golden("chain").split()
    o = [float(x) for x in _kv(line[1])[1].split(",")]
    dl = OS.draft_logits([-1, 0, 1], o)
    assert dl[-1] == pytest.approx(float(line[-1]))


def _connected_subsets(parent, n):
    """All connected n-subsets that contain their parents (brute force)."""
    N = len(parent)
    out = []
    for S in itertools.combinations(range(N), n):
        s = set(S)
        if all(parent[u] < 0 or parent[u] in s for u in S):
            out.append(S)
    return out


def test_layer_search_topn_matches_bruteforce_on_small_trees():
    """With w = dl (non-increasing on paths), S(n) is the max-weight connected n-subtree and
    nested; principle 1 (depth < n) holds for every selected node."""
    rng = np.random.default_rng(2)
    for trial in range(60):
        N = int(rng.integers(2, 12))
        parent, o = make_candidate_tree(rng, N)
        w = OS.draft_logits(parent, o)
        order = OS.layer_search_order(parent, w, N)
        dep = OS.cand_depths(parent)
        for n in range(1, len(order) + 1):
            S = order[:n]
            assert all(dep[u] < n for u in S)
            assert all(parent[u] < 0 or parent[u] in S for u in S)
            best = max(sum(w[list(T)]) for T in _connected_subsets(parent, n))
            assert sum(w[S]) == pytest.approx(best, rel=1e-12)


def test_select_strategy_figure8_al_sum_and_nesting():
    """al(n) = sum of w over S(n) (Fig. 8), so al(n+1) - al(n) = w(u_max) exactly."""
    rng = np.random.default_rng(3)
    trees = [make_candidate_tree(rng, 30) for _ in range(3)]
    kx = np.linspace(0, 1, 16)
    ky = np.clip(0.2 + 0.9 * kx, 0, 1)
    cost = OS.CostModel(0.5, 1.0, 1e-4, 0.02, 1e-3, 64)
    res = OS.select_strategy(trees, [100, 200, 300], kx, ky, cost, n_min=2, n_max=20, patience=100)
    orders = [OS.layer_search_order(p, [OS.acceptance_fit(kx, ky, x) for x in OS.draft_logits(p, o)], 20)
              for p, o in trees]
    for n in range(1, len(res["al_profile"]) + 1):
        exp = sum(OS.acceptance_fit(kx, ky, OS.draft_logits(p, o)[u])
                  for (p, o), od in zip(trees, orders) for u in od[:n])
        assert res["al_profile"][n - 1] == pytest.approx(exp, rel=1e-12)
    assert np.all(np.diff(res["al_profile"]) >= 0)


def test_select_strategy_load_dependence():
    """Fig. 4 shape: under heavier load the best n is not larger."""
    rng = np.random.default_rng(4)
    kx = np.linspace(0, 1, 16)
    ky = np.clip(0.2 + 0.9 * kx, 0, 1)
    cost = OS.CostModel(2e-3, 5e-3, 2e-7, 2e-6, 5e-8, 512)
    light = [make_candidate_tree(rng, 60) for _ in range(4)]
    heavy = light * 16
    n_light = OS.select_strategy(light, [1000] * 4, kx, ky, cost, n_max=48)["n"]
    n_heavy = OS.select_strategy(heavy, [1000] * 64, kx, ky, cost, n_max=48)["n"]
    assert n_heavy <= n_light


def test_bucket_cache_is_piecewise_constant():
    cost = OS.CostModel(1.0, 0.0, 1e-3, 1e-2, 0.0, 0, seq_bucket=256, draft_bucket=4)
    assert cost.t_sd(256, 4) == cost.t_sd(511, 7)
    assert cost.t_sd(512, 4) > cost.t_sd(511, 4)
    assert cost.t_sd(0, 8) > cost.t_sd(0, 7)


# ----------------------------------------------------------------- reallocation
def _parse_realloc(line):
    tok = line.split()
    loads = [int(x) for x in tok[1].split(",")]
    thr = int(_kv(tok[2])[1])
    after = [int(x) for x in tok[4].split(",")]
    return loads, thr, after


@pytest.mark.parametrize("which", [0, 1])
def test_realloc_worked_examples(which):
    lines = [l.strip() for l in open(GOLD) if l.startswith("realloc ")]
    loads, thr, after = _parse_realloc(lines[which])
    plan = OR.plan_reallocation(loads, thr)
    assert OR.apply_plan(loads, plan) == after


def _feasible_best(loads, thr):
    """Brute force of Eq. 6: max total moved into destinations over all plans where each
    instance takes part in at most one transfer, sources stay >= thr, destinations <= thr."""
    G = len(loads)
    srcs = [i for i in range(G) if loads[i] > thr]
    dsts = [i for i in range(G) if loads[i] < thr]
    best = 0

    def rec(si, used_d, total):
        nonlocal best
        best = max(best, total)
        if si == len(srcs):
            return
        rec(si + 1, used_d, total)
        s = srcs[si]
        for d in dsts:
            if d in used_d:
                continue
            k = min(loads[s] - thr, thr - loads[d])
            rec(si + 1, used_d | {d}, total + k)

    rec(0, frozenset(), 0)
    return best


def test_greedy_plan_is_optimal_small_fleets():
    rng = np.random.default_rng(5)
    for _ in range(400):
        G = int(rng.integers(2, 6))
        loads = list(rng.integers(0, 41, size=G))
        thr = int(rng.integers(1, 30))
        plan = OR.plan_reallocation(loads, thr)
        after = OR.apply_plan(loads, plan)
        moved = sum(k for _, _, k in plan)
        involved = [s for s, _, _ in plan] + [d for _, d, _ in plan]
        assert len(set(involved)) == len(involved)                  # m(k) <= 1
        for s, d, _ in plan:
            assert after[s] >= thr and after[d] <= thr               # Eq. 6 constraints
        assert moved == _feasible_best(loads, thr)


def test_knee_and_trigger():
    tok = _golden("knee").split()
    prof = [tuple(int(v) for v in x.split(":")) for x in tok[1].split(",")]
    assert OR.knee_threshold(prof) == int(tok[-1])
    assert OR.knee_threshold([(1, 10), (2, 20), (3, 30)]) == 3
    assert OR.knee_threshold([(1, 10), (2, 10), (3, 10)]) == 1
    assert OR.should_trigger([24, 1], 6, 32)
    assert not OR.should_trigger([24, 1], 6, 31)
    assert not OR.should_trigger([6, 6], 6, 100)


def test_sample_choice_prefers_short_then_low_acceptance():
    samples = [(10, 500, 2.0), (11, 100, 3.0), (12, 100, 1.5), (13, 50, 4.0)]
    assert OR.choose_samples(samples, 3) == [13, 12, 11]
    rng = np.random.default_rng(0)
    perm = [samples[i] for i in rng.permutation(4)]
    assert OR.choose_samples(perm, 3) == [13, 12, 11]


def test_lmsys_length_distribution():
    tok = _golden("lmsys").split()
    med, p95 = int(_kv(tok[1])[1]), int(_kv(tok[2])[1])
    x = lmsys_response_lengths(np.random.default_rng(0), 100_000, cap=10**9)
    assert abs(np.median(x) / med - 1) < 0.03
    assert abs(np.percentile(x, 95) / p95 - 1) < 0.05


def test_verification_tree_paths_are_candidate_paths():
    """f3 oracle: the verification tree for n is the root plus S(n); every node's root path
    spells exactly its candidate's token path (found by walking the candidate parents), the
    node set is S(n) (so the max-weight connected subtree, pinned above), and the array is
    topological."""
    rng = np.random.default_rng(11)
    kx, ky = [0.0, 0.05, 0.2, 0.5, 1.0], [0.0, 0.15, 0.45, 0.75, 0.95]
    for trial in range(40):
        N = int(rng.integers(3, 40))
        parent, o = make_candidate_tree(rng, N)
        token = rng.integers(0, 1000, size=N).astype(np.int32)
        w = [OS.acceptance_fit(kx, ky, x) for x in OS.draft_logits(parent, o)]
        full = OS.layer_search_order(parent, w, N)
        for n in sorted({1, 2, len(full) // 2 + 1, len(full)}):
            pv, tv = OS.verification_tree(parent, o, token, 7, n, kx, ky)
            assert len(pv) == n + 1 and pv[0] == -1 and tv[0] == 7
            assert all(0 <= pv[i] < i for i in range(1, n + 1))
            cand_paths = set()
            for u in full[:n]:
                seq, x = [], u
                while x >= 0:
                    seq.append(int(token[x]))
                    x = int(parent[x])
                cand_paths.add(tuple(reversed(seq)))
            tree_paths = set()
            for i in range(1, n + 1):
                seq, x = [], i
                while x > 0:
                    seq.append(int(tv[x]))
                    x = int(pv[x])
                tree_paths.add(tuple(reversed(seq)))
            assert tree_paths == cand_paths
    with pytest.raises(ValueError):
        OS.verification_tree(np.array([-1, 0], np.int32), np.array([0.5, 0.5]), np.array([1, 2], np.int32), 0, 3,
                             kx, ky)


# ----------------------------------------------------------------- F and t_sd, hand-evaluated
# The acceptance fit F ("a piecewise linear function ... fitted from offline profiling
# data") and the cost regression are pinned by values worked out by hand below,
# independent of np.interp / the oracle's formula, so a planted mistake (extrapolation past the
# last knot, a wrong segment, no clamp, a squared relu, a dropped term) fails one of them.
KX = [0.0, 0.05, 0.2, 0.5, 1.0]
KY = [0.0, 0.15, 0.45, 0.75, 0.95]


@pytest.mark.parametrize("x,expect", [
    (0.0, 0.0), (0.05, 0.15), (0.2, 0.45), (0.5, 0.75), (1.0, 0.95),   # at the knots
    (0.025, 0.075),       # 0 + (0.025 - 0) / 0.05 * 0.15
    (0.1, 0.25),          # 0.15 + (0.1 - 0.05) / 0.15 * 0.30
    (0.35, 0.60),         # 0.45 + (0.35 - 0.2) / 0.3 * 0.30
    (0.75, 0.85),         # 0.75 + (0.75 - 0.5) / 0.5 * 0.20
    (0.9, 0.91),          # 0.75 + 0.4 / 0.5 * 0.20
    (-0.3, 0.0),          # left of the first knot: constant F(x0) (no extrapolation)
    (1.7, 0.95),          # right of the last knot: constant 0.95, not 0.95 + 0.7 * 0.4
])
def test_acceptance_fit_hand_values(x, expect):
    assert OS.acceptance_fit(KX, KY, x) == pytest.approx(expect, abs=1e-12)


def test_acceptance_fit_clamps_to_unit_interval():
    # knots outside [0, 1]: F is a probability, so values clip to [0, 1]
    kx, ky = [0.0, 1.0], [-0.5, 1.5]
    assert OS.acceptance_fit(kx, ky, 0.1) == 0.0          # raw -0.3 -> 0
    assert OS.acceptance_fit(kx, ky, 0.5) == pytest.approx(0.5)
    assert OS.acceptance_fit(kx, ky, 0.9) == 1.0          # raw 1.3 -> 1


def test_cost_regression_hand_values():
    # t_sd = c_draft + b0 + b1 N_seq + b2 N_draft + b3 relu(N_draft - k_sat) N_draft
    cm = OS.CostModel(c_draft=1.0, b0=2.0, b1=0.5, b2=0.25, b3=0.125, k_sat=10)
    # relu inactive: 1 + 2 + 0.5*4 + 0.25*8 = 7
    assert cm.regression(4, 8) == pytest.approx(7.0)
    # relu active: 1 + 2 + 0.5*4 + 0.25*14 + 0.125*(14-10)*14 = 1 + 2 + 2 + 3.5 + 7 = 15.5
    assert cm.regression(4, 14) == pytest.approx(15.5)
    # at the saturation point the relu term is 0: 1 + 2 + 0 + 0.25*10 = 5.5
    assert cm.regression(0, 10) == pytest.approx(5.5)
    # bucket cache: (300, 15) evaluates at the bucket's lower corner (256, 12)   (Z12)
    # 1 + 2 + 0.5*256 + 0.25*12 + 0.125*2*12 = 3 + 128 + 3 + 3 = 137
    assert cm.t_sd(300, 15) == pytest.approx(137.0)


def test_verification_tree_rejects_invalid_fit_and_probabilities():
    rng = np.random.default_rng(3)
    p, o = make_candidate_tree(rng, 30)
    tok = np.arange(30, dtype=np.int32)
    OS.verification_tree(p, o, tok, 7, 6, KX, KY)                         # valid
    for kx, ky in (([0, 0.5, 0.5, 1], [0, .2, .4, .9]),                  # x not strictly increasing
                   ([0, 0.5, 1], [0, .6, .4]),                           # y decreasing (F not monotone)
                   ([0, 0.5, 1], [0, np.nan, .9])):
        with pytest.raises(ValueError, match="MalformedTree"):
            OS.verification_tree(p, o, tok, 7, 6, kx, ky)
    bad = o.copy()
    bad[4] = 1.5
    with pytest.raises(ValueError, match="MalformedTree"):
        OS.verification_tree(p, bad, tok, 7, 6, KX, KY)


# ---------------------------------------------------------------- fit_acceptance
def test_fit_acceptance_pava_hand_example():
    """Hand-computed pool-adjacent-violators: bucket rates 0.2, 0.6, 0.4, 0.9 with counts
    1, 1, 3, 1 -> the violating pair (0.6 | 1 obs, 0.4 | 3 obs) pools to (0.6 + 1.2) / 4 = 0.45;
    knot x = bucket means of dl."""
    # K = 4 buckets over [0, 1]: [0, .25) [.25, .5) [.5, .75) [.75, 1]
    obs = [(0.1, 0.2), (0.3, 0.6), (0.6, 0.4), (0.6, 0.4), (0.7, 0.4), (0.9, 0.9)]
    kx, ky = OS.fit_acceptance([o[0] for o in obs], [o[1] for o in obs], n_buckets=4)
    np.testing.assert_allclose(kx, [0.1, 0.3, (0.6 + 0.6 + 0.7) / 3, 0.9], rtol=0, atol=1e-15)
    np.testing.assert_allclose(ky, [0.2, 0.45, 0.45, 0.9], rtol=0, atol=1e-15)


def test_fit_acceptance_pava_cascade_and_empty_buckets():
    """A later low bucket pools backwards through two earlier blocks: rates 0.5, 0.7, 0.8, 0.1
    (counts 1 each, buckets 2 and 4 of 6 empty): 0.8 | 0.1 -> 0.45, then 0.7 > 0.45 ->
    (0.7 + 0.8 + 0.1) / 3; 0.5 < 1.6 / 3 stays."""
    dl = [0.05, 0.2, 0.55, 0.95]   # buckets 0, 1, 3, 5 of K = 6
    acc = [0.5, 0.7, 0.8, 0.1]
    kx, ky = OS.fit_acceptance(dl, acc, n_buckets=6)
    np.testing.assert_allclose(kx, dl, rtol=0, atol=1e-15)
    np.testing.assert_allclose(ky, [0.5] + [1.6 / 3] * 3, rtol=0, atol=1e-15)


def test_fit_acceptance_spec_examples():
    """identity target -> F within 0.05 of x on [0, 1]; G(x) = min(1, 0.2 + 0.9x),
    10k Bernoulli observations -> within 0.05 of G on [0.05, 0.95]; all accepted -> F == 1."""
    rng = np.random.default_rng(3)
    for G, lo, hi in ((lambda x: x, 0.0, 1.0), (lambda x: np.minimum(1.0, 0.2 + 0.9 * x), 0.05, 0.95)):
        dl = rng.random(10000)
        acc = (rng.random(10000) < G(dl)).astype(float)
        kx, ky = OS.fit_acceptance(dl, acc, n_buckets=20)
        xs = np.linspace(lo, hi, 181)
        F = np.array([OS.acceptance_fit(kx, ky, x) for x in xs])
        assert np.max(np.abs(F - G(xs))) < 0.05 + (1 / 40 if lo == 0.0 else 0.0)
        assert np.all(np.diff(ky) >= 0)
    kx, ky = OS.fit_acceptance(rng.random(500), np.ones(500))
    assert np.all(ky == 1.0)


def test_fit_acceptance_monotone_and_insufficient():
    rng = np.random.default_rng(11)
    for _ in range(50):
        n = int(rng.integers(2, 300))
        dl = rng.random(n)
        acc = rng.random(n)
        kx, ky = OS.fit_acceptance(dl, acc, n_buckets=int(rng.integers(1, 30)))
        assert np.all(np.diff(kx) > 0) and np.all(np.diff(ky) >= -1e-15)
        assert np.all(ky >= acc.min() - 1e-15) and np.all(ky <= acc.max() + 1e-15)
    with pytest.raises(ValueError):
        OS.fit_acceptance([0.3, 0.3, 0.3], [1, 0, 1])
