"""The library's host C++ (select_strategy, the reallocation planner, the page pool) against the
oracle on CPU. These calls do no device work, so they run without a GPU. Exact agreement is
expected: both sides evaluate the same double-precision expressions in the same order
(a0/a6)."""
import numpy as np
import pytest

from oracle import realloc as OR
from oracle import strategy as OS
from synth import make_candidate_tree

KX = [0.0, 0.05, 0.2, 0.5, 1.0]
KY = [0.0, 0.15, 0.45, 0.75, 0.95]


@pytest.fixture(scope="module")
def core():
    from paper_2512_04752_b200 import core as C
    return C


def _cost(seq_bucket=256, draft_bucket=4, k_sat=256.0):
    return OS.CostModel(c_draft=1.2e-3, b0=4e-3, b1=2.5e-8, b2=6e-6, b3=3e-9, k_sat=k_sat,
                        seq_bucket=seq_bucket, draft_bucket=draft_bucket)


@pytest.mark.parametrize("seed", range(40))
def test_select_strategy_matches_oracle(core, seed):
    rng = np.random.default_rng(seed)
    B = int(rng.integers(1, 48))
    trees = [make_candidate_tree(rng, int(rng.integers(4, 80))) for _ in range(B)]
    prefix = rng.integers(16, 8192, size=B)
    cost = _cost(seq_bucket=int(rng.choice([1, 64, 256])), draft_bucket=int(rng.choice([1, 4, 8])),
                 k_sat=float(rng.choice([32, 128, 512])))
    n_max = int(rng.integers(4, 64))
    n_min = int(rng.integers(1, 3))
    feasible = min(len(OS.layer_search_order(p, np.ones(len(p)), n_max)) for p, _ in trees)
    sel = core.Selector(cost, KX, KY)
    if feasible < n_min:
        with pytest.raises(core.RSError):
            sel.select(trees, prefix, n_min=n_min, n_max=n_max)
        return
    ref = OS.select_strategy(trees, prefix, KX, KY, cost, n_min=n_min, n_max=n_max, patience=2)
    got = sel.select(trees, prefix, n_min=n_min, n_max=n_max, patience=2, return_selected=True)
    for k in ("n", "depth", "width", "n_stop"):
        assert got[k] == ref[k], k
    for k in ("al", "t_sd", "objective"):
        assert got[k] == ref[k], k          # same expression, same order: bit-identical
    # the selection order per sample equals the oracle's layer search up to the early stop (the
    # search stops with Eq. 3: rows hold S(n_stop), -1 after)
    ns = got["n_stop"]
    for b, (p, o) in enumerate(trees):
        w = np.array([OS.acceptance_fit(KX, KY, x) for x in OS.draft_logits(p, o)])
        order = OS.layer_search_order(p, w, n_max)
        row = got["selected"][b]
        assert list(row[:ns]) == order[:ns] and np.all(row[ns:] == -1)


def test_selector_bucket_cache_hits(core):
    rng = np.random.default_rng(7)
    trees = [make_candidate_tree(rng, 40) for _ in range(8)]
    sel = core.Selector(_cost(seq_bucket=1024, draft_bucket=16), KX, KY)
    a = sel.select(trees, [1000] * 8)
    b = sel.select(trees, [1010] * 8)       # same seq bucket: every prediction is cached
    assert b["cache_hit"] == 1 and b["cache_entries"] == a["cache_entries"]
    assert (a["n"], a["objective"]) == (b["n"], b["objective"])


def test_selector_rejects_bad_inputs(core):
    with pytest.raises(core.RSError):
        core.Selector(_cost(), [0.0, 0.5, 0.4], [0.0, 0.1, 0.2])    # x not increasing
    with pytest.raises(core.RSError):
        core.Selector(_cost(), [0.0, 1.0], [0.5, 0.2])              # F not monotone
    sel = core.Selector(_cost(), KX, KY)
    with pytest.raises(core.RSError):
        sel.select([(np.array([0], np.int32), np.array([0.5]))], [10])   # parent not < index
    with pytest.raises(core.RSError):
        sel.select([(np.array([1, -1], np.int32), np.array([0.5, 0.5]))], [10])


def test_cost_model_fit_recovers_coefficients(core):
    rng = np.random.default_rng(3)
    truth = _cost(k_sat=128.0)
    ns = rng.integers(1000, 2_000_000, size=200).astype(np.float64)
    nd = rng.integers(8, 1024, size=200).astype(np.float64)
    t = np.array([truth.regression(a, b) for a, b in zip(ns, nd)])
    guess = _cost(k_sat=128.0)
    guess.b0 = guess.b1 = guess.b2 = guess.b3 = 0.0
    fit = core.cost_model_fit(ns, nd, t, guess)
    for k in ("b0", "b1", "b2", "b3"):
        assert getattr(fit, k) == pytest.approx(getattr(truth, k), rel=1e-6, abs=1e-15), k


def test_knee_threshold_matches_oracle(core):
    rng = np.random.default_rng(5)
    for _ in range(300):
        n = int(rng.integers(3, 20))
        counts = np.cumsum(rng.integers(1, 16, size=n)).astype(float)
        tput = np.cumsum(np.sort(rng.random(n))[::-1] * rng.choice([1, -0.2], size=n, p=[0.9, 0.1]))
        frac = float(rng.choice([0.05, 0.1, 0.3]))
        ref = OR.knee_threshold(list(zip(counts, tput)), frac=frac)
        assert core.knee_threshold(counts, tput, frac) == int(ref)


def test_plan_reallocation_and_choose_samples_match_oracle(core):
    rng = np.random.default_rng(6)
    for _ in range(500):
        G = int(rng.integers(1, 17))
        loads = [int(x) for x in rng.integers(0, 200, size=G)]
        thr = int(rng.integers(0, 200))
        assert core.plan_reallocation(loads, thr) == OR.plan_reallocation(loads, thr)
        n = int(rng.integers(0, 40))
        gid = rng.permutation(1000)[:n]
        sl = rng.integers(1, 20, size=n)                  # many ties on length
        aa = rng.integers(0, 4, size=n) / 2.0              # and on accepted tokens
        k = int(rng.integers(0, n + 1))
        ref = OR.choose_samples(list(zip(gid.tolist(), sl.tolist(), aa.tolist())), k)
        assert core.choose_samples(gid, sl, aa, k) == ref


def test_realloc_trigger_matches_oracle(core):
    """rs_realloc_should_trigger equals oracle.realloc.should_trigger on fuzzed fleets,
    including the cooldown boundary and fleets with nobody on one side of the threshold."""
    from oracle import realloc as OR
    rng = np.random.default_rng(17)
    for _ in range(400):
        G = int(rng.integers(1, 9))
        loads = rng.integers(0, 40, size=G).tolist()
        thr = int(rng.integers(0, 40))
        since, cd = int(rng.integers(0, 70)), int(rng.integers(0, 64))
        assert core.realloc_should_trigger(loads, thr, since, cd) == OR.should_trigger(loads, thr, since, cd)
    assert core.realloc_should_trigger([24, 1], 6, 32, 32) and not core.realloc_should_trigger([24, 1], 6, 31, 32)
    assert not core.realloc_should_trigger([6, 6], 6, 100, 32) and not core.realloc_should_trigger([], 6, 100, 32)


def test_page_pool_all_or_nothing(core):
    pool = core.PagePool(10)
    a = pool.alloc(4)
    assert sorted(a.tolist()) == [0, 1, 2, 3] and pool.free_count() == 6
    assert pool.alloc(7) is None and pool.free_count() == 6       # refused: nothing reserved
    rows = pool.reserve([65, 1, 0], page_size=64, max_pages=4)    # needs 2 + 1 + 0 pages
    assert rows is not None and pool.free_count() == 3
    assert len(set(rows[0, :2].tolist()) | {rows[1, 0]}) == 3
    assert set(rows[0, :2].tolist()).isdisjoint(a.tolist())
    assert pool.reserve([64 * 4], page_size=64, max_pages=4) is None and pool.free_count() == 3
    pool.free(a)
    assert pool.free_count() == 7
    with pytest.raises(core.RSError):
        pool.free(a[:1])                                           # double free
    with pytest.raises(core.RSError):
        pool.reserve([64 * 5], page_size=64, max_pages=4)          # longer than a block-table row


@pytest.mark.parametrize("seed", range(12))
def test_acceptance_fit_matches_oracle(core, seed):
    """rs_acceptance_fit (C++) vs oracle.strategy.fit_acceptance on random observations
    (0/1 outcomes or rates, clipped dl, few or many buckets)."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 4000))
    dl = rng.random(n) * 1.2 - 0.1
    acc = (rng.random(n) < np.clip(0.2 + 0.9 * dl, 0, 1)).astype(float) if seed % 2 else rng.random(n)
    K = int(rng.integers(1, 40))
    kx, ky = core.acceptance_fit(dl, acc, K)
    ox, oy = OS.fit_acceptance(dl, acc, K)
    np.testing.assert_allclose(kx, ox, rtol=0, atol=1e-12)
    np.testing.assert_allclose(ky, oy, rtol=0, atol=1e-12)
    with pytest.raises(core.RSError):
        core.acceptance_fit([0.4] * 5, [1, 0, 1, 0, 1], K)


def test_ctx_strategy_state(core):
    """rs_ctx keeps F and the cost model; a refit replaces F; invalid knots leave it unchanged;
    the ctx's selector gives the same result as a standalone selector with the same state."""
    ctx = core.Ctx(rank=0, world=1, page_size=64)
    with pytest.raises(core.RSError):
        ctx.select(np.zeros(1, np.int32), np.ones(1), np.array([0, 1], np.int32), np.array([10], np.int32))
    cost = _cost()
    ctx.set_strategy(cost, KX, KY)
    c, kx, ky = ctx.strategy()
    assert np.array_equal(kx, KX) and np.array_equal(ky, KY) and c["b1"] == cost.b1
    with pytest.raises(core.RSError):
        ctx.set_strategy(None, [0.0, 0.5, 0.4], [0.0, 0.5, 0.6])      # x not increasing
    assert np.array_equal(ctx.strategy()[1], KX)
    rng = np.random.default_rng(5)
    dl = rng.random(3000)
    ctx.fit_acceptance(dl, (rng.random(3000) < 0.2 + 0.7 * dl).astype(float), 10)
    _, kx2, ky2 = ctx.strategy()
    assert len(kx2) == 10 and np.all(np.diff(ky2) >= 0)
    trees = [make_candidate_tree(rng, 60) for _ in range(16)]
    off = np.zeros(17, np.int32)
    off[1:] = np.cumsum([len(p) for p, _ in trees])
    par = np.concatenate([p for p, _ in trees]).astype(np.int32)
    o = np.concatenate([q for _, q in trees]).astype(np.float64)
    pl = rng.integers(100, 4000, size=16).astype(np.int32)
    a = ctx.select(par, o, off, pl, n_min=2, n_max=30)
    b = core.Selector(cost, kx2, ky2).select_flat(par, o, off, pl, n_min=2, n_max=30)
    assert a == b
    ctx.destroy()


def test_draft_logits_matches_oracle(core):
    rng = np.random.default_rng(2)
    trees = [make_candidate_tree(rng, int(rng.integers(1, 90))) for _ in range(30)]
    off = np.zeros(31, np.int32)
    off[1:] = np.cumsum([len(p) for p, _ in trees])
    dl = core.draft_logits(np.concatenate([p for p, _ in trees]), np.concatenate([o for _, o in trees]), off)
    ref = np.concatenate([OS.draft_logits(p, o) for p, o in trees])
    assert np.array_equal(dl, ref)


def test_calibrate_validates_before_any_device_work(core):
    """rs_calibrate / rs_calibrate_workspace_bytes refuse a ctx without a registered LLM KV store,
    too few grid points and too small Q/O scratch — on the host, before touching the device."""
    import ctypes
    ctx = core.Ctx(0, 1, 64)
    ctx.set_strategy(_cost(), KX, KY)
    B = np.array([8, 8, 16, 16], np.int32)
    P = np.array([128, 256, 128, 256], np.int32)
    T = np.array([4, 8, 4, 8], np.int32)
    desc = core.CalibDescC(32, 4, B.ctypes.data, P.ctypes.data, T.ctypes.data, 2, None, None, 0, None, 0, 0.0, None)
    assert core._lib.rs_calibrate_workspace_bytes(ctx._h, ctypes.byref(desc)) == 0
    st = core._lib.rs_calibrate(ctx._h, ctypes.byref(desc), None)
    assert st == 1 and b"no LLM KV" in core._lib.rs_last_error()
    desc.n_points = 3
    assert core._lib.rs_calibrate(ctx._h, ctypes.byref(desc), None) == 1      # < 4 grid points
    ctx.destroy()
