"""f3 on the GPU: rs_tree_select (verification trees from candidate trees for a chosen n) vs the
oracle (oracle/strategy.verification_tree + oracle/tree masks), bit-exact, on config-3-shaped
candidate trees (96 nodes, SPEC S:304 shape) and the edge cases."""
import numpy as np
import pytest
import torch

from oracle import strategy as OS
from oracle import tree as OT
from synth import make_candidate_tree

pytestmark = pytest.mark.gpu

KX = [0.0, 0.05, 0.2, 0.5, 1.0]
KY = [0.0, 0.15, 0.45, 0.75, 0.95]


def _cands(B, N, seed):
    rng = np.random.default_rng(seed)
    trees = [make_candidate_tree(rng, int(N if np.isscalar(N) else rng.integers(*N))) for _ in range(B)]
    toks = [rng.integers(0, 128256, size=len(p)).astype(np.int32) for p, _ in trees]
    off = np.concatenate([[0], np.cumsum([len(p) for p, _ in trees])]).astype(np.int32)
    root = rng.integers(0, 128256, size=B).astype(np.int32)
    return trees, toks, off, root


def _run(core, trees, toks, off, root, n):
    d = lambda x, dt: torch.as_tensor(np.ascontiguousarray(x)).to(dt).cuda()
    par = d(np.concatenate([p for p, _ in trees]), torch.int32)
    o = d(np.concatenate([q for _, q in trees]), torch.float64)
    tok = d(np.concatenate(toks), torch.int32)
    out = core.tree_select(par, o, tok, d(off, torch.int32), d(root, torch.int32), n, d(KX, torch.float64),
                           d(KY, torch.float64))
    torch.cuda.synchronize()
    return [x.cpu().numpy() for x in out]


@pytest.mark.parametrize("n", [1, 5, 17, 40, 63])
def test_tree_select_matches_oracle(cuda_lib, n):
    trees, toks, off, root = _cands(256, 96, seed=n)
    par, tok, mask, dep, flags = _run(cuda_lib, trees, toks, off, root, n)
    T = n + 1
    for b, (p, o) in enumerate(trees):
        pv, tv = OS.verification_tree(p, o, toks[b], root[b], n, KX, KY)
        sl = slice(b * T, (b + 1) * T)
        np.testing.assert_array_equal(par[sl], pv)
        np.testing.assert_array_equal(tok[sl], tv)
        np.testing.assert_array_equal(mask[sl].view(np.uint64), OT.ancestor_mask(pv))
        np.testing.assert_array_equal(dep[sl], OT.depths(pv))
    assert not flags.any()


def test_tree_select_ragged_and_flags(cuda_lib):
    """Ragged candidate counts (2..200), a malformed sample and one with too few nodes."""
    n = 12
    trees, toks, off, root = _cands(40, (2, 200), seed=5)
    trees[3] = (np.array([-1, 2, 0], np.int32), np.array([0.5, 0.5, 0.5]))      # parent 2 of node 1: not topological
    toks[3] = np.array([1, 2, 3], np.int32)
    off = np.concatenate([[0], np.cumsum([len(p) for p, _ in trees])]).astype(np.int32)
    par, tok, mask, dep, flags = _run(cuda_lib, trees, toks, off, root, n)
    T = n + 1
    for b, (p, o) in enumerate(trees):
        sl = slice(b * T, (b + 1) * T)
        if b == 3:
            assert flags[b] == cuda_lib.FLAG_MALFORMED
            continue
        try:
            pv, tv = OS.verification_tree(p, o, toks[b], root[b], n, KX, KY)
        except ValueError:                                    # InsufficientNodes
            assert flags[b] == cuda_lib.FLAG_INSUFFICIENT
            k = len(OS.layer_search_order(p, [OS.acceptance_fit(KX, KY, x) for x in OS.draft_logits(p, o)], n))
            assert (tok[sl][k + 1:] == -1).all() and (par[sl][k + 1:] == 0).all()
            continue
        assert flags[b] == 0
        np.testing.assert_array_equal(par[sl], pv)
        np.testing.assert_array_equal(tok[sl], tv)


def test_tree_select_invalid_knots_and_probabilities(cuda_lib):
    """Knots that do not make F monotone flag every sample MALFORMED (device check); an o(u)
    outside [0, 1] or NaN flags its own sample only. The oracle raises MalformedTree for both."""
    core = cuda_lib
    n = 8
    trees, toks, off, root = _cands(8, 40, seed=9)
    bad_o = trees[2][1].copy()
    bad_o[5] = 1.25
    trees[2] = (trees[2][0], bad_o)
    nan_o = trees[6][1].copy()
    nan_o[0] = np.nan
    trees[6] = (trees[6][0], nan_o)
    _, _, _, _, flags = _run(core, trees, toks, off, root, n)
    assert list(np.nonzero(flags)[0]) == [2, 6] and flags[2] == core.FLAG_MALFORMED
    for b in (2, 6):
        with pytest.raises(ValueError, match="MalformedTree"):
            OS.verification_tree(trees[b][0], trees[b][1], toks[b], root[b], n, KX, KY)
    d = lambda x, dt: torch.as_tensor(np.ascontiguousarray(x)).to(dt).cuda()
    trees, toks, off, root = _cands(8, 40, seed=10)
    par = d(np.concatenate([p for p, _ in trees]), torch.int32)
    o = d(np.concatenate([q for _, q in trees]), torch.float64)
    tok = d(np.concatenate(toks), torch.int32)
    for kx, ky in (([0.0, 0.5, 0.5, 1.0], [0.0, 0.2, 0.4, 0.9]), ([0.0, 0.5, 1.0], [0.0, 0.6, 0.4])):
        out = core.tree_select(par, o, tok, d(off, torch.int32), d(root, torch.int32), n, d(kx, torch.float64),
                               d(ky, torch.float64))
        assert (out[4].cpu().numpy() == core.FLAG_MALFORMED).all()
