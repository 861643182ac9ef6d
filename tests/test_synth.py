"""Input generators: structure checks (no method arithmetic involved)."""
import numpy as np

from oracle import tree as OT
from synth import CONFIGS, VerifyConfig, make_verify_batch, random_tree_parents


def test_random_trees_are_bfs_ordered_and_valid():
    rng = np.random.default_rng(0)
    for T in range(1, 65):
        p = random_tree_parents(rng, T)
        assert OT.validate(list(p))
        assert np.all(np.diff(p[1:]) >= 0)         # BFS order


def test_tiny_batch_shapes_and_pages():
    b = make_verify_batch(CONFIGS["tiny"])
    assert b["NT"] == 8 and b["q"].shape == (1, 8, 1, 64)
    assert b["k_cache"].shape[1:] == (b["num_pages"], 1, 64, 64)
    assert b["logits"].shape == (8, 1000)
    used = set()
    for bb in range(b["B"]):
        n = (b["prefix_len"][bb] + b["T"][bb] + 63) // 64
        pages = set(int(x) for x in b["block_table"][bb, :n])
        assert len(pages) == n and not (pages & used)
        used |= pages


def test_sampling_batch_children_drawn_from_q():
    cfg = VerifyConfig("t", B=4, Hq=2, Hkv=1, d=64, V=50, L=1, prefix=("fixed", 10),
                       tree=("fixed", 12), mode="mss", seed=3)
    b = make_verify_batch(cfg)
    assert b["draft_probs"].shape == (b["NT"], 50)
    np.testing.assert_allclose(b["draft_probs"].sum(-1).numpy(), 1.0, rtol=1e-5)


def test_lm_head_sampling_inputs_shapes_and_draws():
    """synth.make_lm_head_sampling_inputs: seeded (same seed -> same tensors), draft rows are
    probability vectors, every child's token lies in the support of its parent's q, root tokens
    are kept."""
    import torch
    from synth import VerifyConfig, make_lm_head_sampling_inputs, make_verify_batch
    cfg = VerifyConfig("ls", B=3, Hq=2, Hkv=1, d=64, V=48, L=1, prefix=("fixed", 5), tree=("range", 2, 9),
                       mode="mss", seed=2)
    b = make_verify_batch(cfg, device="cpu", with_logits=False)
    a = make_lm_head_sampling_inputs(b, Dm=64, seed=3)
    c = make_lm_head_sampling_inputs(b, Dm=64, seed=3)
    assert a["hidden"].shape == (b["NT"], 64) and a["weight"].shape == (48, 64)
    assert torch.equal(a["hidden"], c["hidden"]) and torch.equal(a["draft_probs"], c["draft_probs"])
    assert np.array_equal(a["token"], c["token"])
    q = a["draft_probs"].float()
    assert torch.all(q >= 0) and torch.allclose(q.sum(-1), torch.ones(b["NT"]), atol=1e-5)
    par, off = b["parent"], b["tree_off"]
    for s in range(b["B"]):
        o = off[s]
        assert a["token"][o] == b["token"][o]
        for i in range(1, off[s + 1] - o):
            assert 0 <= a["token"][o + i] < 48 and q[o + par[o + i], a["token"][o + i]] > 0
