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
