"""Pins for oracle.tree (ancestor masks) by brute-force path enumeration."""
import numpy as np

from oracle import tree as OT
from synth import TINY_PARENT, random_tree_parents


def _brute_mask(parent):
    """Bit j of mask[i] <=> j is reachable from i by following parent links (incl. i)."""
    T = len(parent)
    out = []
    for i in range(T):
        bits = 0
        for j in range(T):
            x = i
            while x != -1 and x != j:
                x = parent[x]
            if x == j:
                bits |= 1 << j
        out.append(bits)
    return out


def test_tiny_tree_masks_and_paths():
    m = OT.ancestor_mask(TINY_PARENT)
    # SURVEY tiny config: root-to-leaf paths [0,1,3,6], [0,1,4,7], [0,2,5]
    assert OT.ancestors_or_self(TINY_PARENT, 6) == [0, 1, 3, 6]
    assert OT.ancestors_or_self(TINY_PARENT, 7) == [0, 1, 4, 7]
    assert OT.ancestors_or_self(TINY_PARENT, 5) == [0, 2, 5]
    assert int(m[6]) == (1 << 0) | (1 << 1) | (1 << 3) | (1 << 6)
    assert list(OT.depths(TINY_PARENT)) == [0, 1, 1, 2, 2, 2, 3, 3]


def test_masks_match_bruteforce_on_random_trees():
    rng = np.random.default_rng(0)
    for T in [1, 2, 5, 16, 33, 64]:
        for _ in range(5):
            par = list(random_tree_parents(rng, T))
            assert OT.validate(par)
            assert [int(x) for x in OT.ancestor_mask(par)] == _brute_mask(par)


def test_chain_of_64_sets_top_bit():
    par = list(range(-1, 63))
    m = OT.ancestor_mask(par)
    assert int(m[63]) == (1 << 64) - 1


def test_validate_rejects_malformed():
    assert not OT.validate([])
    assert not OT.validate([0])
    assert not OT.validate([-1, 1])
    assert not OT.validate([-1, 0, 3, 1])
    assert not OT.validate([-1] + [0] * 64)     # 65 nodes
    assert OT.validate([-1] + [0] * 63)
