"""Pins for oracle.attention (exact tree attention) against brute force and library routines."""
import numpy as np
import pytest
import torch

from oracle import attention as OA
from oracle import tree as OT
from synth import random_tree_parents


def _case(seed, B=3, Hq=4, Hkv=2, d=16, ps=8, prefixes=(0, 5, 70), sizes=(1, 9, 17)):
    rng = np.random.default_rng(seed)
    parents = [random_tree_parents(rng, T) for T in sizes]
    tree_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    P = np.asarray(prefixes, dtype=np.int32)
    npg = (P + np.asarray(sizes) + ps - 1) // ps
    num_pages = int(npg.sum()) + 3
    perm = rng.permutation(num_pages)
    bt = np.zeros((B, int(npg.max())), dtype=np.int32)
    o = 0
    for b in range(B):
        bt[b, :npg[b]] = perm[o:o + npg[b]]
        o += npg[b]
    K = rng.standard_normal((num_pages, Hkv, ps, d))
    V = rng.standard_normal((num_pages, Hkv, ps, d))
    q = rng.standard_normal((int(tree_off[-1]), Hq, d))
    par_all = np.concatenate(parents)
    mask, _, ok = OT.batch_masks(par_all, tree_off)
    assert ok.all()
    return dict(q=q, K=K, V=V, bt=bt, P=P, tree_off=tree_off, mask=mask, parents=parents,
                Hkv=Hkv, ps=ps, scale=1.0 / np.sqrt(d))


def _sdpa_one(qv, keys, vals, scale):
    """Library attention (torch SDPA, fp64) of one query over an explicit key sequence."""
    qt = torch.from_numpy(qv)[None, None, None, :]
    kt = torch.from_numpy(keys)[None, None]
    vt = torch.from_numpy(vals)[None, None]
    return torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, scale=scale)[0, 0, 0].numpy()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_path_decomposition_bruteforce(seed):
    """Row i of tree attention == plain attention over [prefix, Path(root, i)] (SDPA)."""
    c = _case(seed)
    o, lse = OA.tree_verify_attention(c["q"], c["K"], c["V"], c["bt"], c["P"], c["tree_off"],
                                      c["mask"], c["Hkv"], c["ps"], c["scale"])
    Hq = c["q"].shape[1]
    g = Hq // c["Hkv"]
    for b, par in enumerate(c["parents"]):
        P = int(c["P"][b])
        for i in range(len(par)):
            slots = list(range(P)) + [P + j for j in OT.ancestors_or_self(list(par), i)]
            pages = c["bt"][b][np.asarray(slots) // c["ps"]]
            rows = np.asarray(slots) % c["ps"]
            for h in range(Hq):
                kv = h // g
                keys = c["K"][pages, kv, rows, :]
                vals = c["V"][pages, kv, rows, :]
                qv = c["q"][c["tree_off"][b] + i, h]
                ref = _sdpa_one(qv, keys, vals, c["scale"])
                np.testing.assert_allclose(o[c["tree_off"][b] + i, h], ref, rtol=1e-10, atol=1e-12)
                s = torch.from_numpy(keys @ qv * c["scale"])
                np.testing.assert_allclose(lse[c["tree_off"][b] + i, h], torch.logsumexp(s, 0).item(),
                                           rtol=1e-12)


def test_single_node_tree_is_decode_attention():
    c = _case(5, B=1, prefixes=(37,), sizes=(1,))
    o, _ = OA.tree_verify_attention(c["q"], c["K"], c["V"], c["bt"], c["P"], c["tree_off"],
                                    c["mask"], c["Hkv"], c["ps"], c["scale"])
    slots = np.arange(38)
    pages, rows = c["bt"][0][slots // c["ps"]], slots % c["ps"]
    g = c["q"].shape[1] // c["Hkv"]
    # decode: every head attends to all 38 cached keys (SDPA over the whole cache, GQA expand)
    K = torch.from_numpy(c["K"][pages, :, rows, :]).permute(1, 0, 2).repeat_interleave(g, 0)
    V = torch.from_numpy(c["V"][pages, :, rows, :]).permute(1, 0, 2).repeat_interleave(g, 0)
    q = torch.from_numpy(c["q"][0])[:, None, :]
    ref = torch.nn.functional.scaled_dot_product_attention(q, K, V, scale=c["scale"])[:, 0]
    np.testing.assert_allclose(o[0], ref.numpy(), rtol=1e-10, atol=1e-12)


def test_chain_tree_is_causal_prefill():
    """A chain tree (each node the child of the previous) is causal attention with a prefix."""
    T, P, ps, d, Hkv, Hq = 12, 20, 8, 16, 2, 4
    rng = np.random.default_rng(3)
    par = np.arange(-1, T - 1, dtype=np.int32)
    npg = (P + T + ps - 1) // ps
    bt = rng.permutation(npg)[None].astype(np.int32)
    K = rng.standard_normal((npg, Hkv, ps, d))
    V = rng.standard_normal((npg, Hkv, ps, d))
    q = rng.standard_normal((T, Hq, d))
    mask = OT.ancestor_mask(list(par))
    o, _ = OA.tree_verify_attention(q, K, V, bt, np.array([P]), np.array([0, T]), mask, Hkv, ps,
                                    1 / np.sqrt(d))
    slots = np.arange(P + T)
    Ks = torch.from_numpy(K[bt[0][slots // ps], :, slots % ps, :]).permute(1, 0, 2).repeat_interleave(2, 0)
    Vs = torch.from_numpy(V[bt[0][slots // ps], :, slots % ps, :]).permute(1, 0, 2).repeat_interleave(2, 0)
    allowed = torch.ones(T, P + T, dtype=torch.bool)
    allowed[:, P:] = torch.tril(torch.ones(T, T, dtype=torch.bool))
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(q).permute(1, 0, 2), Ks, Vs, attn_mask=allowed, scale=1 / np.sqrt(d))
    np.testing.assert_allclose(o, ref.permute(1, 0, 2).numpy(), rtol=1e-10, atol=1e-12)


def test_gqa_equals_duplicated_kv_heads():
    c = _case(7)
    o, _ = OA.tree_verify_attention(c["q"], c["K"], c["V"], c["bt"], c["P"], c["tree_off"],
                                    c["mask"], c["Hkv"], c["ps"], c["scale"])
    g = c["q"].shape[1] // c["Hkv"]
    K2 = np.repeat(c["K"], g, axis=1)
    V2 = np.repeat(c["V"], g, axis=1)
    o2, _ = OA.tree_verify_attention(c["q"], K2, V2, c["bt"], c["P"], c["tree_off"], c["mask"],
                                     c["q"].shape[1], c["ps"], c["scale"])
    np.testing.assert_allclose(o, o2, rtol=1e-12, atol=1e-14)


def test_invisible_slots_do_not_matter_visible_ones_do():
    c = _case(11, B=1, prefixes=(13,), sizes=(17,))
    o, _ = OA.tree_verify_attention(c["q"], c["K"], c["V"], c["bt"], c["P"], c["tree_off"],
                                    c["mask"], c["Hkv"], c["ps"], c["scale"])
    par = list(c["parents"][0])
    P = 13
    leaf = len(par) - 1
    anc = set(OT.ancestors_or_self(par, leaf))
    for j in range(len(par)):
        K2, V2 = c["K"].copy(), c["V"].copy()
        s = P + j
        K2[c["bt"][0][s // c["ps"]], :, s % c["ps"], :] += 3.0
        V2[c["bt"][0][s // c["ps"]], :, s % c["ps"], :] -= 2.0
        o2, _ = OA.tree_verify_attention(c["q"], K2, V2, c["bt"], c["P"], c["tree_off"],
                                         c["mask"], c["Hkv"], c["ps"], c["scale"])
        changed = not np.allclose(o2[leaf], o[leaf], rtol=0, atol=1e-12)
        assert changed == (j in anc), j


def test_page_permutation_invariance():
    c = _case(13)
    o, _ = OA.tree_verify_attention(c["q"], c["K"], c["V"], c["bt"], c["P"], c["tree_off"],
                                    c["mask"], c["Hkv"], c["ps"], c["scale"])
    perm = np.random.default_rng(0).permutation(c["K"].shape[0])
    inv = np.argsort(perm)
    K2, V2 = c["K"][perm], c["V"][perm]          # page p of K2 is old page perm[p]
    bt2 = inv[c["bt"]].astype(np.int32)
    o2, _ = OA.tree_verify_attention(c["q"], K2, V2, bt2, c["P"], c["tree_off"], c["mask"],
                                     c["Hkv"], c["ps"], c["scale"])
    np.testing.assert_array_equal(o, o2)
