"""Pins for oracle.compact (KV commit) and oracle.migrate (pack/unpack layout)."""
import numpy as np
import torch

from oracle import attention as OA
from oracle import compact as OC
from oracle import migrate as OM
from oracle import tree as OT
from synth import random_tree_parents


def _cache_case(seed, B=4, L=2, Hkv=2, d=8, ps=4):
    rng = np.random.default_rng(seed)
    T = rng.integers(2, 20, size=B)
    P = rng.integers(0, 30, size=B)
    parents = [random_tree_parents(rng, int(t)) for t in T]
    npg = (P + T + ps - 1) // ps
    num_pages = int(npg.sum()) + 2
    perm = rng.permutation(num_pages)
    bt = np.zeros((B, int(npg.max())), dtype=np.int32)
    o = 0
    for b in range(B):
        bt[b, :npg[b]] = perm[o:o + npg[b]]
        o += npg[b]
    caches = [rng.integers(0, 2**16, size=(num_pages, Hkv, ps, d)).astype(np.uint16)
              for _ in range(2 * L)]
    # an accepted path per sample: a random root-to-node path
    acc = np.zeros(B, np.int32)
    path = np.full((B, 64), -1, np.int32)
    for b in range(B):
        node = int(rng.integers(0, T[b]))
        pth = OT.ancestors_or_self(list(parents[b]), node)
        acc[b] = len(pth) - 1
        path[b, :len(pth)] = pth
    return dict(P=P, T=T, parents=parents, bt=bt, caches=caches, acc=acc, path=path, ps=ps)


def test_compact_equals_gather_then_scatter():
    for seed in range(10):
        c = _cache_case(seed)
        ref = [x.copy() for x in c["caches"]]
        # independent formulation: gather every source row first, then write all destinations
        for b in range(len(c["P"])):
            P, a = int(c["P"][b]), int(c["acc"][b])
            srcs = [P + int(c["path"][b, k]) for k in range(1, a + 1)]
            for cache in ref:
                rows = [cache[c["bt"][b][s // c["ps"]], :, s % c["ps"], :].copy() for s in srcs]
                for k, row in enumerate(rows, start=1):
                    dst = P + k
                    cache[c["bt"][b][dst // c["ps"]], :, dst % c["ps"], :] = row
        new_len, moves = OC.kv_compact(c["caches"], c["bt"], c["P"], c["acc"], c["path"], c["ps"])
        for x, y in zip(c["caches"], ref):
            np.testing.assert_array_equal(x, y)
        np.testing.assert_array_equal(new_len, c["P"] + 1 + c["acc"])
        for b in range(len(c["P"])):
            a = c["acc"][b]
            assert np.all(moves[b, a:] == -1)
            assert [tuple(m) for m in moves[b, :a]] == [(c["P"][b] + c["path"][b, k], c["P"][b] + k)
                                                        for k in range(1, a + 1)]


def test_compact_identity_path_changes_nothing():
    c = _cache_case(3)
    for b in range(len(c["P"])):
        a = min(int(c["T"][b]) - 1, 5)
        chain = list(range(a + 1))
        c["acc"][b] = a
        c["path"][b, :] = -1
        c["path"][b, :a + 1] = chain
    before = [x.copy() for x in c["caches"]]
    OC.kv_compact(c["caches"], c["bt"], c["P"], c["acc"], c["path"], c["ps"])
    for x, y in zip(c["caches"], before):
        np.testing.assert_array_equal(x, y)


def test_markov_invariant_decode_after_compaction():
    """after commit, decode attention of the last accepted node over the compacted
    cache equals its tree-attention row before compaction."""
    rng = np.random.default_rng(12)
    ps, Hkv, Hq, d, P, T = 8, 2, 4, 16, 21, 24
    par = random_tree_parents(rng, T)
    npg = (P + T + ps - 1) // ps
    bt = rng.permutation(npg)[None].astype(np.int32)
    K = rng.standard_normal((npg, Hkv, ps, d))
    V = rng.standard_normal((npg, Hkv, ps, d))
    q = rng.standard_normal((T, Hq, d))
    mask = OT.ancestor_mask(list(par))
    o, _ = OA.tree_verify_attention(q, K, V, bt, [P], [0, T], mask, Hkv, ps, 1 / np.sqrt(d))
    leaf = T - 1
    pth = OT.ancestors_or_self(list(par), leaf)
    a = len(pth) - 1
    path = np.full((1, 64), -1, np.int32)
    path[0, :a + 1] = pth
    K2, V2 = K.copy(), V.copy()
    new_len, _ = OC.kv_compact([K2, V2], bt, [P], [a], path, ps)
    n = int(new_len[0])
    slots = np.arange(n)
    g = Hq // Hkv
    Ks = torch.from_numpy(K2[bt[0][slots // ps], :, slots % ps, :]).permute(1, 0, 2).repeat_interleave(g, 0)
    Vs = torch.from_numpy(V2[bt[0][slots // ps], :, slots % ps, :]).permute(1, 0, 2).repeat_interleave(g, 0)
    dec = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(q[leaf])[:, None, :], Ks, Vs, scale=1 / np.sqrt(d))[:, 0]
    np.testing.assert_allclose(o[leaf], dec.numpy(), rtol=1e-10, atol=1e-12)


# ---------------------------------------------------------------- migrate
def test_segment_order_spec_example():
    """SSM 1 layer + LLM 32 layers x 10 tokens -> 33 segments, SSM first."""
    segs, total = OM.segment_table([(1, 1, 64), (32, 8, 128)], [10])
    assert len(segs) == 33
    assert segs[0][:3] == (0, 0, 0) and all(s[0] == 1 for s in segs[1:])
    assert [s[1] for s in segs[1:]] == list(range(32))
    assert total == 2 * (1 * 10 * 64 + 32 * 8 * 10 * 128)
    offs = [s[3] for s in segs]
    assert offs == sorted(offs) and all(s[3] + s[4] == t[3] for s, t in zip(segs, segs[1:]))


def test_pack_unpack_round_trip_bytes():
    rng = np.random.default_rng(0)
    ps = 4
    models = [(1, 1, 8), (3, 2, 8)]
    for trial in range(20):
        lens = list(rng.integers(0, 13, size=int(rng.integers(1, 4))))
        need = [(n + ps - 1) // ps for n in lens]
        src_pages, dst_pages = 40, 50
        sp = rng.permutation(src_pages)
        dp = rng.permutation(dst_pages)
        cuts = np.concatenate([[0], np.cumsum(need)])
        src_bt = [sp[cuts[i]:cuts[i + 1]] for i in range(len(need))]
        dst_bt = [dp[cuts[i]:cuts[i + 1]] for i in range(len(need))]
        src = [[(rng.integers(0, 2**16, size=(src_pages, H, ps, d)).astype(np.uint16),
                 rng.integers(0, 2**16, size=(src_pages, H, ps, d)).astype(np.uint16))
                for _ in range(L)] for (L, H, d) in models]
        dst = [[(np.zeros((dst_pages, H, ps, d), np.uint16), np.zeros((dst_pages, H, ps, d), np.uint16))
                for _ in range(L)] for (L, H, d) in models]
        buf = OM.pack(src, src_bt, lens, ps)
        _, total = OM.segment_table(models, lens)
        assert buf.size == total
        used = OM.unpack(buf, dst, dst_bt, lens, ps)
        assert used == total
        for m in range(len(models)):
            for l in range(models[m][0]):
                for t in range(2):
                    for s, n in enumerate(lens):
                        for j in range(n):
                            a = src[m][l][t][src_bt[s][j // ps], :, j % ps, :]
                            b = dst[m][l][t][dst_bt[s][j // ps], :, j % ps, :]
                            np.testing.assert_array_equal(a, b)


def test_two_stage_ranges_compose():
    """Two-stage migration: stage 1 carries tokens [0, a), stage 2 tokens [a, b)
    (verified on the source meanwhile). Both buffers use the one-shot layout restricted to the
    range, and unpacking both reproduces the one-shot migration of [0, b) byte for byte; a
    buffer's segment (model, layer, sample, K|V, head) is exactly the one-shot segment's token
    range."""
    rng = np.random.default_rng(3)
    ps = 4
    models = [(1, 1, 8), (2, 2, 8)]
    for trial in range(15):
        ns = int(rng.integers(1, 4))
        b_len = [int(x) for x in rng.integers(1, 15, size=ns)]
        a_len = [int(rng.integers(0, x + 1)) for x in b_len]
        need = [(n + ps - 1) // ps for n in b_len]
        cuts = np.concatenate([[0], np.cumsum(need)])
        sp, dp = rng.permutation(40), rng.permutation(40)
        src_bt = [sp[cuts[i]:cuts[i + 1]] for i in range(ns)]
        dst_bt = [dp[cuts[i]:cuts[i + 1]] for i in range(ns)]
        src = [[(rng.integers(0, 2**16, size=(40, H, ps, d)).astype(np.uint16),
                 rng.integers(0, 2**16, size=(40, H, ps, d)).astype(np.uint16)) for _ in range(L)]
               for (L, H, d) in models]
        zero = lambda: [[(np.zeros((40, H, ps, d), np.uint16), np.zeros((40, H, ps, d), np.uint16))
                         for _ in range(L)] for (L, H, d) in models]
        one, two = zero(), zero()
        OM.unpack(OM.pack(src, src_bt, b_len, ps), one, dst_bt, b_len, ps)
        delta = [b - a for a, b in zip(a_len, b_len)]
        buf1 = OM.pack(src, src_bt, a_len, ps)
        buf2 = OM.pack(src, src_bt, delta, ps, starts=a_len)
        assert buf1.size + buf2.size == OM.segment_table(models, b_len)[1]
        OM.unpack(buf1, two, dst_bt, a_len, ps)
        OM.unpack(buf2, two, dst_bt, delta, ps, starts=a_len)
        for m in range(len(models)):
            for l in range(models[m][0]):
                for t in range(2):
                    np.testing.assert_array_equal(one[m][l][t], two[m][l][t])
        # segment check: first segment of buf2 = tokens [a, b) of head 0.. of sample 0, K, SSM layer 0
        H, d = models[0][1], models[0][2]
        full = OM.pack(src, src_bt, b_len, ps)
        segK = full[:H * b_len[0] * d].reshape(H, b_len[0], d)
        np.testing.assert_array_equal(buf2[:H * delta[0] * d].reshape(H, delta[0], d), segK[:, a_len[0]:, :])
