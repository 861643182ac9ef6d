"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): attention max-abs <= 2e-2 and rel-L2 <= 5e-3 vs the fp64
oracle (Z16); acceptance lengths/paths/bonus, compaction bytes/moves, masks, Philox and
exp_spec bit-exact."""
import math

import numpy as np
import pytest
import torch

from oracle import accept as OAcc
from oracle import attention as OA
from oracle import compact as OC
from oracle import tree as OT
from synth import CONFIGS, VerifyConfig, make_verify_batch, random_tree_parents
from tests.helpers import tensor_bf16_bits

pytestmark = pytest.mark.gpu

ATOL, RTOL_L2 = 2e-2, 5e-3


def _dev(x, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(x))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


# ------------------------------------------------------------------ a1 tree masks
def test_tree_mask_matches_oracle(cuda_lib):
    core = cuda_lib
    rng = np.random.default_rng(0)
    sizes = [1, 2, 8, 16, 33, 64] + list(rng.integers(1, 65, size=50))
    parents = [random_tree_parents(rng, int(T)) for T in sizes]
    parents[3] = parents[3].copy(); parents[3][5] = 7          # malformed (parent >= i)
    parents[4] = parents[4].copy(); parents[4][0] = 0          # malformed root
    tree_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    par = np.concatenate(parents).astype(np.int32)
    mask, depth, flags = core.tree_build_mask(_dev(par), _dev(tree_off))
    om, od, ok = OT.batch_masks(par, tree_off)
    np.testing.assert_array_equal(mask.cpu().numpy().view(np.uint64), om)
    np.testing.assert_array_equal(depth.cpu().numpy(), od)
    np.testing.assert_array_equal(flags.cpu().numpy(), np.where(ok, 0, core.FLAG_MALFORMED))


# ------------------------------------------------------------------ RNG / exp_spec
def test_philox_device_bit_exact(cuda_lib):
    core = cuda_lib
    rng = np.random.default_rng(1)
    ctr = rng.integers(0, 2**32, size=(4096, 4), dtype=np.uint64).astype(np.uint32)
    ctr[0] = 0
    ctr[1] = 0xFFFFFFFF
    key = [0xA4093822, 0x299F31D0]
    out = core.philox4x32_10(_dev(ctr.view(np.int32)), key).cpu().numpy().view(np.uint32)
    for i in range(0, 4096, 97):
        assert list(out[i]) == list(OAcc.philox4x32_10(ctr[i], key))


def test_exp_spec_device_bit_exact_exhaustive(cuda_lib):
    """SURVEY 8(c) pin: EVERY fp32 value in [-32, 0] (bit patterns 0x80000000 .. 0xC2000000,
    1.107e9 values, -0 included) gives the same bits on the GPU as in the C oracle; plus the
    values just below -32 (both return 0), +0 and NaN. The oracle runs in threads over slices
    (ctypes releases the GIL); the comparison is on the device."""
    import concurrent.futures as cf
    import os
    core = cuda_lib
    lo, hi = 0x80000000, int(np.float32(-32.0).view(np.uint32))
    chunk = 1 << 26
    nthr = max(1, min(32, os.cpu_count() or 1))
    ex = cf.ThreadPoolExecutor(nthr)

    def oracle(bits):
        x = bits.view(np.float32)
        y = np.empty_like(x)
        parts = np.array_split(np.arange(x.size), nthr)
        def run(ix):
            if ix.size:
                y[ix[0]:ix[-1] + 1] = OAcc.exp_spec_array(x[ix[0]:ix[-1] + 1])
        list(ex.map(run, parts))
        return y
    checked = 0
    for start in range(lo, hi + 1, chunk):
        end = min(start + chunk, hi + 1)
        bits = np.arange(start, end, dtype=np.uint64).astype(np.uint32)
        y_ref = torch.from_numpy(oracle(bits).view(np.int32)).cuda()
        y = core.exp_spec(torch.from_numpy(bits.view(np.float32)).cuda())
        neq = int((y.view(torch.int32) != y_ref).sum().item())
        assert neq == 0, (hex(start), neq)
        checked += end - start
    assert checked == hi - lo + 1 == 1107296257
    edge = np.array([-32.000004, -33.0, -88.0, -1e30, 0.0, np.nan], np.float32)
    y = core.exp_spec(_dev(edge)).cpu().numpy()
    np.testing.assert_array_equal(y.view(np.uint32), OAcc.exp_spec_array(edge).view(np.uint32))


# ------------------------------------------------------------------ a3 accept
def _accept_case(cfg, with_bad=False):
    b = make_verify_batch(cfg, device="cpu", layers=1)
    logits = b["logits"]
    if with_bad:
        logits = logits.clone()
        logits[b["tree_off"][1], 5] = float("nan")          # sample 1 root row non-finite
    return b, logits


def _run_accept_both(core, b, logits, mode, temperature=1.0, seed=11, step=3, parent=None):
    parent = b["parent"] if parent is None else parent
    dp = b["draft_probs"]
    g = core.tree_accept(mode, logits.cuda(), _dev(parent), _dev(b["token"]), _dev(b["tree_off"]),
                         _dev(b["gid"]), draft_probs=None if dp is None else dp.cuda(),
                         temperature=temperature, seed=seed, step=step)
    g = [x.cpu().numpy() for x in g]
    lg = tensor_bf16_bits(logits) if logits.dtype == torch.bfloat16 else logits.numpy()
    o = OAcc.tree_accept(mode, lg, parent, b["token"], b["tree_off"], b["gid"], b["V"],
                         draft_probs=None if dp is None else dp.float().numpy(), temperature=temperature,
                         seed=seed, step=step)
    return g, o


@pytest.mark.parametrize("cfgname", ["tiny", "greedy_ragged", "greedy_bigV"])
def test_accept_greedy_bit_exact(cuda_lib, cfgname):
    core = cuda_lib
    if cfgname == "tiny":
        cfg = CONFIGS["tiny"]
    elif cfgname == "greedy_ragged":
        cfg = VerifyConfig("g", B=40, Hq=4, Hkv=1, d=64, V=1000, L=1, prefix=("fixed", 5),
                           tree=("range", 1, 64), mode="greedy", p_accept=0.85, seed=4)
    else:
        cfg = VerifyConfig("g2", B=6, Hq=4, Hkv=1, d=64, V=128256, L=1, prefix=("fixed", 5),
                           tree=("range", 8, 32), mode="greedy", p_accept=0.9, seed=5)
    b, logits = _accept_case(cfg, with_bad=(cfgname == "greedy_ragged"))
    g, o = _run_accept_both(core, b, logits, core.GREEDY)
    for x, y in zip(g, o):
        np.testing.assert_array_equal(x, y)
    # fp32 logits and a malformed tree
    par = b["parent"].copy()
    if b["B"] > 2:
        par[b["tree_off"][2]] = 0
    g, o = _run_accept_both(core, b, logits.float(), core.GREEDY, parent=par)
    for x, y in zip(g, o):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("mode,V,temp,qdt", [("delta", 1000, 1.0, "f32"), ("mss", 1000, 1.0, "f32"),
                                             ("mss", 1000, 0.7, "f32"), ("mss", 1000, 1.0, "bf16"),
                                             ("delta", 128256, 1.0, "f32"), ("mss", 128256, 1.3, "f32"),
                                             ("mss", 128256, 1.0, "bf16"), ("mss", 1003, 1.0, "bf16")])
def test_accept_sampling_bit_exact(cuda_lib, mode, V, temp, qdt):
    """DELTA / MSS vs the oracle, bit for bit; bf16 draft rows (rs_tree_accept_ex) against the
    oracle fed the same values as fp32 (V = 1003: rows not 16-byte aligned, the scalar path)."""
    core = cuda_lib
    B = 24 if V < 5000 else 4
    cfg = VerifyConfig("s", B=B, Hq=4, Hkv=1, d=64, V=V, L=1, prefix=("fixed", 5), tree=("range", 2, 40),
                       mode=mode, seed=7 + V % 13, draft_dtype=qdt)
    b, logits = _accept_case(cfg)
    m = core.SAMPLE_DELTA if mode == "delta" else core.SAMPLE_MSS
    for step in range(3):
        g, o = _run_accept_both(core, b, logits, m, temperature=temp, seed=1234 + step, step=step)
        for x, y in zip(g, o):
            np.testing.assert_array_equal(x, y)
    if mode == "mss":   # fp32 logits with the same draft rows (the other logits-dtype instance)
        g, o = _run_accept_both(core, b, logits.float(), m, temperature=temp, seed=99, step=7)
        for x, y in zip(g, o):
            np.testing.assert_array_equal(x, y)


def _accept_np_both(core, mode, logits_f32, parent, token, tree_off, gid, V, draft=None, seed=0, step=0):
    """One call on each side with plain numpy inputs (bf16 logits)."""
    lg = torch.as_tensor(np.asarray(logits_f32, np.float32)).to(torch.bfloat16)
    g = core.tree_accept(mode, lg.cuda(), _dev(np.asarray(parent, np.int32)), _dev(np.asarray(token, np.int32)),
                         _dev(np.asarray(tree_off, np.int32)), _dev(np.asarray(gid, np.int64)),
                         draft_probs=None if draft is None else _dev(np.asarray(draft, np.float32)),
                         seed=seed, step=step)
    g = [x.cpu().numpy() for x in g]
    o = OAcc.tree_accept(mode, tensor_bf16_bits(lg), parent, token, tree_off, gid, V,
                         draft_probs=draft, seed=seed, step=step)
    return g, o


def test_accept_degenerate_residual_gpu(cuda_lib):
    """The MSS all-zero-residual fallback (pre-rejection weights kept) on the GPU, bit-exact vs
    the oracle, on the two pinned constructions of tests/test_oracle_accept.py (draft mass 0;
    q exactly proportional to p), batched over gids, at a small and the full vocabulary."""
    core = cuda_lib
    for V in (16, 128256):
        support = [1, 3, 4, 6]
        n = 24
        l = np.full((4, V), -100.0, np.float32)
        l[:, support] = 0.0
        l[3] = -100.0
        l[3, 5] = 0.0
        q0 = np.zeros((4, V), np.float32)
        qp = np.zeros((4, V), np.float32)
        qp[:, support] = 0.25
        par1 = np.tile(np.array([-1, 0, 0, 0], np.int32), n)
        tok1 = np.tile(np.array([0, 9, 11, 3], np.int32), n)
        off = (np.arange(n + 1) * 4).astype(np.int32)
        # both drafts: the two out-of-support children are rejected with an all-zero residual, the
        # kept weights accept the in-support child (q0: qw_x = 0, w_x > 0; qp: certain), bonus 5
        for q in (q0, qp):
            g, o = _accept_np_both(core, core.SAMPLE_MSS, np.tile(l, (n, 1)), par1, tok1, off, np.arange(n), V,
                                   draft=np.tile(q, (n, 1)), seed=77, step=5)
            for x, y in zip(g, o):
                np.testing.assert_array_equal(x, y)
            assert np.all(g[0] == 1) and np.all(g[1][:, 1] == 3) and np.all(g[2] == 5) and np.all(g[3] == 0)
        # q0 without the in-support child: nothing accepted, bonus from the ORIGINAL p (support)
        par3, tok3 = np.tile(np.array([-1, 0, 0], np.int32), n), np.tile(np.array([0, 9, 11], np.int32), n)
        off3 = (np.arange(n + 1) * 3).astype(np.int32)
        l3 = np.tile(l[:3], (n, 1))
        g, o = _accept_np_both(core, core.SAMPLE_MSS, l3, par3, tok3, off3, np.arange(n), V,
                               draft=np.tile(q0[:3], (n, 1)), seed=1, step=2)
        for x, y in zip(g, o):
            np.testing.assert_array_equal(x, y)
        assert np.all(g[0] == 0) and np.isin(g[2], support).all() and np.all(g[3] == 0)


def test_accept_mss_invalid_draft_rows_gpu(cuda_lib):
    """MSS: a visited node whose draft row holds a value outside [0, 1] or NaN is flagged
    NONFINITE (walk stops, bonus -1) exactly as in the oracle; unvisited bad rows are ignored."""
    core = cuda_lib
    V, n = 128256, 12
    rng = np.random.default_rng(8)
    par = np.tile(np.array([-1, 0, 1, 0], np.int32), n)
    tok = np.tile(np.array([0, 2, 3, 7], np.int32), n)
    off = (np.arange(n + 1) * 4).astype(np.int32)
    l = rng.standard_normal((4 * n, V)).astype(np.float32)
    l[0::4, 2] = 40.0
    q = np.full((4 * n, V), 1.0 / V, np.float32)
    for s_ in range(n):
        r = 4 * s_ + (1 if s_ % 3 else 3)          # node 1 (visited) or node 3 (never visited)
        q[r, rng.integers(V)] = [1.5, -0.5, np.nan][s_ % 3]
    g, o = _accept_np_both(core, core.SAMPLE_MSS, l, par, tok, off, np.arange(n), V, draft=q, seed=4, step=2)
    for x, y in zip(g, o):
        np.testing.assert_array_equal(x, y)
    assert (g[3][1::3] == core.FLAG_NONFINITE).all() and (g[3][0::3] == 0).all()


def test_accept_out_of_vocabulary_token_gpu(cuda_lib):
    """A draft token outside [0, V) flags the sample MALFORMED in every mode (no row is indexed
    by it); other samples of the batch are unaffected."""
    core = cuda_lib
    V = 1000
    rng = np.random.default_rng(5)
    n = 6
    par = np.tile(np.array([-1, 0, 0, 1], np.int32), n)
    tok = rng.integers(0, V, size=4 * n).astype(np.int32)
    tok[4 * 1 + 2] = -1
    tok[4 * 3 + 3] = V
    tok[4 * 4 + 0] = -1                      # the root's token is never tested
    off = (np.arange(n + 1) * 4).astype(np.int32)
    l = rng.standard_normal((4 * n, V)).astype(np.float32)
    q = np.asarray(torch.softmax(torch.randn(4 * n, V), -1).numpy(), np.float32)
    for mode in (core.GREEDY, core.SAMPLE_DELTA, core.SAMPLE_MSS):
        g, o = _accept_np_both(core, mode, l, par, tok, off, np.arange(n), V,
                               draft=q if mode == core.SAMPLE_MSS else None, seed=9, step=1)
        for x, y in zip(g, o):
            np.testing.assert_array_equal(x, y)
        assert list(g[3]) == [0, 1, 0, 1, 0, 0]


def test_accept_sampling_distribution_gpu(cuda_lib):
    """1e6 trials on the GPU: the first emitted token follows the target softmax."""
    from tests.helpers import bits_to_f32, chi2_pvalue, softmax64
    core = cuda_lib
    rng = np.random.default_rng(3)
    V, n = 8, 1_000_000
    parent = np.array([-1, 0, 0, 1, 1, 2, 2], np.int32)
    T = len(parent)
    logits = torch.randn((T, V), generator=torch.Generator().manual_seed(1)) * 1.5
    q = torch.softmax(torch.randn((T, V), generator=torch.Generator().manual_seed(2)), -1)
    toks = np.zeros((n, T), np.int32)
    for c in range(T):
        kids = np.nonzero(parent == c)[0]
        if len(kids):
            toks[:, kids] = rng.choice(V, size=(n, len(kids)), p=q[c].double().numpy() / q[c].double().sum().item())
    lg = logits.to(torch.bfloat16).repeat(n, 1).cuda()
    dp = q.repeat(n, 1).cuda()
    tree_off = torch.arange(n + 1, dtype=torch.int32, device="cuda") * T
    acc, path, bonus, flags = core.tree_accept(core.SAMPLE_MSS, lg, _dev(np.tile(parent, n)), _dev(toks.reshape(-1)),
                                               tree_off, torch.arange(n, device="cuda", dtype=torch.int64),
                                               draft_probs=dp, seed=5, step=1)
    acc, path, bonus = acc.cpu().numpy(), path.cpu().numpy(), bonus.cpu().numpy()
    first = np.where(acc >= 1, toks[np.arange(n), np.maximum(path[:, 1], 0)], bonus)
    p = softmax64(bits_to_f32(tensor_bf16_bits(logits.to(torch.bfloat16))))
    pv, _ = chi2_pvalue(np.bincount(first, minlength=V), p[0])
    assert pv > 1e-4, pv


# ------------------------------------------------------------------ a4 compact
def test_kv_compact_bit_exact(cuda_lib):
    core = cuda_lib
    cfg = VerifyConfig("c", B=12, Hq=8, Hkv=2, d=128, V=100, L=3, prefix=("lognormal", 100, 0.8, 0, 400),
                       tree=("range", 1, 64), mode="greedy", seed=9)
    b = make_verify_batch(cfg, device="cpu", with_logits=False)
    rng = np.random.default_rng(9)
    acc = np.zeros(b["B"], np.int32)
    path = np.full((b["B"], 64), -1, np.int32)
    for i in range(b["B"]):
        s, e = b["tree_off"][i], b["tree_off"][i + 1]
        node = int(rng.integers(0, e - s))
        pth = OT.ancestors_or_self(list(b["parent"][s:e]), node)
        acc[i] = len(pth) - 1
        path[i, :len(pth)] = pth
    kc = b["k_cache"].cuda()
    vc = b["v_cache"].cuda()
    ks = [kc[l] for l in range(cfg.L)]
    vs = [vc[l] for l in range(cfg.L)]
    moves = torch.empty((b["B"], 64, 2), dtype=torch.int32, device="cuda")
    new_len, _ = core.kv_compact(ks, vs, _dev(b["block_table"]), _dev(b["prefix_len"]), _dev(acc), _dev(path),
                                 moves=moves)
    caches = [tensor_bf16_bits(b["k_cache"][l]).copy() for l in range(cfg.L)] + \
             [tensor_bf16_bits(b["v_cache"][l]).copy() for l in range(cfg.L)]
    onl, omv = OC.kv_compact(caches, b["block_table"], b["prefix_len"], acc, path, 64)
    np.testing.assert_array_equal(new_len.cpu().numpy(), onl)
    np.testing.assert_array_equal(moves.cpu().numpy(), omv)
    for l in range(cfg.L):
        np.testing.assert_array_equal(tensor_bf16_bits(kc[l]), caches[l])
        np.testing.assert_array_equal(tensor_bf16_bits(vc[l]), caches[cfg.L + l])


# ------------------------------------------------------------------ a2 attention
def _attn_errors(o_gpu, o_ref):
    diff = o_gpu - o_ref
    return float(np.abs(diff).max()), float(np.linalg.norm(diff) / np.linalg.norm(o_ref))


def _run_attention(core, b, num_ctas=0, samples=None, with_lse=True):
    B, Hq, Hkv, d = b["B"], b["Hq"], b["Hkv"], b["d"]
    q = b["q"][0].cuda()
    kc = b["k_cache"][0].cuda()
    vc = b["v_cache"][0].cuda()
    par, to = _dev(b["parent"]), _dev(b["tree_off"])
    mask, _, flags = core.tree_build_mask(par, to)
    assert int(flags.abs().sum()) == 0
    plan = core.AttnPlan(b["prefix_len"], b["tree_off"], Hq, Hkv, d, 64, num_ctas=num_ctas)
    ws = core.alloc_workspace(plan.ws_bytes)
    plan.upload(ws)
    lse = torch.empty((b["NT"], Hq), dtype=torch.float32, device="cuda") if with_lse else None
    out, _ = core.tree_verify_attention(plan, q, kc, vc, _dev(b["block_table"]), _dev(b["prefix_len"]), to, mask,
                                        b["sm_scale"], ws, lse=lse)
    torch.cuda.synchronize()
    o_ref, lse_ref = OA.tree_verify_attention(
        b["q"][0].double().numpy(), b["k_cache"][0].double().numpy(), b["v_cache"][0].double().numpy(),
        b["block_table"], b["prefix_len"], b["tree_off"], mask.cpu().numpy().view(np.uint64), Hkv, 64,
        b["sm_scale"], samples=samples)
    og = out.float().cpu().numpy()
    if samples is not None:
        rows = np.concatenate([np.arange(b["tree_off"][s], b["tree_off"][s + 1]) for s in samples])
        og, o_ref, lse_ref = og[rows], o_ref[rows], lse_ref[rows]
        lg = lse.cpu().numpy()[rows] if with_lse else None
    else:
        lg = lse.cpu().numpy() if with_lse else None
    return og, o_ref, lg, lse_ref, plan.info()


ATTN_CASES = {
    "tiny": CONFIGS["tiny"],
    "c2_small": VerifyConfig("c2s", B=6, Hq=32, Hkv=8, d=128, V=10, L=1, prefix=("fixed", 1024),
                             tree=("fixed", 16), seed=21),
    "ragged_g4": VerifyConfig("rg4", B=20, Hq=32, Hkv=8, d=128, V=10, L=1,
                              prefix=("lognormal", 150, 1.0, 0, 900), tree=("range", 1, 64), seed=22),
    "g8_T64": VerifyConfig("g8", B=3, Hq=64, Hkv=8, d=128, V=10, L=1, prefix=("fixed", 700),
                           tree=("fixed", 64), seed=23),
    "g4_T64_dual": VerifyConfig("g4d", B=5, Hq=32, Hkv=8, d=128, V=10, L=1, prefix=("lognormal", 300, 1.0, 0, 1500),
                                tree=("fixed", 64), seed=26),
    "g8_T60_dual_ragged": VerifyConfig("g8r", B=4, Hq=64, Hkv=8, d=128, V=10, L=1, prefix=("lognormal", 200, 1.0, 0, 900),
                                       tree=("range", 49, 64), seed=27),
    "g8_T48_gang3": VerifyConfig("g8t48", B=3, Hq=64, Hkv=8, d=128, V=10, L=1, prefix=("fixed", 650),
                                 tree=("fixed", 48), seed=29),
    "d64_g8_dual": VerifyConfig("d64d", B=3, Hq=16, Hkv=2, d=64, V=10, L=1, prefix=("lognormal", 400, 1.0, 0, 2000),
                                tree=("range", 49, 64), seed=28),
    "d64_g2": VerifyConfig("d64", B=9, Hq=4, Hkv=2, d=64, V=10, L=1, prefix=("lognormal", 90, 1.2, 0, 500),
                           tree=("range", 1, 64), seed=24),
    "qscale8": VerifyConfig("q8", B=5, Hq=32, Hkv=8, d=128, V=10, L=1, prefix=("fixed", 333),
                            tree=("range", 4, 40), q_scale=8.0, seed=25),
}


@pytest.mark.parametrize("case", list(ATTN_CASES))
def test_attention_parity(cuda_lib, case):
    b = make_verify_batch(ATTN_CASES[case], device="cpu", with_logits=False)
    og, oref, lg, lref, info = _run_attention(cuda_lib, b)
    mae, rel = _attn_errors(og, oref)
    assert mae <= ATOL and rel <= RTOL_L2, (case, mae, rel, info)
    np.testing.assert_allclose(lg, lref, atol=2e-2, rtol=1e-3)


@pytest.mark.parametrize("num_ctas", [1, 3, 7, 29])
def test_attention_split_kv_parity(cuda_lib, num_ctas):
    """Few CTAs force split-KV cuts and the fused split merge (heavy-tailed prefixes, 1-2 tile gangs)."""
    cfg = VerifyConfig("split", B=7, Hq=32, Hkv=8, d=128, V=10, L=1, prefix=("lognormal", 600, 1.0, 0, 4000),
                       tree=("range", 1, 64), seed=30 + num_ctas)
    b = make_verify_batch(cfg, device="cpu", with_logits=False)
    og, oref, lg, lref, info = _run_attention(cuda_lib, b, num_ctas=num_ctas)
    mae, rel = _attn_errors(og, oref)
    assert mae <= ATOL and rel <= RTOL_L2, (mae, rel, info)
    np.testing.assert_allclose(lg, lref, atol=2e-2, rtol=1e-3)
    if num_ctas > 3:      # (with 3 CTAs each tile-count class may get a single gang: no cuts)
        assert info["num_split_units"] > 0


@pytest.mark.parametrize("num_ctas", [2, 5, 13])
def test_attention_dual_split_kv_parity(cuda_lib, num_ctas):
    """Dual items (two query tiles per CTA, kernel RM = 4: T*g in (384, 512], g = 8) with split-KV
    cuts: each warpgroup writes its own tile's partial and merges its own unit."""
    cfg = VerifyConfig("dsplit", B=3, Hq=64, Hkv=8, d=128, V=10, L=1, prefix=("lognormal", 900, 0.8, 100, 3000),
                       tree=("fixed", 64), seed=40 + num_ctas)
    b = make_verify_batch(cfg, device="cpu", with_logits=False)
    og, oref, lg, lref, info = _run_attention(cuda_lib, b, num_ctas=num_ctas)
    mae, rel = _attn_errors(og, oref)
    assert mae <= ATOL and rel <= RTOL_L2, (mae, rel, info)
    np.testing.assert_allclose(lg, lref, atol=2e-2, rtol=1e-3)
    if num_ctas >= 13:    # (2 or 5 CTAs: whole super-tile gangs, no cuts)
        assert info["num_split_units"] > 0


def test_attention_full_config5_sampled(cuda_lib):
    """BASELINE configs[4] per-GPU shard at G = 8 (B = 16, P = 8K, T = 64, 64/8 heads: dual items)
    in the launch configuration bench.py times; oracle on 3 sampled samples."""
    cfg = CONFIGS["c5g8"]
    b = make_verify_batch(cfg, device="cuda", gen_device="cuda", layers=1, with_logits=False)
    for k in ("q", "k_cache", "v_cache"):
        b[k] = b[k].cpu()
    og, oref, lg, lref, info = _run_attention(cuda_lib, b, samples=[0, 7, 15])
    mae, rel = _attn_errors(og, oref)
    assert mae <= ATOL and rel <= RTOL_L2, (mae, rel, info)
    np.testing.assert_allclose(lg, lref, atol=2e-2, rtol=1e-3)


@pytest.mark.parametrize("gpus", [2, 4])
def test_attention_full_config5_shard_sampled(cuda_lib, gpus):
    """BASELINE configs[4] per-GPU shard at G = 2 / 4 (B = 128/G = 64 / 32 samples, P = 8K,
    T = 64, 64/8 heads), as bench.py --config c5 --gpus G runs each rank; one layer, oracle on 3
    sampled samples (first, middle, last)."""
    cfg = CONFIGS["c5g8"]
    cfg = type(cfg)(**{**cfg.__dict__, "name": "c5", "B": 128 // gpus})
    b = make_verify_batch(cfg, device="cuda", gen_device="cuda", layers=1, with_logits=False)
    for k in ("q", "k_cache", "v_cache"):
        b[k] = b[k].cpu()
    og, oref, lg, lref, info = _run_attention(cuda_lib, b, samples=[0, cfg.B // 2, cfg.B - 1])
    mae, rel = _attn_errors(og, oref)
    assert mae <= ATOL and rel <= RTOL_L2, (mae, rel, info)


def test_attention_full_config2_sampled(cuda_lib):
    """BASELINE configs[1] at full size (B=64, P=1K, T=16, 32/8 heads), in the launch
    configuration bench.py times (plan over all SMs); oracle on 6 sampled samples."""
    cfg = CONFIGS["c2"]
    b = make_verify_batch(cfg, device="cuda", gen_device="cuda", layers=1, with_logits=False)
    for k in ("q", "k_cache", "v_cache"):
        b[k] = b[k].cpu()
    samples = [0, 17, 31, 40, 58, 63]
    og, oref, lg, lref, info = _run_attention(cuda_lib, b, samples=samples)
    mae, rel = _attn_errors(og, oref)
    assert mae <= ATOL and rel <= RTOL_L2, (mae, rel, info)


# ------------------------------------------------------------------ full-size, bench launch configuration
def _c3s_batch(layers=1, with_logits=True, calibrate=True):
    """configs[2] as bench.py runs it (c3s): B = 256 long-tail prefixes, every tree = S(n) from
    select_strategy (host C++) with F and t_sd calibrated on this GPU exactly as bench.py does
    (calibrate=False: the prior F / t_sd, a larger n), MSS rejection sampling; generated on the GPU."""
    import bench
    cfg = CONFIGS["c3s"]
    strat = bench.Strategy(cfg, cuda_lib_core(), "cuda", calibrate=calibrate)
    return make_verify_batch(cfg, device="cuda", gen_device="cuda", layers=layers, with_logits=with_logits,
                             parents=strat.parents)


def cuda_lib_core():
    from paper_2512_04752_b200 import core
    return core


@pytest.mark.parametrize("calibrate", [True, False])
def test_attention_full_config3s_sampled(cuda_lib, calibrate):
    """Long-tail config at full size (B=256, P 512-16K, T from select_strategy) in the launch
    configuration bench.py times (calibrated: T*g <= 64, the 16-warp kernel; prior: T*g > 64, the
    12-warp kernel); oracle on 5 sampled samples (longest included)."""
    b = _c3s_batch(with_logits=False, calibrate=calibrate)
    for k in ("q", "k_cache", "v_cache"):
        b[k] = b[k].cpu()
    P = b["prefix_len"]
    samples = sorted({0, 77, 200, int(np.argmax(P)), int(np.argmin(P))})
    og, oref, lg, lref, info = _run_attention(cuda_lib, b, samples=samples)
    mae, rel = _attn_errors(og, oref)
    assert mae <= ATOL and rel <= RTOL_L2, (mae, rel, info)


def test_accept_mss_full_config3s_bit_exact(cuda_lib):
    """MSS acceptance at full size (B=256, V=128256) through the same call the step makes; the
    oracle (independent per sample: keyed by gid) checks 6 sampled samples bit for bit."""
    core = cuda_lib
    b = _c3s_batch(layers=1)
    g = core.tree_accept(core.SAMPLE_MSS, b["logits"], _dev(b["parent"]), _dev(b["token"]), _dev(b["tree_off"]),
                         _dev(b["gid"]), draft_probs=b["draft_probs"], temperature=1.0, seed=11, step=0)
    g = [x.cpu().numpy() for x in g]
    to = b["tree_off"]
    for s in (0, 5, 99, 128, 201, 255):
        sl = slice(int(to[s]), int(to[s + 1]))
        lg = tensor_bf16_bits(b["logits"][sl].cpu())
        o = OAcc.tree_accept(OAcc.MSS, lg, b["parent"][sl], b["token"][sl], np.array([0, sl.stop - sl.start]),
                             b["gid"][s:s + 1], b["V"], draft_probs=b["draft_probs"][sl].float().cpu().numpy(),
                             temperature=1.0, seed=11, step=0)
        assert g[0][s] == o[0][0] and g[2][s] == o[2][0] and g[3][s] == o[3][0], s
        np.testing.assert_array_equal(g[1][s], o[1][0])


def test_accept_and_compact_full_config2_bit_exact(cuda_lib):
    """Greedy acceptance and the KV commit of BASELINE configs[1] at full size (B=64, V=128256,
    32 layers of 8/128 KV) as the step runs them; the oracle checks every sample's walk and the
    compacted bytes of 4 sampled samples in every layer."""
    core = cuda_lib
    cfg = CONFIGS["c2"]
    b = make_verify_batch(cfg, device="cuda", gen_device="cuda", with_logits=True)
    g = core.tree_accept(core.GREEDY, b["logits"], _dev(b["parent"]), _dev(b["token"]), _dev(b["tree_off"]),
                         _dev(b["gid"]))
    acc, path = g[0], g[1]
    o = OAcc.tree_accept(OAcc.GREEDY, tensor_bf16_bits(b["logits"].cpu()), b["parent"], b["token"], b["tree_off"],
                         b["gid"], b["V"])
    np.testing.assert_array_equal(acc.cpu().numpy(), o[0])
    np.testing.assert_array_equal(path.cpu().numpy(), o[1])
    np.testing.assert_array_equal(g[2].cpu().numpy(), o[2])
    samples = [0, 21, 42, 63]
    bt = b["block_table"]
    pages = np.unique(bt[samples])
    L = cfg.L
    before = [tensor_bf16_bits(b[c][l].index_select(0, torch.as_tensor(pages, device="cuda").long()).cpu())
              for c in ("k_cache", "v_cache") for l in range(L)]
    ks = [b["k_cache"][l] for l in range(L)]
    vs = [b["v_cache"][l] for l in range(L)]
    new_len, _ = core.kv_compact(ks, vs, _dev(bt), _dev(b["prefix_len"]), acc, path)
    after = [tensor_bf16_bits(b[c][l].index_select(0, torch.as_tensor(pages, device="cuda").long()).cpu())
             for c in ("k_cache", "v_cache") for l in range(L)]
    remap = {int(p): i for i, p in enumerate(pages)}
    sub_bt = np.vectorize(lambda x: remap[int(x)])(bt[samples]).astype(np.int32)
    onl, _ = OC.kv_compact(before, sub_bt, b["prefix_len"][samples], o[0][samples], o[1][samples], 64)
    np.testing.assert_array_equal(new_len.cpu().numpy()[samples], onl)
    for x, y in zip(after, before):
        np.testing.assert_array_equal(x, y)


def test_accept_greedy_signed_zero_tie(cuda_lib):
    """-0 and +0 are equal logits: the oracle's strict '>' scan keeps the lower vocab id, and so
    must the GPU's packed max + first-index search (Z6)."""
    core = cuda_lib
    V = 4096
    lg = torch.full((3, V), -1.0, dtype=torch.bfloat16)
    lg[0, 100] = -0.0
    lg[0, 3000] = 0.0          # equal to the max, higher id
    lg[1, 7] = 0.0
    lg[1, 5] = -0.0            # lower id wins again
    parent = np.array([-1, 0, 0], np.int32)
    token = np.array([0, 3000, 100], np.int32)   # child 2 carries the winning token 100
    tree_off = np.array([0, 3], np.int32)
    gid = np.array([5], np.int64)
    g = core.tree_accept(core.GREEDY, lg.cuda(), _dev(parent), _dev(token), _dev(tree_off), _dev(gid))
    o = OAcc.tree_accept(OAcc.GREEDY, tensor_bf16_bits(lg), parent, token, tree_off, gid, V)
    assert int(o[0][0]) == 1 and int(o[1][0][1]) == 2
    for x, y in zip(g, o):
        np.testing.assert_array_equal(x.cpu().numpy(), y)
