"""f2 on the GPU: rs_lm_head_argmax (tcgen05 GEMM with an arg-max epilogue) and
rs_tree_accept_greedy_tokens (the c-2 walk over per-node arg-max tokens) vs oracle/lm_head.

Floating point decides an integer here (the arg-max), and the GPU accumulates in fp32 in an
order the oracle cannot reproduce, so the bar is (DESIGN "f2 tolerance"): with
tol_r = Dm * 2^-22 * max_v sum_k |h_rk w_vk| (4x the worst-case recursive-summation bound
for fp32 sums of Dm products of bf16-exact values),
  * the GPU's token is a near-maximum: ref[r, tok] >= max_r - 2 tol_r, and equals the oracle's
    arg-max whenever the oracle's top-2 gap exceeds 2 tol_r;
  * |max_logit_gpu - max_r| <= tol_r;
  * exactly tied logits (duplicated weight rows) resolve to the lowest vocabulary id.
The walk is integer work: bit-exact against the oracle."""
import numpy as np
import pytest
import torch

from oracle import lm_head as LH
from synth import CONFIGS, make_lm_head_inputs, make_verify_batch, random_tree_parents

pytestmark = pytest.mark.gpu


def _reference(Hs, W):
    """Oracle logits for rows Hs (float64 [n, Dm]) against W (torch bf16 [V, Dm], any device),
    by vocabulary chunks so full-size weights need no float64 copy; plus the per-row bound
    tol_r = Dm * 2^-22 * max_v sum_k |h_rk w_vk|."""
    ref, ab = [], []
    for v0 in range(0, W.shape[0], 8192):
        Wc = W[v0:v0 + 8192].double().cpu().numpy()
        ref.append(LH.lm_head_logits(Hs, Wc))
        ab.append((np.abs(Hs) @ np.abs(Wc).T).max(axis=1))
    return np.concatenate(ref, axis=1), Hs.shape[1] * 2.0 ** -22 * np.max(np.stack(ab), axis=0)


def _check_rows(tok, mx, H, W, rows=None, min_exact=0.99):
    """H float64 copy of the bf16 hidden states, W torch bf16; rows: the rows tok/mx refer to."""
    rows = np.arange(H.shape[0]) if rows is None else rows
    ref, tol = _reference(H[rows], W)
    idx, rmax = LH.argmax_rows(ref)
    r = np.arange(len(rows))
    assert np.all(tok >= 0) and np.all(tok < W.shape[0])
    assert np.all(ref[r, tok] >= rmax - 2 * tol), "GPU arg-max is not a near-maximum"
    assert np.all(np.abs(mx - rmax) <= tol), np.abs(mx - rmax).max()
    srt = np.sort(ref, axis=1)
    clear = (srt[:, -1] - srt[:, -2]) > 2 * tol
    assert np.array_equal(tok[clear], idx[clear])
    assert clear.mean() >= min_exact, clear.mean()


def _dev_bf16(x):
    return torch.as_tensor(x, dtype=torch.float32).to(torch.bfloat16).cuda()


@pytest.mark.parametrize("rows,V,Dm", [(200, 1000, 256), (5, 100, 64), (128, 256, 128), (129, 257, 192),
                                       (300, 4099, 512)])
def test_lm_head_argmax_random(cuda_lib, rows, V, Dm):
    rng = np.random.default_rng(rows * 7 + V)
    H = _dev_bf16(rng.standard_normal((rows, Dm)))
    W = _dev_bf16(rng.standard_normal((V, Dm)))
    tok, mx = cuda_lib.lm_head_argmax(H, W)
    torch.cuda.synchronize()
    _check_rows(tok.cpu().numpy(), mx.cpu().numpy(), H.double().cpu().numpy(), W, min_exact=0.95)


def test_lm_head_argmax_ties_lowest_id(cuda_lib):
    """Every weight row appears 20 times across the vocabulary (in different tiles): the tied
    maxima must resolve to the lowest vocabulary id of the winning group."""
    rng = np.random.default_rng(5)
    rows, V, Dm, G = 260, 1000, 128, 50
    base = rng.standard_normal((G, Dm))
    grp = rng.permutation(np.arange(V) % G)
    H = _dev_bf16(rng.standard_normal((rows, Dm)))
    W = _dev_bf16(base[grp])
    tok, mx = cuda_lib.lm_head_argmax(H, W)
    torch.cuda.synchronize()
    tok = tok.cpu().numpy()
    first = np.array([np.flatnonzero(grp == g)[0] for g in range(G)])
    assert np.array_equal(tok, first[grp[tok]])
    # the group chosen is a near-maximum group
    _check_rows(tok, mx.cpu().numpy(), H.double().cpu().numpy(), W, min_exact=0.0)


def test_lm_head_argmax_nan_row(cuda_lib):
    rng = np.random.default_rng(6)
    H = rng.standard_normal((40, 128))
    H[7] = np.nan
    Hd = _dev_bf16(H)
    W = _dev_bf16(rng.standard_normal((300, 128)))
    tok, mx = cuda_lib.lm_head_argmax(Hd, W)
    torch.cuda.synchronize()
    tok = tok.cpu().numpy()
    assert tok[7] == -1
    ok = np.arange(40) != 7
    _check_rows(tok[ok], mx.cpu().numpy()[ok], Hd.double().cpu().numpy()[ok], W, min_exact=0.9)


def test_lm_head_argmax_single_inf_logit(cuda_lib):
    """A row with ONE +Inf logit (fp32 overflow of one product) has no arg-max (-1; Z15 on the
    fused path, as the oracle's argmax_rows); without the rule the +Inf column would win."""
    rng = np.random.default_rng(7)
    H = rng.standard_normal((40, 128))
    H[:, 0] = np.abs(H[:, 0]) + 0.5                 # every row prefers column 5 (finite)...
    H[9, 0] = 1e4                                   # ...row 9 overflows there: logit ~ 1e40 -> +Inf
    W0 = rng.standard_normal((300, 128))
    W0[5, 0] = 1e36
    Hd, W = _dev_bf16(H), _dev_bf16(W0)
    tok, _ = cuda_lib.lm_head_argmax(Hd, W)
    torch.cuda.synchronize()
    tok = tok.cpu().numpy()
    ref, _ = LH.argmax_rows((Hd.double().cpu().numpy() @ W.double().cpu().numpy().T).astype(np.float32))
    assert tok[9] == -1 and ref[9] == -1
    others = np.arange(40) != 9
    assert np.all(tok[others] == 5) and np.all(ref[others] == 5)


@pytest.mark.parametrize("name,Dm", [("c2", 4096), ("c5g8", 8192)])
def test_lm_head_full_size_sampled(cuda_lib, name, Dm):
    """Full config size (c2: 1024 rows x V 128256 x 4096; c5g8: 1024 x 128256 x 8192) in the
    launch configuration the bench times; the oracle checks 48 sampled rows, and the fused greedy
    step (arg-max -> walk) is compared with the oracle walk over those rows' arg-max where the
    planted margins make the arg-max unambiguous."""
    b = make_verify_batch(CONFIGS[name], device="cuda", layers=1, with_logits=False)
    inp = make_lm_head_inputs(b, Dm=Dm, device="cuda")
    tok, mx = cuda_lib.lm_head_argmax(inp["hidden"], inp["weight"])
    torch.cuda.synchronize()
    rng = np.random.default_rng(11)
    rows = np.sort(rng.choice(b["NT"], size=48, replace=False))
    Hd = inp["hidden"].double().cpu().numpy()
    t, m = tok.cpu().numpy(), mx.cpu().numpy()
    _check_rows(t[rows], m[rows], Hd, inp["weight"], rows=rows, min_exact=1.0)
    # the walk on the GPU's tokens vs the oracle walk on the same tokens (integer, bit-exact)
    d = lambda x: torch.as_tensor(np.ascontiguousarray(x, dtype=np.int32)).cuda()
    out = cuda_lib.tree_accept_greedy_tokens(tok, d(b["parent"]), d(b["token"]), d(b["tree_off"]))
    torch.cuda.synchronize()
    acc, path, bonus, flags = (x.cpu().numpy() for x in out)
    racc, rpath, rbonus = LH.greedy_walk(t, b["parent"], b["token"], b["tree_off"])
    assert np.array_equal(acc, racc) and np.array_equal(path, rpath) and np.array_equal(bonus, rbonus)
    assert not flags.any()
    assert acc.sum() > 0


def test_fused_greedy_matches_oracle_end_to_end(cuda_lib):
    """tiny-to-medium shapes, every row checked: hidden/W -> arg-max -> walk on the GPU equals
    the oracle's fp64 arg-max -> walk (planted margins: arg-max unambiguous)."""
    cfg = CONFIGS["c2"]
    b = make_verify_batch(cfg, device="cpu", layers=1, with_logits=False)
    b["V"] = 5003                             # smaller vocabulary: all rows checkable in seconds
    tok_np = np.where(b["token"] >= 5003, b["token"] % 5003, b["token"]).astype(np.int32)
    b["token"] = tok_np
    inp = make_lm_head_inputs(b, Dm=1024, device="cpu")
    H, W = inp["hidden"].cuda(), inp["weight"].cuda()
    tok, _ = cuda_lib.lm_head_argmax(H, W, max_logit=False)
    d = lambda x: torch.as_tensor(np.ascontiguousarray(x, dtype=np.int32)).cuda()
    out = cuda_lib.tree_accept_greedy_tokens(tok, d(b["parent"]), d(tok_np), d(b["tree_off"]))
    torch.cuda.synchronize()
    ridx, _ = LH.lm_head_argmax(inp["hidden"].double().numpy(), inp["weight"].double().numpy())
    assert np.array_equal(tok.cpu().numpy(), ridx)
    racc, rpath, rbonus = LH.greedy_walk(ridx, b["parent"], tok_np, b["tree_off"])
    acc, path, bonus, flags = (x.cpu().numpy() for x in out)
    assert np.array_equal(acc, racc) and np.array_equal(path, rpath) and np.array_equal(bonus, rbonus)


def test_walk_random_and_edge_cases(cuda_lib):
    rng = np.random.default_rng(9)
    V = 40
    parents, toks, ams = [], [], []
    sizes = [1, 2, 64, 63, 33, 32] + [int(x) for x in rng.integers(1, 65, size=200)]
    for T in sizes:
        par = random_tree_parents(rng, T)
        tok = rng.integers(0, V, size=T).astype(np.int32)          # duplicates among siblings allowed
        am = rng.integers(0, V, size=T).astype(np.int32)
        kids = [[x for x in range(T) if par[x] == c] for c in range(T)]
        for c in range(T):
            if kids[c] and rng.random() < 0.8:
                am[c] = tok[rng.choice(kids[c])]
        parents.append(par), toks.append(tok), ams.append(am)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    parent, token, amax = (np.concatenate(x).astype(np.int32) for x in (parents, toks, ams))
    d = lambda x: torch.as_tensor(np.ascontiguousarray(x, dtype=np.int32)).cuda()
    out = cuda_lib.tree_accept_greedy_tokens(d(amax), d(parent), d(token), d(off))
    torch.cuda.synchronize()
    acc, path, bonus, flags = (x.cpu().numpy() for x in out)
    racc, rpath, rbonus = LH.greedy_walk(amax, parent, token, off)
    assert np.array_equal(acc, racc) and np.array_equal(path, rpath) and np.array_equal(bonus, rbonus)
    assert not flags.any()
    # malformed tree (parent[2] = 2) and a NaN row (arg-max -1) at a visited root
    parent2 = parent.copy()
    parent2[off[2] + 2] = 2
    amax2 = amax.copy()
    amax2[off[3]] = -1
    out = cuda_lib.tree_accept_greedy_tokens(d(amax2), d(parent2), d(token), d(off))
    torch.cuda.synchronize()
    acc, path, bonus, flags = (x.cpu().numpy() for x in out)
    assert flags[2] == 1 and acc[2] == 0 and bonus[2] == -1 and path[2, 0] == 0
    assert flags[3] == 2 and bonus[3] == -1
    ok = np.ones(len(sizes), bool)
    ok[[2, 3]] = False
    assert np.array_equal(acc[ok], racc[ok]) and np.array_equal(path[ok], rpath[ok])
    assert not flags[ok].any()


def test_verify_step_with_fused_lm_head(cuda_lib):
    """VerifyStep(lm_head=...) — the bench's c2lm step on one layer: acceptance from hidden
    states equals the oracle's fp64 arg-max -> walk, and compaction follows the accepted path."""
    from paper_2512_04752_b200.step import VerifyStep
    b = make_verify_batch(CONFIGS["c2"], device="cuda", layers=1, with_logits=False)
    inp = make_lm_head_inputs(b, Dm=4096, device="cuda")
    st = VerifyStep(b, mode=cuda_lib.GREEDY, lm_head=(inp["hidden"], inp["weight"]))
    res = st.run(seed=0, step=0)
    rng = np.random.default_rng(3)
    amax = st.amax.cpu().numpy()
    rows = np.sort(rng.choice(b["NT"], size=32, replace=False))
    ref, tol = _reference(inp["hidden"].double().cpu().numpy()[rows], inp["weight"])
    assert np.array_equal(amax[rows], LH.argmax_rows(ref)[0])
    racc, rpath, rbonus = LH.greedy_walk(amax, b["parent"], b["token"], b["tree_off"])
    assert np.array_equal(res["accepted_len"], racc) and np.array_equal(res["path"], rpath)
    assert np.array_equal(res["bonus"], rbonus)
    assert np.array_equal(res["new_len"], b["prefix_len"] + 1 + racc)


def test_lm_head_argmax_all_negative_ragged_tail(cuda_lib):
    """Every logit negative and V ragged (1000 = 3 full 256-wide tiles + 232): the zero-filled
    columns past V must never win; the maximum sits in the tail tile for some rows."""
    rng = np.random.default_rng(12)
    rows, V, Dm = 70, 1000, 128
    H = np.abs(rng.standard_normal((rows, Dm))) + 0.1
    W = -np.abs(rng.standard_normal((V, Dm))) - 0.1
    W[997] = -0.01                       # the least negative row: the arg-max, in the ragged tile
    Hd, Wd = _dev_bf16(H), _dev_bf16(W)
    tok, mx = cuda_lib.lm_head_argmax(Hd, Wd)
    torch.cuda.synchronize()
    t = tok.cpu().numpy()
    assert np.all(t == 997)
    assert np.all(mx.cpu().numpy() < 0)
    _check_rows(t, mx.cpu().numpy(), Hd.double().cpu().numpy(), Wd, min_exact=1.0)


# ------------------------------------------------------------------ f2 for the sampling modes
def _check_logits(lg_gpu, H, W, rows):
    """bf16 logits of `rows` vs the fp64 definition: |gpu - ref| <= tol_r + 2^-8 (|ref| + tol_r)
    (fp32 accumulation bound tol_r as above, then one bf16 round-to-nearest: 2^-8 relative)."""
    ref, tol = _reference(H[rows], W)
    g = lg_gpu[rows].float().cpu().numpy().astype(np.float64)
    bound = tol[:, None] + 2.0 ** -8 * (np.abs(ref) + tol[:, None])
    assert np.all(np.abs(g - ref) <= bound), float(np.max(np.abs(g - ref) - bound))


@pytest.mark.parametrize("rows,V,Dm", [(200, 1000, 256), (5, 104, 64), (128, 256, 128), (129, 264, 192),
                                       (300, 4104, 512)])
def test_lm_head_logits_random(cuda_lib, rows, V, Dm):
    rng = np.random.default_rng(rows * 11 + V)
    H = _dev_bf16(rng.standard_normal((rows, Dm)))
    W = _dev_bf16(rng.standard_normal((V, Dm)))
    lg = cuda_lib.lm_head_logits(H, W)
    torch.cuda.synchronize()
    _check_logits(lg, H.double().cpu().numpy(), W, np.arange(rows))


def test_lm_head_logits_full_size_sampled(cuda_lib):
    """c3s-sized LM head (2304 nodes x 128256 x 4096) through the epilogue-writing GEMM; 48
    sampled rows (every row tile, first / last) checked element by element."""
    rng = np.random.default_rng(3)
    rows, V, Dm = 2304, 128256, 4096
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    H = (0.05 * torch.randn((rows, Dm), generator=gen, device="cuda")).to(torch.bfloat16)
    W = torch.randn((V, Dm), generator=gen, device="cuda").to(torch.bfloat16)
    lg = cuda_lib.lm_head_logits(H, W)
    torch.cuda.synchronize()
    sel = np.unique(np.concatenate([[0, rows - 1], np.arange(0, rows, 128), rng.integers(0, rows, 30)]))
    _check_logits(lg, H.double().cpu().numpy(), W, sel)


def test_verify_step_mss_with_lm_head(cuda_lib):
    """The sampling f2 step (rs_lm_head_logits -> rs_tree_accept_compact, MSS with the draft-row
    map): the GEMM's logits are within the bound of the definition, and the acceptance on them is
    the oracle's, bit for bit, on the same (downloaded) logits."""
    core = cuda_lib
    from oracle import accept as OAcc
    from paper_2512_04752_b200.step import VerifyStep
    from synth import VerifyConfig, make_lm_head_sampling_inputs, make_verify_batch
    from tests.helpers import tensor_bf16_bits
    cfg = VerifyConfig("lmss", B=24, Hq=8, Hkv=2, d=128, V=4104, L=2, prefix=("lognormal", 100, 0.8, 1, 300),
                       tree=("range", 2, 40), mode="mss", draft_dtype="bf16", seed=31)
    b = make_verify_batch(cfg, device="cuda", gen_device="cuda", with_logits=False)
    li = make_lm_head_sampling_inputs(b, Dm=256, device="cuda", gen_device="cuda", hidden_sd=0.2)
    b["token"] = li["token"]
    par, off = np.asarray(b["parent"]), np.asarray(b["tree_off"])
    has = np.zeros(len(par), bool)
    for s in range(b["B"]):
        has[par[off[s] + 1:off[s + 1]] + off[s]] = True
    idx = np.nonzero(has)[0]
    row = np.full(len(par), -1, np.int32)
    row[idx] = np.arange(len(idx))
    dq = li["draft_probs"][torch.as_tensor(idx, device="cuda")].contiguous()
    b["draft_probs"], b["draft_row"] = dq, row
    st = VerifyStep(b, mode=core.SAMPLE_MSS, lm_head=(li["hidden"], li["weight"]))
    res = st.run(seed=9, step=4)
    torch.cuda.synchronize()
    _check_logits(st.logits, li["hidden"].double().cpu().numpy(), li["weight"], np.arange(b["NT"]))
    o = OAcc.tree_accept(OAcc.MSS, tensor_bf16_bits(st.logits.cpu()), b["parent"], b["token"], off, b["gid"],
                         b["V"], draft_probs=dq.float().cpu().numpy(), seed=9, step=4, draft_row=row)
    np.testing.assert_array_equal(res["accepted_len"], o[0])
    np.testing.assert_array_equal(res["path"], o[1])
    np.testing.assert_array_equal(res["bonus"], o[2])
    np.testing.assert_array_equal(res["flags"], o[3])
    assert res["accepted_len"].sum() > 0


def test_fused_walk_commit_equals_two_calls(cuda_lib):
    """rs_tree_accept_greedy_tokens_compact == rs_tree_accept_greedy_tokens then rs_kv_compact:
    outputs, new_len, moves and every K/V byte, on ragged trees with planted arg-max tokens, a
    malformed tree and a -1 (non-finite row) token mid-walk."""
    core = cuda_lib
    from synth import VerifyConfig, make_verify_batch, planted_targets
    cfg = VerifyConfig("wc", B=20, Hq=4, Hkv=2, d=128, V=500, L=3, prefix=("lognormal", 90, 0.7, 1, 300),
                       tree=("range", 1, 64), mode="greedy", seed=12)
    b = make_verify_batch(cfg, device="cuda", gen_device="cpu", with_logits=False)
    rng = np.random.default_rng(4)
    amax = planted_targets(rng, b["parent"], b["tree_off"], b["token"], cfg.V, 0.9).astype(np.int32)
    par = b["parent"].copy()
    to = b["tree_off"]
    if to[3] - to[2] > 2:
        par[to[2] + 2] = 2                      # sample 2 malformed
    amax[to[5] + 1:to[6]] = -1                  # sample 5: no arg-max below the root
    d = lambda x: torch.as_tensor(np.ascontiguousarray(x)).cuda()   # noqa: E731
    L = cfg.L
    kc0, vc0 = b["k_cache"].clone(), b["v_cache"].clone()
    a1 = core.tree_accept_greedy_tokens(d(amax), d(par), d(b["token"]), d(to))
    mv1 = torch.empty((b["B"], 64, 2), dtype=torch.int32, device="cuda")
    nl1, _ = core.kv_compact([b["k_cache"][l] for l in range(L)], [b["v_cache"][l] for l in range(L)],
                             d(b["block_table"]), d(b["prefix_len"]), a1[0], a1[1], moves=mv1)
    k1, v1 = b["k_cache"].clone(), b["v_cache"].clone()
    b["k_cache"].copy_(kc0)
    b["v_cache"].copy_(vc0)
    mv2 = torch.empty((b["B"], 64, 2), dtype=torch.int32, device="cuda")
    a2 = core.tree_accept_greedy_tokens_compact(d(amax), d(par), d(b["token"]), d(to),
                                                [b["k_cache"][l] for l in range(L)], [b["v_cache"][l] for l in range(L)],
                                                d(b["block_table"]), d(b["prefix_len"]), moves=mv2)
    torch.cuda.synchronize()
    for x, y in zip(a1, a2[:4]):
        assert torch.equal(x, y)
    assert torch.equal(nl1, a2[4]) and torch.equal(mv1, mv2)
    assert torch.equal(b["k_cache"], k1) and torch.equal(b["v_cache"], v1)
    f = a2[3].cpu().numpy()
    assert f[2] == core.FLAG_MALFORMED and (f[5] & core.FLAG_NONFINITE) and a2[0].sum() > 0
