"""GPU parity of the fused acceptance + KV commit (rs_tree_accept_compact, a3 + a4 in one launch)
against the oracle composition OAcc.tree_accept -> OC.kv_compact on the same
seeded inputs: accepted_len, path, bonus, flags, new_len, moves and every K/V byte bit-exact.
Covers greedy (bf16 / fp32 logits), DELTA and MSS (fp32 / bf16 drafts), malformed trees and
non-finite rows (flagged samples commit what the two-call sequence commits), and the full-size
configs[1] / configs[2] launches the step makes."""
import numpy as np
import pytest
import torch

from oracle import accept as OAcc
from oracle import compact as OC
from synth import CONFIGS, VerifyConfig, make_verify_batch
from tests.helpers import tensor_bf16_bits

pytestmark = pytest.mark.gpu


def _dev(x):
    return torch.as_tensor(np.ascontiguousarray(x)).cuda()


def _oracle(b, logits, mode_o, draft, temperature, seed, step, samples=None):
    """Oracle acceptance of every sample, then the oracle commit of `samples` (all by default)
    on host copies of their pages. Returns (acc, path, bonus, flags, new_len, moves, pages, caches)."""
    lg = tensor_bf16_bits(logits.cpu()) if logits.dtype == torch.bfloat16 else logits.float().cpu().numpy()
    acc, path, bonus, flags = OAcc.tree_accept(mode_o, lg, b["parent"], b["token"], b["tree_off"], b["gid"], b["V"],
                                               draft_probs=draft, temperature=temperature, seed=seed, step=step)
    samples = list(range(b["B"])) if samples is None else samples
    bt = b["block_table"]
    pages = np.unique(bt[samples])
    idx = torch.as_tensor(pages, device=b["k_cache"].device).long()
    L = b["k_cache"].shape[0]
    caches = [tensor_bf16_bits(b[c][l].index_select(0, idx).cpu()).copy() for c in ("k_cache", "v_cache")
              for l in range(L)]
    remap = {int(p): i for i, p in enumerate(pages)}
    sub_bt = np.vectorize(lambda x: remap[int(x)])(bt[samples]).astype(np.int32)
    new_len, moves = OC.kv_compact(caches, sub_bt, b["prefix_len"][samples], acc[samples], path[samples],
                                   b["page_size"])
    return acc, path, bonus, flags, new_len, moves, pages, caches


def _fused(core, b, logits, mode, draft, temperature, seed, step):
    L = b["k_cache"].shape[0]
    ks = [b["k_cache"][l] for l in range(L)]
    vs = [b["v_cache"][l] for l in range(L)]
    moves = torch.empty((b["B"], 64, 2), dtype=torch.int32, device="cuda")
    r = core.tree_accept_compact(mode, logits.cuda(), _dev(b["parent"]), _dev(b["token"]), _dev(b["tree_off"]),
                                 _dev(b["gid"]), ks, vs, _dev(b["block_table"]), _dev(b["prefix_len"]),
                                 draft_probs=None if draft is None else draft.cuda(), temperature=temperature,
                                 seed=seed, step=step, moves=moves)
    torch.cuda.synchronize()
    return [x.cpu().numpy() for x in r]


def _check(core, b, logits, mode, mode_o, draft=None, temperature=1.0, seed=5, step=2, samples=None):
    o_draft = None if draft is None else draft.float().cpu().numpy()
    o = _oracle(b, logits, mode_o, o_draft, temperature, seed, step, samples)
    acc, path, bonus, flags, new_len, moves = _fused(core, b, logits, mode, draft, temperature, seed, step)
    np.testing.assert_array_equal(acc, o[0])
    np.testing.assert_array_equal(path, o[1])
    np.testing.assert_array_equal(bonus, o[2])
    np.testing.assert_array_equal(flags, o[3])
    s = list(range(b["B"])) if samples is None else samples
    np.testing.assert_array_equal(new_len[s], o[4])
    np.testing.assert_array_equal(moves[s], o[5])
    idx = torch.as_tensor(o[6], device=b["k_cache"].device).long()
    L = b["k_cache"].shape[0]
    after = [tensor_bf16_bits(b[c][l].index_select(0, idx).cpu()) for c in ("k_cache", "v_cache") for l in range(L)]
    for x, y in zip(after, o[7]):
        np.testing.assert_array_equal(x, y)
    return acc, flags


def _small(mode, seed, V=1000, draft_dtype="f32", L=3, B=24):
    cfg = VerifyConfig("ac", B=B, Hq=8, Hkv=2, d=128, V=V, L=L, prefix=("lognormal", 100, 0.8, 1, 400),
                       tree=("range", 1, 64), mode=mode, p_accept=0.85, seed=seed, draft_dtype=draft_dtype)
    return make_verify_batch(cfg, device="cuda", gen_device="cpu")


def _plant_bad(b, logits):
    """sample 1: malformed (parent of node 2 = 2); sample 3: NaN in its root row (flagged at the
    root); sample 5: +Inf in every non-root row (flagged after the first accepted node)."""
    parent = b["parent"].copy()
    to = b["tree_off"]
    if to[2] - to[1] > 2:
        parent[to[1] + 2] = 2
    b = dict(b, parent=parent)
    logits = logits.clone()
    logits[int(to[3]), 7] = float("nan")
    if to[6] - to[5] > 1:
        logits[int(to[5]) + 1:int(to[6]), 3] = float("inf")
    return b, logits


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_fused_greedy_bit_exact(cuda_lib, dtype):
    core = cuda_lib
    b = _small("greedy", 21)
    logits = b["logits"] if dtype == "bf16" else b["logits"].float()
    b, logits = _plant_bad(b, logits)
    acc, flags = _check(core, b, logits, core.GREEDY, OAcc.GREEDY)
    assert (flags & core.FLAG_MALFORMED).any() and (flags & core.FLAG_NONFINITE).any()
    assert acc.sum() > 0


def test_fused_delta_bit_exact(cuda_lib):
    core = cuda_lib
    b = _small("delta", 22)
    b, logits = _plant_bad(b, b["logits"])
    _check(core, b, logits, core.SAMPLE_DELTA, OAcc.DELTA, temperature=0.8)


@pytest.mark.parametrize("draft_dtype", ["f32", "bf16"])
def test_fused_mss_bit_exact(cuda_lib, draft_dtype):
    core = cuda_lib
    b = _small("mss", 23, V=4000, draft_dtype=draft_dtype)
    draft = b["draft_probs"]
    if draft_dtype == "bf16":
        draft = draft.to(torch.bfloat16)
    b, logits = _plant_bad(b, b["logits"])
    acc, _ = _check(core, b, logits, core.SAMPLE_MSS, OAcc.MSS, draft=draft, temperature=1.0)
    assert acc.sum() > 0


def test_fused_equals_two_calls_and_layers_edge(cuda_lib):
    """L = 0 (nothing to commit: new_len and moves only) and L = 1; the fused call leaves the
    same bytes as rs_tree_accept then rs_kv_compact."""
    core = cuda_lib
    b = _small("greedy", 24, L=1)
    L = 1
    kc0, vc0 = b["k_cache"].clone(), b["v_cache"].clone()
    g = core.tree_accept(core.GREEDY, b["logits"], _dev(b["parent"]), _dev(b["token"]), _dev(b["tree_off"]),
                         _dev(b["gid"]))
    nl2, _ = core.kv_compact([b["k_cache"][0]], [b["v_cache"][0]], _dev(b["block_table"]), _dev(b["prefix_len"]),
                             g[0], g[1])
    k2, v2 = b["k_cache"].clone(), b["v_cache"].clone()
    b["k_cache"].copy_(kc0)
    b["v_cache"].copy_(vc0)
    r = _fused(core, b, b["logits"], core.GREEDY, None, 1.0, 0, 0)
    assert torch.equal(b["k_cache"], k2) and torch.equal(b["v_cache"], v2)
    np.testing.assert_array_equal(r[4], nl2.cpu().numpy())
    np.testing.assert_array_equal(r[0], g[0].cpu().numpy())
    # L = 0: no layer pointers, acceptance + new_len only
    acc, path, bonus, flags = (torch.empty(b["B"], dtype=torch.int32, device="cuda"),
                               torch.empty((b["B"], 64), dtype=torch.int32, device="cuda"),
                               torch.empty(b["B"], dtype=torch.int32, device="cuda"),
                               torch.empty(b["B"], dtype=torch.int32, device="cuda"))
    nl0 = torch.empty(b["B"], dtype=torch.int32, device="cuda")
    keep = {k: _dev(b[k]) for k in ("parent", "token", "tree_off", "gid", "block_table", "prefix_len")}
    core._check(core._lib.rs_tree_accept_compact(
        core.GREEDY, core._ptr(b["logits"]), core.DTYPE_BF16, None, core.DTYPE_F32, None, core._ptr(keep["parent"]),
        core._ptr(keep["token"]), core._ptr(keep["tree_off"]), core._ptr(keep["gid"]), b["B"], b["V"], 1.0,
        0, 0, core._ptr(acc), core._ptr(path), core._ptr(bonus), core._ptr(flags), None, 0, None, None, 0, b["Hkv"],
        b["d"], b["page_size"], core._ptr(keep["block_table"]), b["max_pages"], core._ptr(keep["prefix_len"]),
        core._ptr(nl0), None, None), "rs_tree_accept_compact")
    torch.cuda.synchronize()
    np.testing.assert_array_equal(nl0.cpu().numpy(), nl2.cpu().numpy())
    assert L == 1


def test_fused_full_config2_bit_exact(cuda_lib):
    """configs[1] at full size (B = 64, V = 128256, 32 layers of 8 x 128 KV) as the step launches
    it: every walk bit-exact, the committed bytes of 4 sampled samples in every layer."""
    core = cuda_lib
    b = make_verify_batch(CONFIGS["c2"], device="cuda", gen_device="cuda", with_logits=True)
    acc, _ = _check(core, b, b["logits"], core.GREEDY, OAcc.GREEDY, samples=[0, 21, 42, 63])
    assert acc.sum() > 0


def test_fused_full_config3s_mss_bit_exact(cuda_lib):
    """configs[2] (c3s: B = 256 long-tail prefixes, S(n) trees from select_strategy, MSS with
    bf16 draft rows) through the fused launch, 2 layers of KV; the oracle walks every sample and
    commits 5 sampled samples (incl. the longest and the shortest prefix)."""
    core = cuda_lib
    from tests.test_gpu_parity import _c3s_batch
    b = _c3s_batch(layers=2)
    P = b["prefix_len"]
    samples = sorted({0, 99, 201, int(np.argmax(P)), int(np.argmin(P))})
    draft = b["draft_probs"]
    acc, _ = _check(core, b, b["logits"], core.SAMPLE_MSS, OAcc.MSS, draft=draft, temperature=1.0, seed=11, step=0,
                    samples=samples)
    assert acc.sum() > 0


def _packed_rows(b, draft):
    """Rows of the nodes with children + the node -> row map (-1: no children), Z29."""
    par, off = np.asarray(b["parent"]), np.asarray(b["tree_off"])
    has = np.zeros(len(par), bool)
    for s in range(len(off) - 1):
        has[par[off[s] + 1:off[s + 1]] + off[s]] = True
    idx = np.nonzero(has)[0]
    row = np.full(len(par), -1, np.int32)
    row[idx] = np.arange(len(idx), dtype=np.int32)
    return draft[torch.as_tensor(idx, device=draft.device)].contiguous(), row, has


def _fused_rows(core, b, logits, draft, row, seed=5, step=2):
    L = b["k_cache"].shape[0]
    ks = [b["k_cache"][l] for l in range(L)]
    vs = [b["v_cache"][l] for l in range(L)]
    moves = torch.empty((b["B"], 64, 2), dtype=torch.int32, device="cuda")
    r = core.tree_accept_compact(core.SAMPLE_MSS, logits.cuda(), _dev(b["parent"]), _dev(b["token"]),
                                 _dev(b["tree_off"]), _dev(b["gid"]), ks, vs, _dev(b["block_table"]),
                                 _dev(b["prefix_len"]), draft_probs=draft.cuda(), temperature=1.0, seed=seed,
                                 step=step, moves=moves, draft_row=None if row is None else _dev(row))
    torch.cuda.synchronize()
    return [x.cpu().numpy() for x in r]


@pytest.mark.parametrize("draft_dtype", ["f32", "bf16"])
def test_fused_mss_draft_row_map_bit_exact(cuda_lib, draft_dtype):
    """MSS through the row map (draft rows of the nodes with children only) vs the oracle with the
    same map, bit for bit; one sample whose internal node has no row is MALFORMED; and garbage in
    the rows of leaves (full layout, identity map) changes nothing (Z29: never read)."""
    core = cuda_lib
    b = _small("mss", 25, V=4000, draft_dtype=draft_dtype, L=2)
    draft = b["draft_probs"] if draft_dtype == "f32" else b["draft_probs"].to(torch.bfloat16)
    dq, row, has = _packed_rows(b, draft)
    off = b["tree_off"]
    victim = next(s for s in range(2, b["B"]) if off[s + 1] - off[s] > 2 and has[off[s] + 1])
    row[off[victim] + 1] = -1                      # an internal node without a row
    o = OAcc.tree_accept(OAcc.MSS, tensor_bf16_bits(b["logits"].cpu()), b["parent"], b["token"], off, b["gid"],
                         b["V"], draft_probs=dq.float().cpu().numpy(), temperature=1.0, seed=5, step=2, draft_row=row)
    g = _fused_rows(core, b, b["logits"], dq, row)
    for x, y in zip(g[:4], o):
        np.testing.assert_array_equal(x, y)
    assert o[3][victim] == OAcc.FLAG_MALFORMED and g[0].sum() > 0
    # leaves' rows hold garbage in the full layout: identical to clean rows
    dg = draft.clone()
    leaves = torch.as_tensor(np.nonzero(~has)[0], device=dg.device)
    dg[leaves] = float("nan")
    ref = OAcc.tree_accept(OAcc.MSS, tensor_bf16_bits(b["logits"].cpu()), b["parent"], b["token"], off, b["gid"],
                           b["V"], draft_probs=draft.float().cpu().numpy(), temperature=1.0, seed=5, step=2)
    g2 = _fused_rows(core, b, b["logits"], dg, None)
    for x, y in zip(g2[:4], ref):
        np.testing.assert_array_equal(x, y)
    assert not (g2[3] & core.FLAG_NONFINITE).any()


def test_fused_full_config3s_packed_rows(cuda_lib):
    """configs[2] as bench.py runs it: draft rows of the nodes with children only (half the rows
    of an S(n) tree), fused launch over 2 layers of KV; the oracle (same map) walks every sample."""
    core = cuda_lib
    from tests.test_gpu_parity import _c3s_batch
    b = _c3s_batch(layers=2)
    dq, row, has = _packed_rows(b, b["draft_probs"])
    assert 0.3 < has.mean() < 0.8
    o = OAcc.tree_accept(OAcc.MSS, tensor_bf16_bits(b["logits"].cpu()), b["parent"], b["token"], b["tree_off"],
                         b["gid"], b["V"], draft_probs=dq.float().cpu().numpy(), temperature=1.0, seed=11, step=0,
                         draft_row=row)
    g = _fused_rows(core, b, b["logits"], dq, row, seed=11, step=0)
    for x, y in zip(g[:4], o):
        np.testing.assert_array_equal(x, y)
    assert g[0].sum() > 0
