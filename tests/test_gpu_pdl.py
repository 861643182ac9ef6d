"""PDL hazard (header rs_attn_plan_set_early_prefix): a kernel that writes the tree-slot K/V
IMMEDIATELY before rs_tree_verify_attention on the same stream, and lets it start early
(griddepcontrol.launch_dependents, then a 200 us spin, then the writes). The attention output
must equal the oracle computed with the NEW tree K/V, with early prefix streaming on and off;
with it off, even prefix rows written by the preceding kernel are seen."""
import numpy as np
import pytest
import torch

from oracle import attention as OA
from synth import VerifyConfig, make_verify_batch

pytestmark = pytest.mark.gpu


def _slot_rows(b, slots_of):
    """Element-row indices (units of head_dim) of [page, kv head, row] for the chosen slots."""
    rows = []
    for s in range(b["B"]):
        for j in slots_of(s):
            page = b["block_table"][s, j // 64]
            for h in range(b["Hkv"]):
                rows.append((page * b["Hkv"] + h) * 64 + j % 64)
    return np.asarray(rows, np.int64)


@pytest.mark.parametrize("early_prefix,which", [(True, "tree"), (False, "tree"), (False, "prefix+tree")])
def test_attention_sees_upstream_kv_writes(cuda_lib, early_prefix, which):
    from tests.native import pdl_writer
    core = cuda_lib
    lib = pdl_writer()
    cfg = VerifyConfig("pdl", B=16, Hq=32, Hkv=8, d=128, V=10, L=1, prefix=("lognormal", 300, 0.8, 1, 2000),
                       tree=("range", 4, 40), seed=41)
    b = make_verify_batch(cfg, device="cpu")
    P, T = b["prefix_len"], b["T"]
    if which == "tree":
        slots = lambda s: range(P[s], P[s] + T[s])
    else:   # also the last prefix page's rows (only allowed when early_prefix is off)
        slots = lambda s: range(max(0, P[s] - 40), P[s] + T[s])
    rows = _slot_rows(b, slots)
    d = b["d"]
    gen = torch.Generator().manual_seed(5)
    new_k = torch.randn((len(rows), d), generator=gen).to(torch.bfloat16)
    new_v = torch.randn((len(rows), d), generator=gen).to(torch.bfloat16)
    # host copy with the new values (the oracle's input)
    kc = b["k_cache"][0].clone()
    vc = b["v_cache"][0].clone()
    kc.view(-1, d)[torch.as_tensor(rows)] = new_k
    vc.view(-1, d)[torch.as_tensor(rows)] = new_v
    # device cache holds the OLD values until the writer kernel runs
    kd, vd = b["k_cache"][0].cuda(), b["v_cache"][0].cuda()
    q = b["q"][0].cuda()
    to = torch.as_tensor(b["tree_off"]).cuda()
    mask, _, _ = core.tree_build_mask(torch.as_tensor(b["parent"]).cuda(), to)
    plan = core.AttnPlan(P, b["tree_off"], cfg.Hq, cfg.Hkv, d, 64, early_prefix=early_prefix)
    ws = core.alloc_workspace(plan.ws_bytes)
    plan.upload(ws)
    rows_d = torch.as_tensor(rows).cuda()
    nk, nv = new_k.cuda(), new_v.cuda()
    bt, pl = torch.as_tensor(b["block_table"]).cuda(), torch.as_tensor(P).cuda()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    rc = lib.pdl_test_write_rows(kd.data_ptr(), vd.data_ptr(), rows_d.data_ptr(), len(rows), d * 2, nk.data_ptr(),
                                 nv.data_ptr(), 200_000, st.cuda_stream)
    assert rc == 0
    out, _ = core.tree_verify_attention(plan, q, kd, vd, bt, pl, to, mask, b["sm_scale"], ws, stream=st)
    torch.cuda.synchronize()
    o_ref, _ = OA.tree_verify_attention(b["q"][0].double().numpy(), kc.double().numpy(), vc.double().numpy(),
                                        b["block_table"], P, b["tree_off"], mask.cpu().numpy().view(np.uint64),
                                        cfg.Hkv, 64, b["sm_scale"])
    og = out.float().cpu().numpy()
    err = np.abs(og - o_ref).max()
    rel = np.linalg.norm(og - o_ref) / np.linalg.norm(o_ref)
    assert err <= 2e-2 and rel <= 5e-3, (err, rel)
