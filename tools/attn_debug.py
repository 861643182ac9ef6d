"""Debug helper: per-sample / per-item attention errors vs the oracle for a parity case."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import attention as OA  # noqa: E402
from paper_2512_04752_b200 import core  # noqa: E402
from synth import VerifyConfig, make_verify_batch  # noqa: E402


def main():
    num_ctas = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    cfg = VerifyConfig("rg4", B=20, Hq=32, Hkv=8, d=128, V=10, L=1, prefix=("lognormal", 150, 1.0, 0, 900),
                       tree=("range", 1, 64), seed=22)
    b = make_verify_batch(cfg, device="cpu", with_logits=False)
    par, to = torch.as_tensor(b["parent"]).cuda(), torch.as_tensor(b["tree_off"]).cuda()
    mask, _, _ = core.tree_build_mask(par, to)
    plan = core.AttnPlan(b["prefix_len"], b["tree_off"], 32, 8, 128, 64, num_ctas=num_ctas)
    ws = core.alloc_workspace(plan.ws_bytes)
    plan.upload(ws)
    out, _ = core.tree_verify_attention(plan, b["q"][0].cuda(), b["k_cache"][0].cuda(), b["v_cache"][0].cuda(),
                                        torch.as_tensor(b["block_table"]).cuda(),
                                        torch.as_tensor(b["prefix_len"]).cuda(), to, mask, b["sm_scale"], ws)
    torch.cuda.synchronize()
    o_ref, _ = OA.tree_verify_attention(b["q"][0].double().numpy(), b["k_cache"][0].double().numpy(),
                                        b["v_cache"][0].double().numpy(), b["block_table"], b["prefix_len"],
                                        b["tree_off"], mask.cpu().numpy().view(np.uint64), 8, 64, b["sm_scale"])
    og = out.float().cpu().numpy()
    err = np.abs(og - o_ref).max(axis=2)   # [NT, Hq]
    cta, items = plan.schedule()
    print("plan", plan.info())
    for s in range(b["B"]):
        sl = slice(b["tree_off"][s], b["tree_off"][s + 1])
        e = err[sl]
        T = sl.stop - sl.start
        if e.max() > 0.02:
            bad_heads = sorted(set(np.nonzero(e > 0.02)[1] // 4))
            bad_nodes = sorted(set(np.nonzero(e > 0.02)[0]))
            its = [(c, list(items[i])) for c in range(len(cta) - 1) for i in range(cta[c], cta[c + 1])
                   if items[i][0] == s]
            print(f"sample {s} P={b['prefix_len'][s]} T={T} maxerr={e.max():.3f} kvheads={bad_heads} "
                  f"nodes={bad_nodes[:8]}.. items={its[:6]}")


if __name__ == "__main__":
    main()
