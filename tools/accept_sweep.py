"""Profiling: tree_accept alone on config-2-shaped inputs (B=64, T=16, V=128256, bf16) with the
walk length controlled (p_accept 0 -> 1 row per sample, 1 -> the full depth), timed with CUDA
events over repeated launches. Env RS_ACC_CS / RS_ACC_PF select the variant."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04752_b200 import core  # noqa: E402
from synth import CONFIGS, make_verify_batch  # noqa: E402

res = {}
for p_acc in (0.0, 0.8, 1.0):
    cfg = CONFIGS["c2"]
    cfg = type(cfg)(**{**cfg.__dict__, "L": 1, "p_accept": p_acc})
    b = make_verify_batch(cfg, device="cuda", gen_device="cuda")
    dev = lambda x, dt=torch.int32: torch.as_tensor(np.asarray(x)).to(dt).cuda()
    par, tok, to, gid = dev(b["parent"]), dev(b["token"]), dev(b["tree_off"]), dev(b["gid"], torch.int64)
    out = core.tree_accept(core.GREEDY, b["logits"], par, tok, to, gid)
    torch.cuda.synchronize()
    rows = int(out[0].sum().item()) + b["B"]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(5):
        core.tree_accept(core.GREEDY, b["logits"], par, tok, to, gid, out=out)
    n = 50
    ev[0].record()
    for _ in range(n):
        core.tree_accept(core.GREEDY, b["logits"], par, tok, to, gid, out=out)
    ev[1].record()
    torch.cuda.synchronize()
    us = ev[0].elapsed_time(ev[1]) * 1e3 / n
    res[str(p_acc)] = {"us": round(us, 2), "rows_visited": rows, "max_rows": int(out[0].max().item()) + 1}
print(json.dumps({"cs": os.environ.get("RS_ACC_CS", "auto"), "pf": os.environ.get("RS_ACC_PF", "0"), **res}))
