"""MSS acceptance alone on the c3s workload (BASELINE configs[2] as the method runs it): times
rs_tree_accept(SAMPLE_MSS) with CUDA events over repeated launches and reports the walk's
structure (visited rows, child tests, rejections) and the algorithmic-byte roofline fraction.
Profiling tool; not part of the product. Usage: python tools/mss_bench.py [reps]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2512_04752_b200 import core  # noqa: E402
from synth import CONFIGS, make_verify_batch  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
cfg = CONFIGS["c3s"]
dev = torch.device("cuda", 0)
strat = bench.Strategy(cfg, core, "cuda", calibrate=False, force_n=int(os.environ.get("MSS_N", "8")))
b = make_verify_batch(cfg, device=dev, gen_device=dev, layers=1, parents=strat.parents)
lg, dp = b["logits"], b["draft_probs"]
d32 = lambda x: torch.as_tensor(np.asarray(x), dtype=torch.int32, device=dev)
par, tok, off = d32(b["parent"]), d32(b["token"]), d32(b["tree_off"])
gid = torch.as_tensor(b["gid"], dtype=torch.int64, device=dev)
out = None
for w in range(3):
    out = core.tree_accept(core.SAMPLE_MSS, lg, par, tok, off, gid, draft_probs=dp, temperature=cfg.temperature,
                           seed=11, step=w, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for r in range(reps):
    core.tree_accept(core.SAMPLE_MSS, lg, par, tok, off, gid, draft_probs=dp, temperature=cfg.temperature,
                     seed=11, step=0, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
acc, path = out[0].cpu().numpy(), out[1].cpu().numpy()
P, T = b["parent"], np.diff(b["tree_off"])
V = b["V"]
tests = rej = visited = 0
for s in range(b["B"]):
    o = b["tree_off"][s]
    p = P[o:o + T[s]]
    pth = path[s, :acc[s] + 1]
    visited += len(pth)
    for k, c in enumerate(pth):
        kids = [x for x in range(T[s]) if p[x] == c]
        if k + 1 < len(pth):
            r = kids.index(pth[k + 1])
            tests += r + 1
            rej += r
        else:
            tests += len(kids)
            rej += len(kids)
alg = visited * V * (lg.element_size() + dp.element_size())   # logits + draft row
print(json.dumps(dict(ms=round(ms, 4), B=b["B"], T=int(T[0]), visited_rows=int(visited), child_tests=int(tests),
                      rejections=int(rej), accepted=int(acc.sum()), alg_bytes=int(alg),
                      GBps=round(alg / ms / 1e6, 1), frac_hbm=round(alg / ms / 1e6 / 6536.4, 4))))
