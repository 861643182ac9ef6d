import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2512_04752_b200 import core
from synth import CONFIGS, make_verify_batch
cfg = CONFIGS["c2"]
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cfg = type(cfg)(**{**cfg.__dict__, "B": nb})
b = make_verify_batch(cfg, device="cuda", gen_device="cuda", layers=1, with_logits=False)
par = torch.as_tensor(b["parent"]).cuda(); to = torch.as_tensor(b["tree_off"]).cuda()
mask, _, _ = core.tree_build_mask(par, to)
nc = int(sys.argv[2]) if len(sys.argv) > 2 else 0
plan = core.AttnPlan(b["prefix_len"], b["tree_off"], b["Hq"], b["Hkv"], b["d"], 64, num_ctas=nc)
ws = core.alloc_workspace(plan.ws_bytes); plan.upload(ws)
bt = torch.as_tensor(b["block_table"]).cuda(); pl = torch.as_tensor(b["prefix_len"]).cuda()
out = torch.empty_like(b["q"][0])
print("plan", plan.info(), flush=True)
core.tree_verify_attention(plan, b["q"][0], b["k_cache"][0], b["v_cache"][0], bt, pl, to, mask, b["sm_scale"], ws, out=out)
torch.cuda.synchronize()
print("ok", flush=True)
