"""Attention-only timing for kernel tuning: L layers back to back (distinct K/V per layer, each far
larger than L2) through rs_tree_verify_attention_layers, CUDA events, median of reps; HBM
fraction from the algorithmic bytes of SURVEY 8(d) against MEASURED_PEAKS.json. With --trace,
one launch's per-CTA start / end times (tail analysis).

    python tools/attn_bench.py c2|c3s:<n>|c5g8 [--layers 8] [--reps 10] [--trace]
RS_CORE_LIB=<variant .so> selects a library variant (tools/build_variant.sh)."""
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_04752_b200 import core  # noqa: E402
from synth import CONFIGS, draw_prefix_lengths, make_candidate_tree, make_verify_batch  # noqa: E402


def batch(spec, layers):
    name, _, n = spec.partition(":")
    cfg = CONFIGS[name]
    parents = None
    if cfg.tree[0] == "strategy":
        from types import SimpleNamespace
        import bench
        n = int(n or 9)
        P = draw_prefix_lengths(np.random.default_rng(cfg.seed), cfg)
        rng = np.random.default_rng(cfg.seed + 77)
        cands = [make_candidate_tree(rng, int(cfg.tree[1])) for _ in range(cfg.B)]
        sel = core.Selector(SimpleNamespace(**bench.STRATEGY_COST), bench.STRATEGY_KX, bench.STRATEGY_KY)
        res = sel.select(cands, P, n_min=n, n_max=n, patience=2, return_selected=True)
        parents = bench.Strategy._trees(cands, res["selected"], n)
    return cfg, make_verify_batch(cfg, device="cuda", gen_device="cuda", layers=layers, with_logits=False,
                                  parents=parents)


def main():
    spec = sys.argv[1] if len(sys.argv) > 1 else "c2"
    L = int(sys.argv[sys.argv.index("--layers") + 1]) if "--layers" in sys.argv else 8
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 10
    cfg, b = batch(spec, L)
    if "--contiguous" in sys.argv:   # (experiment) every sample's pages consecutive in the pool
        bt = b["block_table"]
        npg = (b["prefix_len"] + b["T"] + 63) // 64
        o = 0
        for i in range(len(npg)):
            bt[i, :npg[i]] = np.arange(o, o + npg[i])
            bt[i, npg[i]:] = o + npg[i] - 1
            o += npg[i]
    dev = "cuda"
    par = torch.as_tensor(b["parent"]).to(dev)
    to = torch.as_tensor(b["tree_off"]).to(dev)
    mask, _, _ = core.tree_build_mask(par, to)
    plan = core.AttnPlan(b["prefix_len"], b["tree_off"], b["Hq"], b["Hkv"], b["d"], 64, early_prefix=True)
    ws = core.alloc_workspace(plan.ws_bytes)
    plan.upload(ws)
    bt = torch.as_tensor(b["block_table"]).to(dev)
    pl = torch.as_tensor(b["prefix_len"]).to(dev)
    out = torch.empty((L,) + tuple(b["q"][0].shape), dtype=torch.bfloat16, device=dev)
    call = core.AttentionLayersCall(plan, [b["q"][l] for l in range(L)], [b["k_cache"][l] for l in range(L)],
                                    [b["v_cache"][l] for l in range(L)], bt, pl, to, mask, b["sm_scale"], ws,
                                    [out[l] for l in range(L)])
    for _ in range(3):
        call()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / L)
    P = b["prefix_len"].astype(np.float64)
    T = b["T"].astype(np.float64)
    Hkv, Hq, d = b["Hkv"], b["Hq"], b["d"]
    alg = float(np.sum(4 * Hkv * d * (P + T) + 4 * Hq * d * T + 8 * T + 4 * np.ceil((P + T) / 64)))
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = float(peaks.get("hbm_gbs", 6544.0))
    us = float(np.median(ts))
    res = {"config": spec, "lib": core.LIB_PATH, "layers": L, "us_per_layer": round(us, 2),
           "us_min": round(float(np.min(ts)), 2), "GBps": round(alg / us / 1e3, 1), "frac_hbm": round(alg / us / 1e3 / hbm, 4),
           "plan": plan.info(), "T_set": sorted(set(int(x) for x in T))[:6]}
    if "--trace" in sys.argv:
        n = plan.info()["num_ctas"]
        tr = torch.zeros(n * 256 * 16, dtype=torch.int64, device=dev)
        core.attn_set_trace(tr)
        core.tree_verify_attention(plan, b["q"][1], b["k_cache"][1], b["v_cache"][1], bt, pl, to, mask,
                                   b["sm_scale"], ws, out=out[1])
        torch.cuda.synchronize()
        core.attn_set_trace(None)
        t = tr.view(n, 256, 16).cpu().numpy().astype(np.float64)
        g0, g1 = t[:, 255, 14], t[:, 255, 15]
        end = (g1 - g0.min()) / 1e3
        start = (g0 - g0.min()) / 1e3
        res["trace_us"] = {"start_max": round(float(start.max()), 2), "end_min": round(float(end.min()), 2),
                           "end_p10": round(float(np.percentile(end, 10)), 2),
                           "end_median": round(float(np.median(end)), 2),
                           "end_p90": round(float(np.percentile(end, 90)), 2), "end_max": round(float(end.max()), 2)}
        if "--dump" in sys.argv:
            cta, items = plan.schedule()
            res["per_cta"] = {"smid": t[:, 255, 13].astype(int).tolist(), "start_us": start.round(2).tolist(),
                              "end_us": end.round(2).tolist(),
                              "blocks": [int(sum(items[i, 4] - items[i, 3] for i in range(cta[c], cta[c + 1])))
                                         for c in range(n)],
                              "items": [int(cta[c + 1] - cta[c]) for c in range(n)],
                              "split_items": [int(sum(items[i, 5] >= 0 for i in range(cta[c], cta[c + 1])))
                                              for c in range(n)]}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
