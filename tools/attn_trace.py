"""Per-block pipeline timeline of the attention kernel (rs_attn_set_trace), for tuning.

    python tools/attn_trace.py [config] [--layers N]
Prints median latencies between pipeline events and per-CTA block throughput."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04752_b200 import core  # noqa: E402
from synth import CONFIGS, make_verify_batch  # noqa: E402

EV = ["tma_issue", "kv_landed", "s_issued", "s_ready", "p_written", "pv_issued", "epi_start", "epi_end"]


def main():
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    b = make_verify_batch(cfg, device="cuda", gen_device="cuda", layers=2, with_logits=False)
    par = torch.as_tensor(b["parent"]).cuda()
    to = torch.as_tensor(b["tree_off"]).cuda()
    mask, _, _ = core.tree_build_mask(par, to)
    plan = core.AttnPlan(b["prefix_len"], b["tree_off"], b["Hq"], b["Hkv"], b["d"], 64)
    ws = core.alloc_workspace(plan.ws_bytes)
    plan.upload(ws)
    n = plan.info()["num_ctas"]
    tr = torch.zeros(n * 256 * 16, dtype=torch.int64, device="cuda")
    bt = torch.as_tensor(b["block_table"]).cuda()
    pl = torch.as_tensor(b["prefix_len"]).cuda()
    out = torch.empty_like(b["q"][0])
    for l in (0, 1, 0, 1):
        core.tree_verify_attention(plan, b["q"][l], b["k_cache"][l], b["v_cache"][l], bt, pl, to, mask, b["sm_scale"],
                                   ws, out=out)
    core.attn_set_trace(tr)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    core.tree_verify_attention(plan, b["q"][1], b["k_cache"][1], b["v_cache"][1], bt, pl, to, mask, b["sm_scale"],
                               ws, out=out)
    ev1.record()
    torch.cuda.synchronize()
    core.attn_set_trace(None)
    t = tr.view(n, 256, 16).cpu().numpy().astype(np.float64)
    cta, items = plan.schedule()
    res = {"kernel_us": ev0.elapsed_time(ev1) * 1e3}
    lat = {}
    pairs = [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5)]
    rows = []
    per_cta_rate = []
    for c in range(n):
        nb = int(sum(items[i, 4] - items[i, 3] for i in range(cta[c], cta[c + 1])))
        nb = min(nb, 255)
        if nb < 2:
            continue
        tc = t[c, :nb]
        rows.append(tc)
        span = tc[nb - 1, 4] - tc[0, 0]
        per_cta_rate.append(span / nb)
    allb = np.concatenate(rows)
    for a, z in pairs:
        d = allb[:, z] - allb[:, a]
        lat[f"{EV[a]}->{EV[z]}"] = float(np.median(d[allb[:, z] > 0]))
    # inter-block interval of each event
    for e in (0, 3, 4, 5):
        d = np.concatenate([np.diff(r[:, e]) for r in rows])
        lat[f"interval {EV[e]}"] = float(np.median(d))
    for name, (a, z) in {"K_issue->K_landed": (0, 8), "V_issue->V_landed": (1, 9), "K_landed->S_issue": (8, 2),
                         "V_landed->PV_issue": (9, 5), "K_issue->S_issue": (0, 2), "V_issue->PV_issue": (1, 5), "S_issue->S_ready": (2, 3),
                         "S_ready->P_written": (3, 4), "P_written->PV_issue": (4, 5)}.items():
        d = allb[:, z] - allb[:, a]
        lat[name] = float(np.median(d))
    res["median_cycles"] = lat
    # epilogue sub-phases (rows with an epilogue: event 6 set)
    epi = {}
    seq = [(6, 10, "pv_wait"), (10, 11, "ml_barrier"), (11, 14, "stage_wait"), (14, 15, "first_o_chunk"),
           (15, 12, "o_loop_rest"), (12, 13, "store_issue"), (13, 7, "tail"), (6, 7, "total")]
    er = allb[allb[:, 6] > 0]
    for a, z, nm in seq:
        ok = (er[:, a] > 0) & (er[:, z] > 0)
        if ok.any():
            epi[nm] = float(np.median(er[ok, z] - er[ok, a]))
    res["epilogue_cycles_median"] = epi
    res["epilogues_per_cta"] = float(len(er) / max(1, len(rows)))
    # longest gaps between consecutive K TMA issues per CTA (load starvation)
    gaps = np.concatenate([np.sort(np.diff(r[:, 0]))[-4:] for r in rows])
    res["k_issue_gap_top4_median"] = float(np.median(gaps))
    res["k_issue_gap_sum_over_3000_per_cta"] = float(np.median([np.sum(np.clip(np.diff(r[:, 0]) - 3000, 0, None))
                                                                 for r in rows]))
    c0 = t[0, :40]
    base = c0[0, 0]
    res["cta0_timeline"] = [[int(x - base) if x > 0 else -1 for x in row] for row in c0]
    res["cta0_items"] = items[cta[0]:cta[1]].tolist()
    g0 = t[:, 255, 14].copy()
    g1 = t[:, 255, 15].copy()
    smid = t[:, 255, 13].copy().astype(int)
    t[:, 255, 13] = 0
    res["per_cta"] = {"smid": smid.tolist(), "start_ns": (g0 - g0.min()).tolist(), "end_ns": (g1 - g0.min()).tolist(),
                      "blocks": [int(sum(items[i, 4] - items[i, 3] for i in range(cta[c], cta[c + 1]))) for c in range(n)],
                      "items": [int(cta[c + 1] - cta[c]) for c in range(n)]}
    ok = (g0 > 0) & (g1 > 0)
    res["globaltimer_us"] = {"kernel_span": float((g1[ok].max() - g0[ok].min()) / 1e3),
                             "start_skew": float((g0[ok].max() - g0[ok].min()) / 1e3),
                             "cta_median": float(np.median(g1[ok] - g0[ok]) / 1e3),
                             "cta_max": float(np.max(g1[ok] - g0[ok]) / 1e3)}
    t[:, 255, 14] = 0
    t[:, 255, 15] = 0
    spans = []
    for c in range(n):
        v = t[c][t[c] > 0]
        if v.size:
            spans.append((v.max() - v.min()) / 1.92e3)
    spans = np.array(spans)
    res["cta_span_us"] = {"min": float(spans.min()), "median": float(np.median(spans)), "max": float(spans.max()),
                          "p90": float(np.percentile(spans, 90))}
    res["cycles_per_block_per_cta_median"] = float(np.median(per_cta_rate))
    # per-CTA span (globaltimer, us) vs its blocks and items: calibrates the plan's item overhead
    nblk_c = np.array([sum(items[i, 4] - items[i, 3] for i in range(cta[c], cta[c + 1])) for c in range(n)], float)
    nit_c = np.array([cta[c + 1] - cta[c] for c in range(n)], float)
    span_c = (g1 - g0) / 1e3
    okc = (g0 > 0) & (g1 > 0)
    A = np.stack([nblk_c[okc], nit_c[okc], np.ones(okc.sum())], 1)
    coef = np.linalg.lstsq(A, span_c[okc], rcond=None)[0]
    res["span_fit_us"] = {"per_block": float(coef[0]), "per_item": float(coef[1]), "const": float(coef[2]),
                          "item_in_blocks": float(coef[1] / coef[0]) if coef[0] else None,
                          "blocks_min_max": [float(nblk_c.min()), float(nblk_c.max())],
                          "items_min_max": [float(nit_c.min()), float(nit_c.max())]}
    # Little's law per CTA: mean loads in flight = sum(latency) / span (K: ev 0 -> 8, V: ev 1 -> 9)
    infl_k, infl_v, lat_k, lat_v = [], [], [], []
    for r in rows:
        ok = (r[:, 0] > 0) & (r[:, 8] > 0) & (r[:, 1] > 0) & (r[:, 9] > 0)
        r = r[ok]
        if len(r) < 4:
            continue
        span = max(r[:, 8].max(), r[:, 9].max()) - min(r[:, 0].min(), r[:, 1].min())
        infl_k.append(np.sum(r[:, 8] - r[:, 0]) / span)
        infl_v.append(np.sum(r[:, 9] - r[:, 1]) / span)
        lat_k.append(np.mean(r[:, 8] - r[:, 0]))
        lat_v.append(np.mean(r[:, 9] - r[:, 1]))
    res["inflight_mean"] = {"K": float(np.mean(infl_k)), "V": float(np.mean(infl_v)),
                            "lat_K_mean": float(np.mean(lat_k)), "lat_V_mean": float(np.mean(lat_v))}
    res["blocks_per_cta"] = float(np.mean([len(r) for r in rows]))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
