"""Warm per-kernel timings (CUDA events, median of N launches) for one config's verify step."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04752_b200 import core  # noqa: E402
from paper_2512_04752_b200.step import VerifyStep  # noqa: E402
from synth import CONFIGS, make_verify_batch  # noqa: E402


def timeit(fn, n=20):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    layers = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    cfg = CONFIGS[name]
    if cfg.tree[0] == "strategy":   # c3s: verification trees = S(n) from select_strategy, as bench.py
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import bench
        strat = bench.Strategy(cfg, core, "cuda", calibrate=True)
        b = make_verify_batch(cfg, device="cuda", gen_device="cuda", layers=layers, parents=strat.parents)
    else:
        b = make_verify_batch(cfg, device="cuda", gen_device="cuda", layers=layers)
    mode = {"greedy": core.GREEDY, "delta": core.SAMPLE_DELTA, "mss": core.SAMPLE_MSS}[cfg.mode]
    st = VerifyStep(b, mode=mode)
    st.device_step()
    torch.cuda.synchronize()
    res = {"config": name, "layers_in_test": layers, "plan": st.plan.info()}
    res["mask_us"] = timeit(lambda: st.mask_step())
    res["attention_us_per_layer"] = timeit(lambda: st.attention_step()) / layers
    res["accept_us"] = timeit(lambda: core.tree_accept(st.mode, st.logits, st.parent, st.token, st.tree_off, st.gid,
                                                        draft_probs=st.draft, out=(st.acc, st.path, st.bonus, st.flags)))
    res["compact_us_%d_layers" % layers] = timeit(
        lambda: core.kv_compact(st.k_layers, st.v_layers, st.block_table, st.prefix_len, st.acc, st.path, st.ps,
                                new_len=st.new_len))
    r = st.results()
    res["accepted_mean"] = float(np.mean(r["accepted_len"]))
    res["accepted_max"] = int(np.max(r["accepted_len"]))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
