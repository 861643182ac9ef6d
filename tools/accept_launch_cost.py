"""How much of the bench's accept part is the kernel: replays the accept graph alone back to back,
and the mask | attention | accept graphs as bench.py does, timing each part with events (config 2
or c3s). Profiling only."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04752_b200 import core  # noqa: E402
from paper_2512_04752_b200.step import VerifyStep  # noqa: E402
from synth import CONFIGS, make_verify_batch  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
b = make_verify_batch(cfg, device="cuda", gen_device="cuda")
st = VerifyStep(b, mode=core.GREEDY)
g_mask, g_attn, g_acc, _ = st.capture_parts(seed=1, step=0)
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
res = {}
for w in range(3):
    g_acc.replay()
torch.cuda.synchronize()
e0, e1 = E(), E()
e0.record()
for _ in range(50):
    g_acc.replay()
e1.record()
torch.cuda.synchronize()
res["accept_graph_alone_us"] = round(e0.elapsed_time(e1) * 1e3 / 50, 2)
ev = [[E() for _ in range(3)] for _ in range(20)]
for k in range(20):
    g_mask.replay()
    ev[k][0].record()
    g_attn.replay()
    ev[k][1].record()
    g_acc.replay()
    ev[k][2].record()
torch.cuda.synchronize()
res["accept_part_in_step_us"] = round(sum(x[1].elapsed_time(x[2]) for x in ev[2:]) * 1e3 / 18, 2)
# an empty kernel-free reference: event to event on an idle stream
e0.record(); e1.record(); torch.cuda.synchronize()
res["event_pair_us"] = round(e0.elapsed_time(e1) * 1e3, 2)
print(json.dumps(res))
