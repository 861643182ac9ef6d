"""rs_lm_head_logits alone at the c3s shape (2304 nodes x 128256 x 4096): CUDA-event timing over
repeated launches (profiling tool; the ncu capture of this run is the f2-sampling evidence)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04752_b200 import core  # noqa: E402

rows, V, Dm = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (2304, 128256, 4096)))
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
g = torch.Generator(device="cuda")
g.manual_seed(1)
H = (0.05 * torch.randn((rows, Dm), generator=g, device="cuda")).to(torch.bfloat16)
W = torch.randn((V, Dm), generator=g, device="cuda").to(torch.bfloat16)
out = core.lm_head_logits(H, W)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    core.lm_head_logits(H, W, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
fl = 2.0 * rows * V * Dm
print(json.dumps({"rows": rows, "V": V, "Dm": Dm, "ms": round(ms, 4), "TFLOPs": round(fl / ms / 1e9, 1)}))
