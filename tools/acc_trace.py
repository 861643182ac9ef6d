"""Greedy-walk timeline of the fused acceptance at config 2 (profiling variant built with
-DRS_ACC_TRACE: tools/build_variant.sh acctrace -DRS_ACC_TRACE=1; RS_CORE_LIB=<that .so>).
Prints per-sample row durations, prologue, commit and the kernel span. Profiling only."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04752_b200 import core  # noqa: E402
from paper_2512_04752_b200.step import VerifyStep  # noqa: E402
from synth import CONFIGS, make_verify_batch  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
b = make_verify_batch(cfg, device="cuda", gen_device="cuda")
st = VerifyStep(b, mode=core.GREEDY)
for w in range(3):
    st.device_step(seed=1, step=w)
torch.cuda.synchronize()
st.accept_compact_step(1, 0)
torch.cuda.synchronize()
B = b["B"]
buf = (ctypes.c_ulonglong * (8 * B))()
assert core._lib.rs_debug_acc_trace(buf, B) == 0
t = np.array(buf, dtype=np.float64).reshape(B, 8)
acc = st.acc.cpu().numpy()
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
rows = {}
for s_ in range(B):
    a = int(acc[s_])
    stamps = [rel[s_, 0]] + [rel[s_, k] for k in range(1, min(a, 5) + 1)] + [rel[s_, 6]]
    for k in range(len(stamps) - 1):
        rows.setdefault(k, []).append(stamps[k + 1] - stamps[k])
res = {"kernel_span_us": float(rel[:, 7].max()), "start_skew_us": float(rel[:, 0].max()),
       "walk_end_max_us": float(rel[:, 6].max()), "commit_us_median": float(np.median(rel[:, 7] - rel[:, 6])),
       "commit_us_max": float(np.max(rel[:, 7] - rel[:, 6])),
       "rows_hist": np.bincount(acc + 1).tolist(),
       "segment_us_median": {k: round(float(np.median(v)), 2) for k, v in rows.items()},
       "segment_us_max": {k: round(float(np.max(v)), 2) for k, v in rows.items()},
       "longest_walk": [round(float(x), 2) for x in rel[int(np.argmax(acc))]]}
print(json.dumps(res))
