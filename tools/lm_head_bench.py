"""Time rs_lm_head_argmax (f2) alone at the configs' shapes against the bf16 tensor peak, with
the unfused alternative beside it (cuBLAS logits GEMM via torch.matmul, then rs_tree_accept
GREEDY over the materialised bf16 logits). CUDA events on the launching stream, warm-up first,
inputs resident in HBM. Usage: python tools/lm_head_bench.py [--iters N]"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2512_04752_b200 import core  # noqa: E402


def timeit(fn, iters):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--shapes", default="1024x128256x4096,4608x128256x4096,1024x128256x8192")
    a = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0}
    peak = peaks["bf16_tflops"]
    g = torch.Generator(device="cuda").manual_seed(0)
    for sh in a.shapes.split(","):
        R, V, Dm = (int(x) for x in sh.split("x"))
        H = torch.randn((R, Dm), generator=g, device="cuda").to(torch.bfloat16)
        W = torch.empty((V, Dm), dtype=torch.bfloat16, device="cuda")
        for v0 in range(0, V, 16384):
            W[v0:v0 + 16384].copy_(torch.randn((min(V, v0 + 16384) - v0, Dm), generator=g, device="cuda"))
        tok = torch.empty(R, dtype=torch.int32, device="cuda")
        ws = torch.empty(core.lm_head_argmax_workspace_bytes(R), dtype=torch.uint8, device="cuda")
        fused = timeit(lambda: core.lm_head_argmax(H, W, out=(tok, None), ws=ws), a.iters)
        flops = 2.0 * R * V * Dm
        logits = torch.empty((R, V), dtype=torch.bfloat16, device="cuda")
        gemm = timeit(lambda: torch.matmul(H, W.t(), out=logits), a.iters)
        am = timeit(lambda: torch.argmax(logits, dim=1), a.iters)
        line = {"shape": sh, "fused_ms": round(fused, 4), "fused_tflops": round(flops / fused / 1e9, 1),
                "frac_of_peak": round(flops / fused / 1e9 / peak, 4), "peak_tflops": peak,
                "cublas_logits_ms": round(gemm, 4), "cublas_tflops": round(flops / gemm / 1e9, 1),
                "torch_argmax_over_logits_ms": round(am, 4), "logits_bytes_avoided": R * V * 2}
        print(json.dumps(line), flush=True)
        del H, W, logits


if __name__ == "__main__":
    main()
