"""rs_calibrate (P:213-215 offline profiling of the t_sd regression) on the GPU: the library
times its own verification attention on a (B, P, T) grid over registered KV pools and refits
the ctx's cost model; the fit reproduces the measured points and the ctx's selector uses it."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_calibrate_fits_measured_attention(cuda_lib):
    core = cuda_lib
    L, pages, Hkv, d, Hq = 4, 2200, 8, 128, 32
    k = [torch.randn(pages, Hkv, 64, d, device="cuda").to(torch.bfloat16) for _ in range(L)]
    v = [torch.randn(pages, Hkv, 64, d, device="cuda").to(torch.bfloat16) for _ in range(L)]
    ctx = core.Ctx(0, 1, 64)
    ctx.register_kv(1, k, v)
    from oracle.strategy import CostModel
    ctx.set_strategy(CostModel(1e-3, 0, 0, 0, 0, k_sat=1e12), [0, 0.5, 1], [0.1, 0.6, 0.9])
    grid = [(B, P, T) for B in (16, 64) for P in (512, 2048) for T in (4, 16, 32)]
    dense = 2e-6
    t = ctx.calibrate(Hq, grid, reps=3, dense_s_per_token=dense)
    assert np.all(t > 0)
    # more KV -> more time (HBM-bound attention): the largest N_seq point is the slowest class
    ns = np.array([B * P for B, P, _ in grid], float)
    assert t[np.argmax(ns)] > t[np.argmin(ns)]
    c, _, _ = ctx.strategy()
    assert c["b1"] > 0 and c["c_draft"] == 1e-3
    # the fit reproduces the points it was fitted to (t_attn = fit - c_draft - dense*N_draft)
    nd = np.array([B * T for B, _, T in grid], float)
    pred = c["b0"] + c["b1"] * ns + c["b2"] * nd
    rel = np.abs(pred - (t + dense * nd)) / (t + dense * nd)
    assert np.median(rel) < 0.15, rel
    # b1 ~ the cost of streaming one token's K/V through L layers at a fraction of HBM peak
    per_tok = L * 2 * Hkv * d * 2
    assert 0.2e12 < per_tok / c["b1"] < 8e12
    ctx.destroy()
