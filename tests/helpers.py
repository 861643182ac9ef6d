"""Shared test helpers (no method arithmetic)."""
import numpy as np
import torch


def bf16_bits(x) -> np.ndarray:
    """float array -> bf16 bit patterns (uint16), round-to-nearest-even via torch."""
    t = torch.as_tensor(np.asarray(x, dtype=np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16)


def bits_to_f32(bits) -> np.ndarray:
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return b.view(np.float32)


def tensor_bf16_bits(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def softmax64(l, tau=1.0):
    l = np.asarray(l, dtype=np.float64) / tau
    e = np.exp(l - l.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def chi2_pvalue(counts, probs):
    """Pearson chi-square goodness of fit, bins with expected count < 5 merged into one."""
    from scipy.stats import chi2
    counts = np.asarray(counts, dtype=np.float64)
    n = counts.sum()
    exp = np.asarray(probs, dtype=np.float64) * n
    big = exp >= 5
    c = list(counts[big]) + ([counts[~big].sum()] if (~big).any() else [])
    e = list(exp[big]) + ([exp[~big].sum()] if (~big).any() else [])
    c, e = np.asarray(c), np.asarray(e)
    keep = e > 0
    stat = (((c - e) ** 2)[keep] / e[keep]).sum() + (c[~keep].sum() > 0) * 1e9
    df = max(int(keep.sum()) - 1, 1)
    return float(chi2.sf(stat, df)), stat
