"""Pins for the oracle's RNG (Philox4x32-10) and exp_spec against external facts."""
import math
import os

import numpy as np

from oracle import accept as A

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def _kats():
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        w = [int(x, 16) for x in line.split()]
        yield w[:4], w[4:6], w[6:10]


def test_philox_known_answer_vectors():
    n = 0
    for ctr, key, out in _kats():
        assert list(A.philox4x32_10(ctr, key)) == out
        n += 1
    assert n == 3


def test_philox_uniformity_and_counter_sensitivity():
    # word 0 over 2^16 counters: mean ~ 2^31, every bit ~ 1/2 (a dropped round/xor fails this)
    words = np.array([A.philox4x32_10([i, 7, 0, 0], [1, 2])[0] for i in range(1 << 14)],
                     dtype=np.uint64)
    assert abs(words.mean() / 2**32 - 0.5) < 0.01
    for bit in range(32):
        frac = ((words >> np.uint64(bit)) & np.uint64(1)).mean()
        assert abs(frac - 0.5) < 0.02, bit
    # each counter word and key word changes the output
    base = A.philox4x32_10([1, 2, 3, 4], [5, 6])
    for k in range(4):
        c = [1, 2, 3, 4]
        c[k] ^= 1
        assert list(A.philox4x32_10(c, [5, 6])) != list(base)
    assert list(A.philox4x32_10([1, 2, 3, 4], [5, 7])) != list(base)


def _ulp_err(y, ref):
    y = np.asarray(y, dtype=np.float64)
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    return np.abs(y - ref) / ulp


def test_exp_spec_accuracy_vs_libm():
    """exp_spec(x) within 4 ulp of the true exp over [-32, 0] (dense sweep + random points)."""
    x = np.concatenate([np.linspace(-32.0, 0.0, 400001, dtype=np.float32),
                        -np.random.default_rng(0).random(200000).astype(np.float32) * 32.0])
    y = A.exp_spec_array(x)
    ref = np.exp(x.astype(np.float64))
    err = _ulp_err(y, ref)
    assert err.max() <= 4.0, (err.max(), x[err.argmax()])
    assert np.median(err) <= 0.6


def test_exp_spec_special_values():
    assert A.exp_spec(0.0) == np.float32(1.0)
    assert A.exp_spec(-0.0) == np.float32(1.0)
    assert A.exp_spec(-32.5) == 0.0
    assert A.exp_spec(float("-inf")) == 0.0
    assert A.exp_spec(float("nan")) == 0.0
    # near multiples of ln 2 (the range-reduction boundaries): within 4 ulp of exp
    for k in range(1, 47):
        for dx in (-1e-6, 0.0, 1e-6):
            x = np.float32(-k * math.log(2.0) + dx)
            if x < -32.0:
                continue
            y = A.exp_spec(x)
            assert _ulp_err(y, math.exp(float(x))) <= 4.0


def test_exp_spec_monotone():
    x = np.sort(np.random.default_rng(1).random(100000).astype(np.float32) * -32.0)
    y = A.exp_spec_array(x)
    assert np.all(np.diff(y.astype(np.float64)) >= 0)
