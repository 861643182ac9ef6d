"""Config 4 generation loop (paper_2512_04752_b200.instance): bookkeeping of the long-tailed
verify loop on one GPU, and one of its steps against the oracle (greedy walk, bit-exact)."""
import numpy as np
import pytest
import torch

from oracle import accept as OAcc
from tests.helpers import tensor_bf16_bits

pytestmark = pytest.mark.gpu


def _instance(n=24, seed=3, T=8):
    from paper_2512_04752_b200.instance import GenerationInstance
    rng = np.random.default_rng(seed)
    samples = [(100 + i, int(rng.integers(5, 300)), int(rng.integers(1, 40))) for i in range(n)]
    inst = GenerationInstance(samples, Hq=8, Hkv=2, d=128, L=2, V=1000, T=T, p_accept=0.7, num_pages=256,
                              max_pages=16, seed=seed)
    return inst, samples


def test_instance_runs_every_sample_to_completion(cuda_lib):
    inst, samples = _instance()
    total = 0
    for _ in range(200):
        if inst.load == 0:
            break
        total += inst.step(seed=5)
    assert inst.load == 0
    assert total == sum(r for _, _, r in samples)          # every sample produced exactly its response
    assert inst.finished == len(samples)
    assert inst.pool.free_count() == 256                 # every page came back to the pool


def test_instance_lengths_advance_by_accepted_plus_one(cuda_lib):
    inst, _ = _instance(n=16, seed=4)
    before = {s.gid: (s.length, s.remaining) for s in inst.samples}
    inst.step(seed=9)
    acc = inst.res_h.numpy()[:16]
    gids = [g for g in before]
    for i, g in enumerate(gids):
        L0, R0 = before[g]
        made = min(int(acc[i]) + 1, R0)
        live = {s.gid: s for s in inst.samples}
        if R0 - made > 0:
            assert live[g].length == L0 + 1 + int(acc[i])
            assert live[g].remaining == R0 - made
        else:
            assert g not in live


def test_instance_step_accept_matches_oracle(cuda_lib):
    """The step's tree_accept outputs (through the instance's packed metadata) equal the oracle's
    greedy walk on the same logits rows, tree and tokens."""
    inst, _ = _instance(n=20, seed=6)
    inst.step(seed=13, commit=False)
    B, T = 20, inst.T
    NT = B * T
    m = inst.meta_h.numpy()
    o = B
    tree_off = m[o:o + B + 1].copy(); o += B + 1
    parent = m[o:o + NT].copy(); o += NT
    token = m[o:o + NT].copy()
    gid = inst.gid_h.numpy()[:B].copy()
    lg = tensor_bf16_bits(inst.logits[:NT].cpu())
    acc, path, bonus, flags = OAcc.tree_accept(OAcc.GREEDY, lg, parent, token, tree_off, gid, inst.V)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(inst.acc[:B].cpu().numpy(), acc)
    np.testing.assert_array_equal(inst.path[:B].cpu().numpy(), path)
    np.testing.assert_array_equal(inst.bonus[:B].cpu().numpy(), bonus)
    assert acc.sum() > 0    # the synthetic tokens do get accepted
