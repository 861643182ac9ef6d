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


class _LoopbackRebalancer:
    """Plans one transfer of `count` samples from instance 0 to itself (the reallocation data
    plane through a size-1 NCCL communicator: send and receive on the same GPU)."""

    def __init__(self, count):
        self.count = count

    def plan(self, local_load, force=False):
        from paper_2512_04752_b200.realloc import Transfer
        return [Transfer(0, 0, self.count)]

    def share(self, tr, payload):
        return payload

    def choose(self, transfers, metas):
        transfers[0].samples = sorted(metas, key=lambda m: (m.seq_len, m.gid))[:self.count]
        return transfers


def test_instance_rebalance_loopback_moves_kv_bit_exact(cuda_lib):
    core = cuda_lib
    inst, samples = _instance(n=12, seed=8)
    for _ in range(3):
        inst.step(seed=5)
    before = {s.gid: (s.length, s.remaining, s.steps, s.accepted, s.pages.copy()) for s in inst.samples}
    comm = core.Comm(0, 1)
    staging = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    scratch = torch.empty(2 * 64 + 64 * inst.max_pages, dtype=torch.int32, device="cuda")
    try:
        sent, recv, moved = inst.rebalance(_LoopbackRebalancer(5), comm, staging, scratch)
    finally:
        comm.destroy()
    assert sent == recv == 5 and moved > 0
    assert sorted(s.gid for s in inst.samples) == sorted(before)
    pools = inst.k_llm + inst.v_llm + inst.k_ssm + inst.v_ssm
    for s in inst.samples:
        L0, R0, st0, a0, pg0 = before[s.gid]
        assert (s.length, s.remaining, s.steps, s.accepted) == (L0, R0, st0, a0)
        if not np.array_equal(s.pages[:len(pg0)], pg0):            # a moved sample: new pages, same bytes
            for t in pools:
                old = t[torch.as_tensor(pg0, device="cuda").long()]
                new = t[torch.as_tensor(s.pages, device="cuda").long()]
                # committed slots only: token j of the sample -> (page j // 64, row j % 64)
                for j in range(0, s.length, 7):
                    assert torch.equal(old[j // 64, :, j % 64], new[j // 64, :, j % 64])
    while inst.load:                                              # the moved samples keep generating
        inst.step(seed=6)
    assert inst.finished == len(samples) and inst.pool.free_count() == 256


def test_instance_rebalance_two_stage_loopback(cuda_lib):
    """f1 in the generation loop: stage 1 streams the chosen samples' prefixes while the instance
    runs a verify step (the migrating samples included), stage 2 moves the tokens committed
    meanwhile (SSM first). Every committed token of a moved sample is bit-identical in its new
    pages (LLM and SSM pools), its state carries the overlap step, and the run completes with
    every page back in the pool."""
    core = cuda_lib
    inst, samples = _instance(n=12, seed=9)
    for _ in range(2):
        inst.step(seed=5)
    comm = core.Comm(0, 1)
    staging = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    scratch = torch.empty(3 * 64 + 64 * inst.max_pages, dtype=torch.int32, device="cuda")
    steps_before = {s.gid: s.steps for s in inst.samples}
    try:
        sent, recv, moved, timing = inst.rebalance_two_stage(_LoopbackRebalancer(4), comm, staging, scratch,
                                                             overlap_steps=1, seed=7)
    finally:
        comm.destroy()
    assert sent == recv == 4 and moved > 0
    assert timing["stage2_stall_ms"] >= 0 and timing["delta_tokens"] > 0 and "ssm_ready_ms" in timing
    old = inst._migrated_from
    pools = inst.k_llm + inst.v_llm + inst.k_ssm + inst.v_ssm
    by_gid = {s.gid: s for s in inst.samples}
    assert set(old) <= set(by_gid)
    for g, pg0 in old.items():
        s = by_gid[g]
        assert s.steps == steps_before[g] + 1                      # the overlap step counted
        assert not np.array_equal(s.pages[:len(pg0)], pg0)        # new pages
        for t in pools:
            a = t[torch.as_tensor(pg0, device="cuda").long()]
            b = t[torch.as_tensor(s.pages, device="cuda").long()]
            for j in range(s.length):                              # every committed token
                assert torch.equal(a[j // 64, :, j % 64], b[j // 64, :, j % 64]), (g, j)
    while inst.load:
        inst.step(seed=8)
    assert inst.finished == len(samples) and inst.pool.free_count() == 256
