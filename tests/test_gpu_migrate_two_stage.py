"""GPU parity for f1 (two-stage migration): the token-range pack/unpack kernels
against oracle.migrate byte for byte, and rs_migrate_stage1/2 end to end on one GPU (NCCL
communicator of size 1, src == dst) with the source writing newly verified tokens on another
stream while stage 1 is in flight. Bar: bit-exact (north_star)."""
import numpy as np
import pytest
import torch

from oracle import migrate as OM
from synth import VerifyConfig, make_verify_batch
from tests.helpers import tensor_bf16_bits

pytestmark = pytest.mark.gpu


def _dev(x):
    return torch.as_tensor(np.ascontiguousarray(x)).cuda()


def _batch(L, Hkv, d, B=8, seed=5, spare=0, prefix=("lognormal", 150, 0.9, 1, 700)):
    cfg = VerifyConfig("m", B=B, Hq=Hkv, Hkv=Hkv, d=d, V=100, L=L, prefix=prefix, tree=("fixed", 64),
                       mode="greedy", seed=seed)
    return make_verify_batch(cfg, device="cpu", with_logits=False, spare_pages=spare)


def _layers(b):
    kc, vc = b["k_cache"].cuda(), b["v_cache"].cuda()
    return [kc[l] for l in range(kc.shape[0])], [vc[l] for l in range(vc.shape[0])], kc, vc


def test_kv_pack_unpack_range_bit_exact(cuda_lib):
    core = cuda_lib
    b = _batch(L=3, Hkv=4, d=128)
    B, bt = b["B"], b["block_table"]
    rng = np.random.default_rng(0)
    rows = np.array([5, 0, 3, 7], np.int32)
    cap = (b["prefix_len"] + b["T"])[rows]
    starts = np.array([rng.integers(0, c) for c in cap], np.int32)
    starts[1] = 0
    starts[2] = 64                                       # page-aligned start
    lens = np.array([rng.integers(0, c - s + 1) for c, s in zip(cap, starts)], np.int32)
    lens[3] = 0                                          # empty range
    K, V, kc, vc = _layers(b)
    e = core.kv_pack_elems(3, 4, 128, lens)
    buf = torch.full((e,), -1, dtype=torch.int16, device="cuda")
    core.kv_pack_range(K, V, _dev(bt), _dev(rows), _dev(starts), _dev(lens), buf)
    torch.cuda.synchronize()
    bits = [(tensor_bf16_bits(kc[l]), tensor_bf16_bits(vc[l])) for l in range(3)]
    ref = OM.pack([bits], [bt[r] for r in rows], lens, 64, starts=starts)
    np.testing.assert_array_equal(buf.cpu().numpy().view(np.uint16), ref)
    # unpack into zeroed caches at the same pages and compare with the oracle's unpack
    k2, v2 = torch.zeros_like(kc), torch.zeros_like(vc)
    core.kv_unpack_range([k2[l] for l in range(3)], [v2[l] for l in range(3)], _dev(bt), _dev(rows), _dev(starts),
                         _dev(lens), buf)
    torch.cuda.synchronize()
    refc = [[(np.zeros(kc.shape[1:], np.uint16), np.zeros(kc.shape[1:], np.uint16)) for _ in range(3)]]
    OM.unpack(ref, refc, [bt[r] for r in rows], lens, 64, starts=starts)
    for l in range(3):
        np.testing.assert_array_equal(tensor_bf16_bits(k2[l]), refc[0][l][0])
        np.testing.assert_array_equal(tensor_bf16_bits(v2[l]), refc[0][l][1])


def test_two_stage_self_nccl_overlapped(cuda_lib):
    """Stage 1 moves [0, len1) on a side stream while the compute stream writes the tokens
    [len1, len2) the source verifies meanwhile (slots beyond the prefix only: P:303); stage 2
    moves [len1, len2), SSM first. The destination's pages then hold every token of [0, len2)
    bit-identical to the source, for both models; samples that outgrew their reservation get
    extra pages; stage-2 refusal leaves the pool unchanged."""
    core = cuda_lib
    llm = _batch(L=3, Hkv=8, d=128, seed=12, spare=256)
    ssm = _batch(L=1, Hkv=2, d=64, seed=12, spare=256)   # same seed: same lengths / block tables
    bt = llm["block_table"]
    maxp = bt.shape[1]
    Kl, Vl, kcl, vcl = _layers(llm)
    Ks, Vs, kcs, vcs = _layers(ssm)
    used = set(np.unique(bt).tolist())
    pool = core.PagePool(llm["num_pages"])
    taken = pool.alloc(llm["num_pages"])
    pool.free([p for p in taken.tolist() if p not in used])
    sel = np.array([1, 4, 6], np.int64)
    len1 = llm["prefix_len"][sel].astype(np.int32)
    len2 = (len1 + np.array([3, 40, 70])).astype(np.int32)      # 70 crosses past the reservation
    len2 = np.minimum(len2, llm["prefix_len"][sel] + llm["T"][sel]).astype(np.int32)
    reserve = (len1 + 8).astype(np.int32)
    comm = core.Comm(0, 1)
    side = torch.cuda.Stream()
    try:
        nbytes = 2 * (core.kv_pack_elems(3, 8, 128, len2) + core.kv_pack_elems(1, 2, 64, len2))
        staging = torch.empty(nbytes // 2, dtype=torch.int16, device="cuda")
        scratch = torch.empty(3 * len(sel) + len(sel) * maxp, dtype=torch.int32, device="cuda")
        src_bt = _dev(bt[sel])
        mig = core.TwoStageMigration(comm, 0, 0, (Kl, Vl), (Ks, Vs), 64, pool, maxp, staging, scratch, side)
        torch.cuda.synchronize()
        mig.stage1(llm["gid"][sel], len1, reserve, src_bt)
        # meanwhile the source keeps verifying: new K/V for slots [len1, len2) on the compute stream
        g = torch.Generator(device="cuda").manual_seed(3)
        for i, s in enumerate(sel):
            for t in range(int(len1[i]), int(len2[i])):
                p, r = int(bt[s, t // 64]), t % 64
                for cache in (kcl, vcl, kcs, vcs):
                    cache[:, p, :, r, :] = torch.randn(cache[:, p, :, r, :].shape, generator=g,
                                                       device="cuda").to(torch.bfloat16)
        torch.cuda.synchronize()
        rows1 = mig.dst_rows().copy()
        mig.stage2(len2, src_bt)
        side.synchronize()
        assert mig.ssm_ready.elapsed_time(mig.done) >= 0.0
        rows = mig.dst_rows()
        fresh = set()
        for i in range(len(sel)):
            fresh |= set(rows[i, :(int(len2[i]) + 63) // 64].tolist())
            n1 = (int(reserve[i]) + 63) // 64
            assert np.array_equal(rows[i, :n1], rows1[i, :n1])              # stage-1 pages kept
        assert fresh.isdisjoint(used)
        assert np.all(mig.capacity >= len2)
        for cache in (kcl, vcl, kcs, vcs):
            bits = tensor_bf16_bits(cache)
            for i, s in enumerate(sel):
                t = np.arange(int(len2[i]))
                sp, dp = bt[s, t // 64], rows[i, t // 64]
                np.testing.assert_array_equal(bits[:, dp, :, t % 64], bits[:, sp, :, t % 64])
        # stage-2 refusal: a request the pool cannot hold -> NO_MEMORY, pool unchanged
        mig2 = core.TwoStageMigration(comm, 0, 0, (Kl, Vl), None, 64, pool, maxp, staging, scratch, side)
        small = np.array([10], np.int32)
        mig2.stage1(np.array([99]), small, small, _dev(bt[sel[:1]]))
        side.synchronize()
        hog = pool.alloc(pool.free_count())                 # nothing left for the extra page
        with pytest.raises(core.RSError, match="status 6"):
            mig2.stage2(np.array([70]), _dev(bt[sel[:1]]))   # 10 -> 70 tokens: a second page
        assert pool.free_count() == 0
        pool.free(hog)
    finally:
        side.synchronize()
        comm.destroy()


def test_two_stage_zero_delta_and_llm_only(cuda_lib):
    """Edge cases: stage 2 with no tokens verified meanwhile (an empty transfer) and a store with
    no SSM model; the prefix moved by stage 1 is intact and nothing else changes."""
    core = cuda_lib
    llm = _batch(L=2, Hkv=8, d=128, B=4, seed=13, spare=64)
    bt = llm["block_table"]
    maxp = bt.shape[1]
    K, V, kc, vc = _layers(llm)
    used = set(np.unique(bt).tolist())
    pool = core.PagePool(llm["num_pages"])
    taken = pool.alloc(llm["num_pages"])
    pool.free([p for p in taken.tolist() if p not in used])
    sel = np.array([0, 2], np.int64)
    len1 = llm["prefix_len"][sel].astype(np.int32)
    comm = core.Comm(0, 1)
    side = torch.cuda.Stream()
    try:
        staging = torch.empty(core.kv_pack_elems(2, 8, 128, len1), dtype=torch.int16, device="cuda")
        scratch = torch.empty(3 * 2 + 2 * maxp, dtype=torch.int32, device="cuda")
        mig = core.TwoStageMigration(comm, 0, 0, (K, V), None, 64, pool, maxp, staging, scratch, side)
        mig.stage1(llm["gid"][sel], len1, len1, _dev(bt[sel]))
        free_mid = pool.free_count()
        mig.stage2(len1, _dev(bt[sel]))                # nothing verified meanwhile
        side.synchronize()
        assert pool.free_count() == free_mid            # no extra pages
        rows = mig.dst_rows()
        for cache in (kc, vc):
            bits = tensor_bf16_bits(cache)
            for i, s in enumerate(sel):
                t = np.arange(int(len1[i]))
                np.testing.assert_array_equal(bits[:, rows[i, t // 64], :, t % 64], bits[:, bt[s, t // 64], :, t % 64])
    finally:
        side.synchronize()
        comm.destroy()
