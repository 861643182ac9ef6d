"""GPU parity for a5 (KV migration): the pack/unpack kernels against oracle.migrate
byte for byte, and rs_migrate_samples end to end on one GPU (NCCL communicator of size 1,
src == dst: header, handshake, pack, send/recv to self, unpack). Bar: bit-exact (north_star)."""
import numpy as np
import pytest
import torch

from oracle import migrate as OM
from synth import VerifyConfig, make_verify_batch
from tests.helpers import tensor_bf16_bits

pytestmark = pytest.mark.gpu


def _dev(x):
    return torch.as_tensor(np.ascontiguousarray(x)).cuda()


def _batch(L, Hkv, d, B=10, seed=4, spare=0):
    cfg = VerifyConfig("m", B=B, Hq=Hkv, Hkv=Hkv, d=d, V=100, L=L, prefix=("lognormal", 150, 0.9, 0, 700),
                       tree=("range", 1, 16), mode="greedy", seed=seed)
    return make_verify_batch(cfg, device="cpu", with_logits=False, spare_pages=spare)


def _bits_layers(cache):
    return [(tensor_bf16_bits(cache[0][l]), tensor_bf16_bits(cache[1][l])) for l in range(cache[0].shape[0])]


@pytest.mark.parametrize("rows_sel", ["all", "subset", "with_empty"])
def test_kv_pack_unpack_bit_exact(cuda_lib, rows_sel):
    core = cuda_lib
    llm = _batch(L=3, Hkv=4, d=128, seed=4)
    ssm = _batch(L=1, Hkv=2, d=64, seed=4)            # same seed: same lengths / block tables
    B = llm["B"]
    rows = {"all": np.arange(B), "subset": np.array([7, 2, 5]), "with_empty": np.array([1, 3, 0])}[rows_sel]
    lens = (llm["prefix_len"][rows]).astype(np.int32)
    if rows_sel == "with_empty":
        lens[1] = 0
    bt = llm["block_table"]
    e_ssm = core.kv_pack_elems(1, 2, 64, lens)
    e_llm = core.kv_pack_elems(3, 4, 128, lens)
    buf = torch.full((e_ssm + e_llm,), -1, dtype=torch.int16, device="cuda")
    models = []
    for b in (ssm, llm):
        kc, vc = b["k_cache"].cuda(), b["v_cache"].cuda()
        models.append(([kc[l] for l in range(kc.shape[0])], [vc[l] for l in range(vc.shape[0])], kc, vc))
    d_rows, d_lens, d_bt = _dev(rows.astype(np.int32)), _dev(lens), _dev(bt)
    core.kv_pack(models[0][0], models[0][1], d_bt, d_rows, d_lens, buf, 0)
    core.kv_pack(models[1][0], models[1][1], d_bt, d_rows, d_lens, buf, e_ssm)
    torch.cuda.synchronize()
    ref = OM.pack([_bits_layers((ssm["k_cache"], ssm["v_cache"])), _bits_layers((llm["k_cache"], llm["v_cache"]))],
                  [bt[r] for r in rows], lens, 64)
    got = buf.cpu().numpy().view(np.uint16)
    assert got.size == ref.size
    np.testing.assert_array_equal(got, ref)

    # unpack into a second store with its own (permuted) pages and compare with the oracle's unpack
    pool = core.PagePool(llm["num_pages"])
    dst_rows = pool.reserve(lens, 64, bt.shape[1])
    assert dst_rows is not None
    dst_models, ref_models = [], []
    for (_, _, kc, vc) in models:
        k2, v2 = torch.zeros_like(kc), torch.zeros_like(vc)
        dst_models.append(([k2[l] for l in range(k2.shape[0])], [v2[l] for l in range(v2.shape[0])], k2, v2))
        ref_models.append([(np.zeros(kc.shape[1:], np.uint16), np.zeros(kc.shape[1:], np.uint16))
                           for _ in range(kc.shape[0])])
    dbt = _dev(dst_rows)
    seq = _dev(np.arange(len(rows), dtype=np.int32))
    core.kv_unpack(dst_models[0][0], dst_models[0][1], dbt, seq, d_lens, buf, 0)
    core.kv_unpack(dst_models[1][0], dst_models[1][1], dbt, seq, d_lens, buf, e_ssm)
    torch.cuda.synchronize()
    OM.unpack(ref, ref_models, [dst_rows[i] for i in range(len(rows))], lens, 64)
    for m in range(2):
        for l, (rk, rv) in enumerate(ref_models[m]):
            np.testing.assert_array_equal(tensor_bf16_bits(dst_models[m][2][l]), rk)
            np.testing.assert_array_equal(tensor_bf16_bits(dst_models[m][3][l]), rv)


def test_migrate_samples_self_nccl(cuda_lib):
    """Full three-phase migration through NCCL on one rank (src == dst): the samples' K/V land
    in freshly reserved pages of the same store, bit-identical to the source pages."""
    core = cuda_lib
    llm = _batch(L=2, Hkv=8, d=128, B=6, seed=11, spare=64)
    B, bt = llm["B"], llm["block_table"]
    kc, vc = llm["k_cache"].cuda(), llm["v_cache"].cuda()
    K, V = [kc[l] for l in range(2)], [vc[l] for l in range(2)]
    used = set(np.unique(bt).tolist())
    pool = core.PagePool(llm["num_pages"])
    taken = pool.alloc(llm["num_pages"])                            # mark the live samples' pages used
    pool.free([p for p in taken.tolist() if p not in used])
    taken = np.array(sorted(used), np.int32)
    comm = core.Comm(0, 1)
    try:
        gids = llm["gid"][[1, 4]]
        lens = llm["prefix_len"][[1, 4]].astype(np.int32)
        src_bt = _dev(bt[[1, 4]])
        nbytes = 2 * core.kv_pack_elems(2, 8, 128, lens)
        staging = torch.empty(nbytes // 2, dtype=torch.int16, device="cuda")
        scratch = torch.empty(2 * 2 + 2 * bt.shape[1], dtype=torch.int32, device="cuda")
        before = [tensor_bf16_bits(t).copy() for t in K + V]
        new_rows = core.migrate_samples(comm, 0, 0, (K, V), None, 64, pool, gids, lens, src_bt, bt.shape[1],
                                        staging, scratch)
        torch.cuda.synchronize()
        assert new_rows.shape == (2, bt.shape[1])
        fresh = set(new_rows.ravel().tolist())
        assert fresh.isdisjoint(set(taken.tolist()))
        after = [tensor_bf16_bits(t) for t in K + V]
        for i, s in enumerate([1, 4]):
            for t in range(int(lens[i])):
                sp, so = bt[s, t // 64], t % 64
                dp = new_rows[i, t // 64]
                for li in range(4):
                    np.testing.assert_array_equal(after[li][dp, :, so], before[li][sp, :, so])
        # the source pages are untouched (migration copies; the caller frees them afterwards)
        for li in range(4):
            for p in used:
                np.testing.assert_array_equal(after[li][p], before[li][p])
        # refusal: more pages than are free -> NO_MEMORY, nothing reserved, nothing written
        free_before = pool.free_count()
        big = np.array([64 * bt.shape[1]] * 8, np.int32)
        staging = torch.empty(core.kv_pack_elems(2, 8, 128, big), dtype=torch.int16, device="cuda")
        scratch = torch.empty(2 * 8 + 8 * bt.shape[1], dtype=torch.int32, device="cuda")
        with pytest.raises(core.RSError, match="status 6"):
            core.migrate_samples(comm, 0, 0, (K, V), None, 64, pool, np.arange(8), big,
                                 _dev(np.repeat(bt[:1], 8, 0)), bt.shape[1], staging, scratch)
        assert pool.free_count() == free_before
    finally:
        comm.destroy()
