"""KV-migration data-plane throughput on one GPU (a5): pack and unpack kernel GB/s
for samples of the paper's long-tail lengths (LLM 32 layers + SSM 1 layer, Llama-3-8B shapes),
and the NCCL transfer of the packed buffer through a size-1 communicator (self send/recv: a
device-local copy through NCCL's p2p path; NVLink between GPUs needs >= 2 GPUs).

    python tools/bench_migrate.py [n_samples] [tokens_per_sample]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_04752_b200 import core  # noqa: E402


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e-3


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    tok = int(sys.argv[2]) if len(sys.argv) > 2 else 1536
    ps, Hkv, d, L = 64, 8, 128, 32
    npg = (tok + ps - 1) // ps
    pages = 2 * n * npg + 16
    g = torch.Generator(device="cuda").manual_seed(0)
    K = [torch.randn((pages, Hkv, ps, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(L)]
    V = [torch.randn((pages, Hkv, ps, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(L)]
    Ks = [torch.randn((pages, Hkv, ps, d), generator=g, device="cuda").to(torch.bfloat16)]
    Vs = [torch.randn((pages, Hkv, ps, d), generator=g, device="cuda").to(torch.bfloat16)]
    perm = torch.randperm(pages, generator=torch.Generator().manual_seed(1)).int()
    bt = perm[:n * npg].view(n, npg).contiguous().cuda()
    rows = torch.arange(n, dtype=torch.int32, device="cuda")
    lens = torch.full((n,), tok, dtype=torch.int32, device="cuda")
    e_ssm = core.kv_pack_elems(1, Hkv, d, [tok] * n)
    e_llm = core.kv_pack_elems(L, Hkv, d, [tok] * n)
    buf = torch.empty(e_ssm + e_llm, dtype=torch.int16, device="cuda")
    nbytes = buf.numel() * 2

    def pack():
        core.kv_pack(Ks, Vs, bt, rows, lens, buf, 0)
        core.kv_pack(K, V, bt, rows, lens, buf, e_ssm)

    def unpack():
        core.kv_unpack(Ks, Vs, bt, rows, lens, buf, 0)
        core.kv_unpack(K, V, bt, rows, lens, buf, e_ssm)

    t_pack, t_unpack = timeit(pack), timeit(unpack)
    res = {"samples": n, "tokens_per_sample": tok, "bytes": nbytes,
           "bytes_per_token": nbytes // (n * tok),
           "pack_GBps": round(2 * nbytes / t_pack / 1e9, 1), "unpack_GBps": round(2 * nbytes / t_unpack / 1e9, 1),
           "pack_us": round(t_pack * 1e6, 1), "unpack_us": round(t_unpack * 1e6, 1),
           "note": "GB/s counts read + write (2 x buffer bytes)"}
    try:
        comm = core.Comm(0, 1)
        staging = torch.empty_like(buf)
        scratch = torch.empty(2 * n + n * npg + 64, dtype=torch.int32, device="cuda")
        pool = core.PagePool(pages)
        used = set(bt.flatten().tolist())
        taken = pool.alloc(pages)
        pool.free([p for p in taken.tolist() if p not in used])
        gids = np.arange(n)
        lens_h = np.full(n, tok, np.int32)

        def migrate():
            rows_new = core.migrate_samples(comm, 0, 0, (K, V), (Ks, Vs), ps, pool, gids, lens_h, bt, npg,
                                            staging, scratch)
            flat = rows_new[:, :npg].ravel()
            pool.free(np.unique(flat))
        t_mig = timeit(migrate, n=5)
        res.update({"migrate_self_us": round(t_mig * 1e6, 1),
                    "migrate_self_GBps": round(nbytes / t_mig / 1e9, 1),
                    "migrate_note": "blocking rs_migrate_samples, src == dst (header, handshake, pack, "
                                    "NCCL send/recv to self, unpack); GB/s = buffer bytes / call time"})
        comm.destroy()
    except core.RSError as e:
        res["migrate_error"] = str(e)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
