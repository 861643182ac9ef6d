"""Worker processes of the two-rank peer-memory migration tests (tests/test_gpu_peer.py). One
process per instance; ranks use distinct GPUs when there are enough, else share cuda:0 (CUDA
IPC works between two processes on one device). Control plane: gloo over 127.0.0.1. Expected
bytes come from oracle/migrate.py (pack of the source's pages = what must land; unpack into a
copy of the destination's pools = every byte of the destination afterwards)."""
import os
import traceback

import numpy as np
import torch
import torch.distributed as dist

from oracle import migrate as OM

PS = 64


def _bits(t):
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def _pools(dev, L, Hkv, d, num_pages, seed):
    """Per-layer pools filled with random bit patterns (NaN/Inf encodings included: a copy must
    move bytes, not values)."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    mk = lambda: torch.randint(-32768, 32767, (num_pages, Hkv, PS, d), generator=g,
                               dtype=torch.int16).view(torch.bfloat16).to(dev)
    return [mk() for _ in range(L)], [mk() for _ in range(L)]


def _host(model):
    k, v = model
    return [(_bits(a).copy(), _bits(b).copy()) for a, b in zip(k, v)]


def _bcast(obj, src):
    o = [obj]
    dist.broadcast_object_list(o, src=src)
    return o[0]


def case_core(rank, dev):
    """rs_peer_* between two processes: full push 0 -> 1 (dst-only branch on rank 1), range push
    with SSM first 1 -> 0 (dst-only branch on rank 0), and a refused reservation."""
    from paper_2512_04752_b200 import core
    Hkv, d, num_pages, maxp = 2, 128, 48, 8
    llm = _pools(dev, 3, Hkv, d, num_pages, 10 + rank)
    ssm = _pools(dev, 1, Hkv, d, num_pages, 20 + rank)
    pool = core.PagePool(num_pages)
    store = core.peer_connect(core.PeerStore(llm, ssm, PS, rank))
    st = torch.cuda.Stream(dev)

    def src_rows(lens):
        rows = np.zeros((len(lens), maxp), np.int32)
        perm = np.random.default_rng(rank).permutation(num_pages)   # scattered source pages
        o = 0
        for i, n in enumerate(lens):
            npg = (n + PS - 1) // PS
            rows[i, :npg] = perm[o:o + npg]
            rows[i, npg:] = rows[i, npg - 1]
            o += npg
        return rows

    dt = lambda x: torch.as_tensor(np.ascontiguousarray(x, np.int32), device=dev)

    def transfer(src, dst, lens, starts=None, ssm_first=False):
        reserve = lens if starts is None else [a + b for a, b in zip(starts, lens)]
        before = _host(ssm) + _host(llm) if rank == dst else None
        rows = pool.reserve(reserve, PS, maxp) if rank == dst else None
        rows = _bcast(rows, dst)
        if rows is None:
            return None
        sr = src_rows(reserve) if rank == src else None
        if rank == src:
            with torch.cuda.stream(st):
                sbt, dbt, ln = dt(sr), dt(rows), dt(lens)
                sd = dt(starts) if starts is not None else None
            if ssm_first:
                store.push(dst, sbt, dbt, ln, starts=sd, parts=core.PEER_SSM, stream=st)
                store.signal(core.PEER_SSM_READY, st)
                store.push(dst, sbt, dbt, ln, starts=sd, parts=core.PEER_LLM, stream=st)
            else:
                store.push(dst, sbt, dbt, ln, starts=sd, stream=st)
            store.signal(core.PEER_DONE, st)
        src_state = _bcast((_host(ssm) + _host(llm), sr) if rank == src else None, src)
        if rank == dst:
            if ssm_first:
                store.wait(src, core.PEER_SSM_READY, st)
            store.wait(src, core.PEER_DONE, st)
            with torch.cuda.stream(st):       # a reader on the waiting stream sees the bytes
                got = [(_bits(a), _bits(b)) for a, b in zip(ssm[0] + llm[0], ssm[1] + llm[1])]
            caches, srows = src_state
            buf = OM.pack([caches[:1], caches[1:]], list(srows), lens, PS, starts=starts)
            exp = [(a.copy(), b.copy()) for a, b in before]
            n = OM.unpack(buf, [exp[:1], exp[1:]], list(rows), lens, PS, starts=starts)
            assert n == buf.size
            for (ga, gb), (ea, eb) in zip(got, exp):
                assert np.array_equal(ga, ea) and np.array_equal(gb, eb)
        torch.cuda.synchronize(dev)
        dist.barrier()
        return rows

    assert transfer(0, 1, [1, 63, 64, 65, 200, 130]) is not None
    assert transfer(1, 0, [10, 64, 1, 30], starts=[5, 0, 64, 100], ssm_first=True) is not None
    # refusal: rank 1's pool cannot hold the request -> nothing moves, both sides see None
    if rank == 1:
        hold = pool.alloc(pool.free_count() - 2)
    assert transfer(0, 1, [200, 200]) is None
    store.destroy()


def _instance(rank, dev, n, gid0, seed):
    from paper_2512_04752_b200.instance import GenerationInstance
    rng = np.random.default_rng(seed)
    samples = [(gid0 + i, int(rng.integers(5, 300)), int(rng.integers(20, 60))) for i in range(n)]
    inst = GenerationInstance(samples, Hq=8, Hkv=2, d=128, L=2, V=1000, T=8, p_accept=0.7, num_pages=512,
                              max_pages=16, max_batch=40, seed=seed, device=dev)
    return inst, samples


def case_instance(rank, dev, two_stage):
    """Two generation instances with unequal loads rebalance (forced trigger) over peer memory;
    every committed token of every moved sample is bit-identical on the destination (LLM and SSM
    pools), sample state travels, and both run to completion with every page back."""
    from paper_2512_04752_b200 import core
    from paper_2512_04752_b200.realloc import Rebalancer
    inst, samples = _instance(rank, dev, 20 if rank == 0 else 4, 1000 * rank, 5 + rank)
    for _ in range(2):
        inst.step(seed=3)
    store = inst.connect_peers(rank)
    reb = Rebalancer(threshold=12, cooldown=1)
    torch.cuda.synchronize(dev)
    snap = {s.gid: (s.length, s.remaining, s.steps, s.accepted, s.bt_row.copy()) for s in inst.samples}
    host = [_host((inst.k_ssm, inst.v_ssm)), _host((inst.k_llm, inst.v_llm))]
    if two_stage:
        sent, recv, moved, timing = inst.rebalance_two_stage(reb, store, None, None, overlap_steps=1, seed=4,
                                                             force=True)
        torch.cuda.synchronize(dev)
        host = [_host((inst.k_ssm, inst.v_ssm)), _host((inst.k_llm, inst.v_llm))]   # after the overlap step
    else:
        sent, recv, moved = inst.rebalance(reb, store, None, None, force=True)
    torch.cuda.synchronize(dev)
    if rank == 0:
        assert sent > 0 and recv == 0 and moved > 0
    else:
        assert recv > 0 and sent == 0
    mine = {s.gid: s for s in inst.samples}
    gone = [g for g in snap if g not in mine] if rank == 0 else None
    if rank == 0:
        assert sorted(inst._migrated) == sorted(gone)
        lens = [inst._migrated[g][1] for g in gone]       # the length each sample had when it left
        rows = [inst._migrated[g][0] for g in gone]
        if not two_stage:
            assert lens == [snap[g][0] for g in gone]
        ref = OM.pack(host, rows, lens, PS)
        payload = (gone, lens, ref, {g: snap[g][:4] for g in gone})
    else:
        payload = None
    gone, lens, ref, state = _bcast(payload, 0)
    if rank == 1:
        assert sorted(g for g in mine if g < 1000) == sorted(gone)
        got = OM.pack([_host((inst.k_ssm, inst.v_ssm)), _host((inst.k_llm, inst.v_llm))],
                      [mine[g].bt_row for g in gone], lens, PS)
        assert np.array_equal(got, ref)
        for g, ln in zip(gone, lens):
            assert mine[g].length == ln
            if not two_stage:
                assert (mine[g].remaining, mine[g].steps, mine[g].accepted) == tuple(state[g][1:])
    total = 0
    for _ in range(400):
        done = torch.tensor([inst.load == 0], dtype=torch.int32)
        dist.all_reduce(done, op=dist.ReduceOp.MIN)
        if done.item():
            break
        total += inst.step(seed=6)
    assert inst.load == 0 and inst.pool.free_count() == 512
    dist.barrier()
    store.destroy()


def case_nccl(rank, dev):
    """rs_migrate_samples between two processes over NCCL (source-only and destination-only
    branches, and a refusal). Needs NCCL to accept the two ranks' devices (distinct GPUs)."""
    from paper_2512_04752_b200 import core
    Hkv, d, num_pages, maxp = 2, 128, 48, 8
    llm = _pools(dev, 3, Hkv, d, num_pages, 10 + rank)
    ssm = _pools(dev, 1, Hkv, d, num_pages, 20 + rank)
    pool = core.PagePool(num_pages)
    comm = core.Comm(rank, 2)
    staging = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
    scratch = torch.empty(2 * 64 + 64 * maxp, dtype=torch.int32, device=dev)
    lens = [1, 63, 64, 65, 200]
    src_rows = np.zeros((len(lens), maxp), np.int32)
    perm = np.random.default_rng(rank).permutation(num_pages)
    o = 0
    for i, n in enumerate(lens):
        npg = (n + PS - 1) // PS
        src_rows[i, :npg] = perm[o:o + npg]
        src_rows[i, npg:] = src_rows[i, npg - 1]
        o += npg
    before = _host(ssm) + _host(llm)
    src_bt = torch.as_tensor(src_rows, device=dev) if rank == 0 else None
    rows = core.migrate_samples(comm, 0, 1, llm, ssm, PS, pool if rank == 1 else None, list(range(len(lens))), lens,
                                src_bt, maxp, staging, scratch)
    src_state = _bcast((before, src_rows) if rank == 0 else None, 0)
    if rank == 1:
        torch.cuda.synchronize(dev)
        got = _host(ssm) + _host(llm)
        caches, srows = src_state
        buf = OM.pack([caches[:1], caches[1:]], list(srows), lens, PS)
        exp = [(a.copy(), b.copy()) for a, b in before]
        OM.unpack(buf, [exp[:1], exp[1:]], list(rows), lens, PS)
        for (ga, gb), (ea, eb) in zip(got, exp):
            assert np.array_equal(ga, ea) and np.array_equal(gb, eb)
    dist.barrier()
    comm.destroy()


def worker(rank, world, port, case, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    try:
        if case == "core":
            case_core(rank, dev)
        elif case == "nccl":
            case_nccl(rank, dev)
        else:
            case_instance(rank, dev, two_stage=(case == "two_stage"))
        open(os.path.join(outdir, f"ok{rank}"), "w").write("ok")
    except Exception:
        open(os.path.join(outdir, f"err{rank}"), "w").write(traceback.format_exc())
        raise
    finally:
        dist.destroy_process_group()
