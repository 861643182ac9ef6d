"""Multi-process control plane of sample reallocation over gloo on CPU: every rank
computes the same plan as the oracle from the all-gathered loads, each source's chosen samples
equal the oracle's choice, and applying the plan conserves samples and lands every instance
on the threshold side Eq. 6 requires. The KV data plane (NCCL) is covered by the GPU tests."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import realloc as OR


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _samples_of(rank, seed):
    rng = np.random.default_rng(seed * 100 + rank)
    n = int(rng.integers(0, 40))
    from paper_2512_04752_b200.realloc import SampleMeta
    return [SampleMeta(gid=rank * 1000 + i, seq_len=int(rng.integers(1, 30)),
                       avg_accepted=float(rng.integers(0, 6)) / 2.0) for i in range(n)]


def _worker(rank, world, port, seed, thr, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_04752_b200.realloc import Rebalancer
        rb = Rebalancer(threshold=thr, cooldown=3)
        mine = _samples_of(rank, seed)
        plans = [rb.plan(len(mine)) for _ in range(3)]     # triggers on the 3rd call (cooldown)
        assert plans[0] == [] and plans[1] == []
        trs = rb.choose(plans[2], mine)
        # apply the metadata side of the plan
        out_g = {s.gid for tr in trs if tr.src == rank for s in tr.samples}
        kept = [s for s in mine if s.gid not in out_g]
        got = [s for tr in trs if tr.dst == rank for s in tr.samples]
        # two-stage migration's state hand-over (f1): each source shares its updated sample
        # state after the overlap steps; every rank sees the source's payload, in plan order
        shared = [rb.share(t, [(s.gid, s.seq_len + 3) for s in t.samples] if t.src == rank else None) for t in trs]
        res = dict(plan=[(t.src, t.dst, t.count) for t in trs],
                   chosen={t.src: [s.gid for s in t.samples] for t in trs},
                   shared=shared,
                   final=sorted(s.gid for s in kept + got))
        np.save(os.path.join(outdir, f"r{rank}.npy"), np.array([res], dtype=object), allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,seed,thr", [(2, 0, 25), (4, 1, 18), (4, 2, 8), (2, 0, 40)])
def test_rebalancer_gloo(world, seed, thr):
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, _free_port(), seed, thr, d), nprocs=world, join=True,
                           start_method="spawn")
        res = [np.load(os.path.join(d, f"r{r}.npy"), allow_pickle=True)[0] for r in range(world)]
    samples = [_samples_of(r, seed) for r in range(world)]
    loads = [len(s) for s in samples]
    ref_plan = OR.plan_reallocation(loads, thr)
    for r in range(world):
        assert res[r]["plan"] == ref_plan, r                 # every rank agrees with the oracle
    assert bool(ref_plan) == (thr != 40)                     # the no-destination case plans nothing
    for s, dd, k in ref_plan:
        ref_choice = OR.choose_samples([(x.gid, x.seq_len, x.avg_accepted) for x in samples[s]], k)
        assert sorted(res[0]["chosen"][s]) == sorted(ref_choice)
    for r in range(world):                                           # share(): the source's payload everywhere
        for (s, dd, k), sh in zip(ref_plan, res[r]["shared"]):
            assert [g for g, _ in sh] == res[0]["chosen"][s] and len(sh) == k
    final_loads = [len(res[r]["final"]) for r in range(world)]
    assert final_loads == OR.apply_plan(loads, ref_plan)
    all_final = sorted(g for r in range(world) for g in res[r]["final"])
    assert all_final == sorted(x.gid for s in samples for x in s)   # conservation, no duplicates
    for s, dd, _ in ref_plan:                                        # Eq. 6 constraints
        assert final_loads[s] >= thr and final_loads[dd] <= thr


def _worker_filtered(rank, world, port, seed, thr, outdir):
    """Sources offer only a filtered subset (as two-stage migration does: samples that outlive
    the overlap), possibly fewer than the planned count: the choice is clamped and broadcast
    (short or empty payload) instead of failing on the source while the others wait."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_04752_b200.realloc import Rebalancer
        rb = Rebalancer(threshold=thr, cooldown=1)
        mine = _samples_of(rank, seed)
        trs = rb.choose(rb.plan(len(mine)), [s for s in mine if s.seq_len > 28])
        res = dict(plan=[(t.src, t.dst, t.count) for t in trs], chosen={t.src: [s.gid for s in t.samples] for t in trs})
        np.save(os.path.join(outdir, f"r{rank}.npy"), np.array([res], dtype=object), allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,seed,thr", [(2, 0, 25), (4, 1, 18)])
def test_rebalancer_choose_clamps_to_eligible(world, seed, thr):
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker_filtered, args=(world, _free_port(), seed, thr, d), nprocs=world, join=True,
                           start_method="spawn")
        res = [np.load(os.path.join(d, f"r{r}.npy"), allow_pickle=True)[0] for r in range(world)]
    samples = [_samples_of(r, seed) for r in range(world)]
    plan = OR.plan_reallocation([len(s) for s in samples], thr)
    assert plan
    short = 0
    for s, dd, k in plan:
        elig = [(x.gid, x.seq_len, x.avg_accepted) for x in samples[s] if x.seq_len > 28]
        short += len(elig) < k                                 # the case the clamp exists for
        ref = OR.choose_samples(elig, min(k, len(elig))) if elig else []
        for r in range(world):
            assert sorted(res[r]["chosen"][s]) == sorted(ref)
    assert short > 0
