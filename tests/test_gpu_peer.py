"""a5 over peer memory between two processes (rs_peer_*: CUDA IPC mappings of the peer's KV
pools, one push kernel from the source's pages into the destination's reserved pages, completion
by an inter-process event). Two ranks on distinct GPUs when the box has them, else both on
cuda:0 — every branch (source-only, destination-only, refusal, SSM-first range push) runs in a
real second process either way. Bytes are compared with oracle/migrate.py pack/unpack."""
import os
import socket
import tempfile
import time

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(case, timeout=240):
    from tests import peer_worker
    with tempfile.TemporaryDirectory() as out:
        ctx = mp.get_context("spawn")
        port = _free_port()
        procs = [ctx.Process(target=peer_worker.worker, args=(r, 2, port, case, out)) for r in range(2)]
        for p in procs:
            p.start()
        deadline = time.time() + timeout
        for p in procs:
            p.join(max(1.0, deadline - time.time()))
        alive = [p for p in procs if p.is_alive()]
        for p in alive:
            p.kill()
        errs = [open(os.path.join(out, f)).read() for f in sorted(os.listdir(out)) if f.startswith("err")]
        assert not errs, "\n".join(errs)
        assert not alive, f"{case}: workers hung"
        assert all(os.path.exists(os.path.join(out, f"ok{r}")) for r in range(2)), [p.exitcode for p in procs]


def test_peer_core_two_processes(cuda_lib):
    _run("core")


def test_peer_rebalance_two_instances(cuda_lib):
    _run("stop")


def test_peer_rebalance_two_stage_two_instances(cuda_lib):
    _run("two_stage")


def test_peer_loopback_in_process(cuda_lib):
    """Same process (own blob imported by raw pointer): push from one set of pages to another
    in the same pools, range + SSM-first; bytes equal oracle pack/unpack."""
    import numpy as np
    from oracle import migrate as OM
    from tests.peer_worker import PS, _host, _pools
    core = cuda_lib
    dev = torch.device("cuda", 0)
    llm = _pools(dev, 2, 4, 64, 40, 1)
    ssm = _pools(dev, 1, 4, 64, 40, 2)
    store = core.PeerStore(llm, ssm, PS, 0)
    store.import_(store.export())
    lens, starts = [3, 64, 100], [0, 10, 27]
    src = np.array([[0, 1, 2, 2], [3, 4, 5, 5], [6, 7, 8, 8]], np.int32)
    dst = np.array([[20, 21, 22, 22], [23, 24, 25, 25], [26, 27, 28, 28]], np.int32)
    before = _host(ssm) + _host(llm)
    dt = lambda x: torch.as_tensor(np.ascontiguousarray(x, np.int32), device=dev)
    st = torch.cuda.current_stream()
    store.push(0, dt(src), dt(dst), dt(lens), starts=dt(starts), parts=core.PEER_SSM, stream=st)
    store.signal(core.PEER_SSM_READY, st)
    store.push(0, dt(src), dt(dst), dt(lens), starts=dt(starts), parts=core.PEER_LLM, stream=st)
    store.signal(core.PEER_DONE, st)
    store.wait(0, core.PEER_DONE, st)
    torch.cuda.synchronize()
    buf = OM.pack([before[:1], before[1:]], list(src), lens, PS, starts=starts)
    exp = [(a.copy(), b.copy()) for a, b in before]
    OM.unpack(buf, [exp[:1], exp[1:]], list(dst), lens, PS, starts=starts)
    got = _host(ssm) + _host(llm)
    for (ga, gb), (ea, eb) in zip(got, exp):
        assert np.array_equal(ga, ea) and np.array_equal(gb, eb)
    # a second import of the same rank is refused; a shape mismatch is refused
    with pytest.raises(core.RSError):
        store.import_(store.export())
    other = core.PeerStore(_pools(dev, 2, 4, 128, 40, 3), ssm, PS, 1)
    with pytest.raises(core.RSError):
        other.import_(store.export())
    other.destroy()
    store.destroy()


def test_nccl_migrate_two_processes(cuda_lib):
    """rs_migrate_samples over NCCL between two processes (the source-only and destination-only
    branches of the handshake and transfer). NCCL needs one GPU per rank: skipped on a one-GPU box."""
    if torch.cuda.device_count() < 2:
        pytest.skip("NCCL needs one GPU per rank (this box has one); the peer transport covers the two-process path")
    _run("nccl")
