"""Probe: can rs_migrate_samples (NCCL) run with two ranks on this box? (NCCL normally refuses two
ranks on one GPU.) Runs tests/peer_worker.py's "nccl" case in two spawned processes."""
import os
import socket
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch.multiprocessing as mp
    from tests import peer_worker
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tempfile.mkdtemp()
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=peer_worker.worker, args=(r, 2, port, "nccl", out)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    for p in ps:
        if p.is_alive():
            p.kill()
    for f in sorted(os.listdir(out)):
        print(f, open(os.path.join(out, f)).read()[-1500:])


if __name__ == "__main__":
    main()
