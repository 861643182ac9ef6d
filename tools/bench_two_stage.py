"""f1 measurement on one GPU: stall of a stop-the-world migration against the
two-stage one, with the source instance's verify step (config 2, CUDA graph) running while
stage 1 is in flight. NCCL communicator of size 1 (src == dst: NCCL's device-local p2p path;
NVLink needs two GPUs, which one gpurun box does not have).

Reports: verify-step time alone and while stage 1 streams (interference), stage-1 duration
(hidden behind computation), the stop-the-world stall (blocking rs_migrate_samples of the
whole KV) and the two-stage stall (stage 2: the tokens verified meanwhile, SSM first; time to
the SSM-ready event = when drafting can resume on the destination).

    python tools/bench_two_stage.py [n_samples] [tokens_per_sample]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_04752_b200 import core  # noqa: E402
from paper_2512_04752_b200.step import VerifyStep  # noqa: E402
from synth import CONFIGS, make_verify_batch  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    tok = int(sys.argv[2]) if len(sys.argv) > 2 else 1536
    ps, Hkv, d, L = 64, 8, 128, 32
    dev = torch.device("cuda", 0)
    b = make_verify_batch(CONFIGS["c2"], device=dev, gen_device=dev)
    step = VerifyStep(b, mode=core.GREEDY)
    g_step = step.capture(seed=1, step=0)
    # the migrating samples' KV store (LLM 32 layers + SSM 1 layer), room for src and dst pages
    npg = (tok + 512 + ps - 1) // ps
    pages = 2 * n * npg + 64
    gen = torch.Generator(device="cuda").manual_seed(0)
    K = [torch.randn((pages, Hkv, ps, d), generator=gen, device="cuda").to(torch.bfloat16) for _ in range(L)]
    V = [torch.randn((pages, Hkv, ps, d), generator=gen, device="cuda").to(torch.bfloat16) for _ in range(L)]
    Ks = [torch.randn((pages, 8, ps, d), generator=gen, device="cuda").to(torch.bfloat16)]
    Vs = [torch.randn((pages, 8, ps, d), generator=gen, device="cuda").to(torch.bfloat16)]
    pool = core.PagePool(pages)
    src_pages = pool.alloc(n * npg)
    bt = torch.as_tensor(src_pages.reshape(n, npg)).cuda()
    gids = np.arange(n)
    len1 = np.full(n, tok, np.int32)
    comm = core.Comm(0, 1)
    side = torch.cuda.Stream()
    e_all = core.kv_pack_elems(L, Hkv, d, [tok + 512] * n) + core.kv_pack_elems(1, 8, d, [tok + 512] * n)
    staging = torch.empty(e_all, dtype=torch.int16, device="cuda")
    scratch = torch.empty(3 * n + n * npg, dtype=torch.int32, device="cuda")
    compute = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def steps_alone(k):
        a, z = ev(), ev()
        a.record(compute)
        for _ in range(k):
            g_step.replay()
        z.record(compute)
        torch.cuda.synchronize()
        return a.elapsed_time(z) / k

    for _ in range(3):
        g_step.replay()
    t_step = steps_alone(20)

    # stop-the-world: the whole KV in one blocking call (the samples and the caller wait)
    def stw():
        rows = core.migrate_samples(comm, 0, 0, (K, V), (Ks, Vs), ps, pool, gids, len1, bt, npg, staging, scratch)
        pool.free(np.unique(rows[:, :(tok + ps - 1) // ps].ravel()))
    stw()
    a, z = ev(), ev()
    torch.cuda.synchronize()
    a.record(compute)
    stw()
    z.record(compute)
    torch.cuda.synchronize()
    t_stw = a.elapsed_time(z)

    # two-stage: stage 1 on the side stream while verify steps run on the compute stream
    res_runs = []
    for rep in range(3):
        mig = core.TwoStageMigration(comm, 0, 0, (K, V), (Ks, Vs), ps, pool, npg, staging, scratch, side)
        torch.cuda.synchronize()
        s0 = ev()
        s0.record(side)
        mig.stage1(gids, len1, len1 + 256, bt)
        a, z = ev(), ev()
        a.record(compute)
        k = 0
        while not mig.done.query() or k < 2:
            g_step.replay()
            k += 1
            if k % 4 == 0:
                compute.synchronize()
        z.record(compute)
        torch.cuda.synchronize()
        t_stage1 = s0.elapsed_time(mig.done)
        t_step_during = a.elapsed_time(z) / k
        # tokens verified on the source meanwhile: committed per sample per step (c2 acceptance)
        acc_per_step = float(step.acc.float().mean().item()) + 1.0
        len2 = np.minimum(len1 + np.int32(np.ceil(acc_per_step * k)), tok + 512).astype(np.int32)
        t0 = ev()
        t0.record(side)
        mig.stage2(len2, bt)
        side.synchronize()
        res_runs.append(dict(stage1_ms=t_stage1, steps_during_stage1=k, step_ms_during=t_step_during,
                             stage2_stall_ms=t0.elapsed_time(mig.done), ssm_ready_ms=t0.elapsed_time(mig.ssm_ready),
                             delta_tokens=int(len2[0] - len1[0])))
        rows = mig.dst_rows()
        pool.free(np.unique(np.concatenate([rows[i, :(int(len2[i]) + ps - 1) // ps] for i in range(n)])))
    comm.destroy()
    # the same two measurements over peer memory (rs_peer_push: one kernel straight into the
    # destination's reserved pages; loopback: this process's own store, a device-local copy)
    store = core.PeerStore((K, V), (Ks, Vs), ps, 0)
    store.import_(store.export())
    d32 = lambda x: torch.as_tensor(np.ascontiguousarray(x, np.int32), device="cuda")
    peer = {}
    rows = pool.reserve(len1, ps, npg)
    dbt, ln1 = d32(rows), d32(len1)
    for rep in range(3):   # stop-the-world push of the whole KV
        a, z = ev(), ev()
        torch.cuda.synchronize()
        a.record(compute)
        store.push(0, bt, dbt, ln1, stream=compute)
        z.record(compute)
        torch.cuda.synchronize()
        peer["stop_the_world_stall_ms"] = round(a.elapsed_time(z), 3)
    pool.free(np.unique(rows.ravel()))
    rows = pool.reserve(len1 + 256, ps, npg)
    dbt = d32(rows)
    s0, s1 = ev(), ev()
    torch.cuda.synchronize()
    s0.record(side)
    store.push(0, bt, dbt, ln1, stream=side)
    s1.record(side)
    a, z = ev(), ev()
    a.record(compute)
    k = 0
    while not s1.query() or k < 2:
        g_step.replay()
        k += 1
        if k % 4 == 0:
            compute.synchronize()
    z.record(compute)
    torch.cuda.synchronize()
    acc_per_step = float(step.acc.float().mean().item()) + 1.0
    len2 = np.minimum(len1 + np.int32(np.ceil(acc_per_step * k)), tok + 256).astype(np.int32)
    t0, t_ssm, t1 = ev(), ev(), ev()
    dl2 = d32(len2 - len1)              # (the stage-2 lengths on the device before the clock starts)
    torch.cuda.synchronize()
    t0.record(side)
    store.push(0, bt, dbt, dl2, starts=ln1, parts=core.PEER_SSM, stream=side)
    t_ssm.record(side)
    store.push(0, bt, dbt, dl2, starts=ln1, parts=core.PEER_LLM, stream=side)
    t1.record(side)
    side.synchronize()
    peer.update(stage1_ms_overlapped=round(s0.elapsed_time(s1), 3), steps_during_stage1=k,
                step_ms_during=round(a.elapsed_time(z) / k, 4), two_stage_stall_ms=round(t0.elapsed_time(t1), 3),
                two_stage_ssm_ready_ms=round(t0.elapsed_time(t_ssm), 3),
                push_GBps_stage1=round(2 * (core.kv_pack_elems(L, Hkv, d, len1) + core.kv_pack_elems(1, 8, d, len1))
                                       / (s0.elapsed_time(s1) * 1e-3) / 1e9, 1))
    pool.free(np.unique(rows.ravel()))
    store.destroy()
    r = res_runs[-1]
    nbytes = 2 * (core.kv_pack_elems(L, Hkv, d, len1) + core.kv_pack_elems(1, 8, d, len1))
    out = {"samples": n, "tokens_per_sample": tok, "bytes_stage1": int(nbytes),
           "verify_step_ms_alone": round(t_step, 4), "verify_step_ms_during_stage1": round(r["step_ms_during"], 4),
           "step_slowdown_during_stage1": round(r["step_ms_during"] / t_step, 3),
           "stage1_ms_overlapped": round(r["stage1_ms"], 3), "steps_during_stage1": r["steps_during_stage1"],
           "stop_the_world_stall_ms": round(t_stw, 3),
           "two_stage_stall_ms": round(r["stage2_stall_ms"], 3), "two_stage_ssm_ready_ms": round(r["ssm_ready_ms"], 3),
           "stage2_delta_tokens_per_sample": r["delta_tokens"],
           "stall_ratio_two_stage_vs_stw": round(r["stage2_stall_ms"] / t_stw, 4),
           "runs": res_runs,
           "peer_transport": peer,
           "note": "size-1 NCCL communicator (device-local p2p); LLM 32 layers + SSM 1 layer, Llama-3-8B KV "
                   "shapes; stall = time the migrating samples cannot be verified"}
    print(json.dumps(out), flush=True)   # (NCCL may print its version line before it)


if __name__ == "__main__":
    main()
