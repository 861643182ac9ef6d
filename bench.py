#!/usr/bin/env python
"""Benchmark of the RLHFSpec verification hot path on B200 (contract: see DESIGN.md §6).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c5g8|tiny] [--impl ours|reference]

A step = mask build + L x tree_verify_attention + tree_accept + kv_compact over one synthetic
batch (all §8(a) rows of the verify path), through the C ABI. Metric: committed
("verified-and-accepted") tokens per second, sum over ranks (weak scaling: every rank is an
independent instance with its own samples). One JSON line is printed by rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "accepted tokens/sec per GPU (verify step) at 1/2/4/8 B200; % roofline"
UNIT = "tokens/s"

WORKLOAD_DESC = {
    "c2": "BASELINE configs[1]: Llama-3-8B shapes (32 q / 8 kv heads, d=128, 32 layers, V=128256), "
          "batch 64, prefix 1K, 16-node tree, greedy",
    "c5g8": "BASELINE configs[4] per-GPU shard at 8 GPUs: Llama-3-70B shapes (64 q / 8 kv, d=128, 80 layers), "
            "16 samples, prefix 8K, 64-node trees, greedy",
    "tiny": "BASELINE configs[0]: 1 sample, prefix 32, 8-node tree, 1 head, d=64, V=1000, greedy",
    "c3": "BASELINE configs[2]: Llama-3-8B shapes, batch 256, prefixes 512-16K lognormal, trees 4-64 "
          "(drawn per sample), rejection sampling (MSS)",
    "c4": "BASELINE configs[3]: one instance per B200, 256 samples per instance (2048 at 8), long-tail "
          "response lengths (LMSYS-shaped lognormal, cap 2048), Llama-3-8B shapes + 1 SSM layer, 16-node "
          "trees, greedy; samples finish and leave; periodic sample reallocation with KV migration (NCCL)",
    "c2lm": "BASELINE configs[1] with the LM head in the step (SURVEY 8(f) f2): Llama-3-8B shapes, batch 64, "
            "prefix 1K, 16-node tree, greedy acceptance from the nodes' final hidden states (4096) through the "
            "fused LM-head arg-max (V=128256), logits never materialised",
    "c5g8lm": "BASELINE configs[4] per-GPU shard at 8 GPUs with the LM head in the step (f2): Llama-3-70B shapes, "
              "16 samples, prefix 8K, 64-node trees, greedy from hidden states (8192) via the fused LM-head arg-max",
    "c5": "BASELINE configs[4]: Llama-3-70B shapes (64 q / 8 kv, d=128, 80 layers), batch 128 sample-sharded "
          "over the N GPUs (128/N per GPU), prefix 8K, 64-node trees, greedy; when 80 layers of KV do not fit one "
          "GPU (N <= 2) a pool of 16 distinct layer buffers is cycled (every launch still reads a full layer)",
    "c3s": "BASELINE configs[2] as the method runs it: Llama-3-8B shapes, batch 256, prefixes 512-16K "
           "lognormal, every tree = S(n) for the n select_strategy picks (host C++, called every step), "
           "rejection sampling (MSS)",
}


# f2 configs: (base config, hidden size of the model whose LM head feeds acceptance)
LM_HEAD = {"c2lm": ("c2", 4096), "c5g8lm": ("c5g8", 8192)}

# select_strategy inputs for configs with ("strategy", n_cand) trees: acceptance
# fit F (knots) and a cost model t_sd = c_draft + b0 + b1*N_seq + b2*N_draft (seconds): b1 from the
# measured attention bytes per token (32 layers x 4 KB at ~4.4 TB/s), b2 the per-token GEMM time of
# an 8B model at the bf16 tensor peak (2 x 8e9 FLOP / 1.5e15), c_draft a ~1 ms draft pass.
STRATEGY_KX = [0.0, 0.05, 0.2, 0.5, 1.0]
STRATEGY_KY = [0.0, 0.15, 0.45, 0.75, 0.95]
STRATEGY_COST = dict(c_draft=1.0e-3, b0=2.0e-4, b1=3.0e-8, b2=1.07e-5, b3=0.0, k_sat=4096.0, seq_bucket=256,
                     draft_bucket=4)


# Llama-3-8B: GEMM parameters a verified token passes through (all projections + FFN of 32 layers +
# the LM head; the embedding lookup is not a GEMM) — the non-attention part of t_sd per token.
GEMM_PARAMS_8B = 8.03e9   # 8.03e9 total - 0.525e9 embedding table + 0.525e9 LM head


class Strategy:
    """a0 as the method runs it on this box: an rs_ctx whose acceptance fit F comes
    from profiling data of this workload and whose t_sd regression comes from rs_calibrate (the
    library's own verification attention timed on a (B, P, T) grid + the dense per-token cost at
    this box's measured GEMM rate); then one n per batch from the candidate trees."""

    def __init__(self, cfg, core, dev, calibrate=True, force_n=None):
        from types import SimpleNamespace
        from synth import draw_prefix_lengths, make_candidate_tree
        self.core, self.cfg = core, cfg
        t0 = time.perf_counter()
        self.ctx = core.Ctx(0, 1, cfg.page_size)
        self.ctx.set_strategy(SimpleNamespace(**STRATEGY_COST), STRATEGY_KX, STRATEGY_KY)   # prior
        self.info = {"prior": {"knots": [STRATEGY_KX, STRATEGY_KY], "cost": STRATEGY_COST}}
        if calibrate:
            self._fit_acceptance(dev)
            self._calibrate_cost(dev)
        self.info["seconds"] = round(time.perf_counter() - t0, 2)
        c, kx, ky = self.ctx.strategy()
        self.knots = (kx, ky)
        self.info["fitted"] = {"knots_x": [round(x, 5) for x in kx], "knots_y": [round(y, 5) for y in ky],
                               "cost": {k: (round(v, 12) if isinstance(v, float) else v) for k, v in c.items()}}
        # the batch: prefixes and candidate trees, flattened once for the per-step host call
        self.P = draw_prefix_lengths(np.random.default_rng(cfg.seed), cfg).astype(np.int32)
        rng = np.random.default_rng(cfg.seed + 77)
        self.cands = [make_candidate_tree(rng, int(cfg.tree[1])) for _ in range(cfg.B)]
        self.flat = self._flatten(self.cands)
        self.selected = np.full((cfg.B, 63), -1, np.int32)
        self.res = self.select() if force_n is None else self.select(n_min=force_n, n_max=force_n)
        self.parents = self._trees(self.cands, self.selected, self.res["n"])

    @staticmethod
    def _flatten(cands):
        off = np.zeros(len(cands) + 1, np.int32)
        off[1:] = np.cumsum([len(p) for p, _ in cands])
        return (np.concatenate([p for p, _ in cands]).astype(np.int32),
                np.concatenate([o for _, o in cands]).astype(np.float64), off)

    @staticmethod
    def _trees(cands, selected, n):
        """Verification trees: root + S(n) in ascending candidate index (Z21)."""
        parents, chosen_all = [], []
        for b in range(len(cands)):
            chosen = sorted(int(x) for x in selected[b][:n])
            idx = {c: i + 1 for i, c in enumerate(chosen)}
            cp = cands[b][0]
            parents.append(np.array([-1] + [0 if cp[c] < 0 else idx[int(cp[c])] for c in chosen], np.int32))
            chosen_all.append(chosen)
        return parents

    def select(self, n_min=3, n_max=63):
        par, o, off = self.flat
        if self.selected.shape[1] != n_max:      # rows of the selection order are [B, n_max]
            self.selected = np.full((self.cfg.B, n_max), -1, np.int32)
        return self.ctx.select(par, o, off, self.P, n_min=n_min, n_max=n_max, patience=2, selected=self.selected)

    def _fit_acceptance(self, dev, B=64, n_prof=48, seeds=8):
        """Offline profiling data for F: a B-sample batch of this workload's recipe (own
        seed), each verification tree = the first n_prof nodes of its candidate tree's search
        (every depth represented), MSS acceptance on the GPU for `seeds` RNG streams; a draft node
        is an observation (dl, accepted) with accepted = 1 iff it is on the accepted path."""
        from dataclasses import replace
        from synth import make_candidate_tree, make_verify_batch
        core = self.core
        pcfg = replace(self.cfg, B=B, L=1, seed=self.cfg.seed + 5000)
        rng = np.random.default_rng(pcfg.seed + 77)
        cands = [make_candidate_tree(rng, int(self.cfg.tree[1])) for _ in range(B)]
        par, o, off = self._flatten(cands)
        sel = np.full((B, n_prof), -1, np.int32)
        self.ctx.select(par, o, off, np.full(B, 1024, np.int32), n_min=n_prof, n_max=n_prof, selected=sel)
        parents = self._trees(cands, sel, n_prof)
        dl_c = core.draft_logits(par, o, off)
        dl_nodes = [dl_c[off[b] + np.array(sorted(int(x) for x in sel[b][:n_prof]))] for b in range(B)]
        vb = make_verify_batch(pcfg, device=dev, gen_device=dev, parents=parents)
        d32 = lambda x: torch.as_tensor(np.asarray(x, np.int32), device=dev)
        args = (vb["logits"], d32(vb["parent"]), d32(vb["token"]), d32(vb["tree_off"]),
                torch.as_tensor(vb["gid"], device=dev))
        xs, ys = [], []
        for s_ in range(seeds):
            acc, path, _, _ = core.tree_accept(core.SAMPLE_MSS, *args, draft_probs=vb["draft_probs"],
                                               temperature=self.cfg.temperature, seed=900 + s_, step=s_)
            acc, path = acc.cpu().numpy(), path.cpu().numpy()
            for b in range(B):
                on = set(int(x) for x in path[b][1:acc[b] + 1])
                xs.append(dl_nodes[b])
                ys.append(np.array([1.0 if i + 1 in on else 0.0 for i in range(n_prof)]))
        x, y = np.concatenate(xs), np.concatenate(ys)
        self.ctx.fit_acceptance(x, y, 16)   # <= 16 knots (rs_tree_select)
        self.info["acceptance_profile"] = {"observations": int(len(x)), "samples": B, "nodes_per_tree": n_prof,
                                           "seeds": seeds, "mean_accepted": round(float(y.mean()), 4)}
        del vb
        torch.cuda.empty_cache()

    def _calibrate_cost(self, dev, layers_distinct=8):
        """t_sd regression on this box (rs_calibrate): dense per-token cost from the library's
        tcgen05 GEMM (rs_lm_head_argmax) rate x the model's GEMM parameters, attention timed on
        a (B, P, T) grid over 32 layers (8 distinct layer pools cycled: each far larger than L2)."""
        core, cfg = self.core, self.cfg
        rows, V, Dm = 4096, cfg.V, 4096
        h = torch.randn(rows, Dm, device=dev).to(torch.bfloat16)
        w = (torch.randn(V, Dm, device=dev) * 0.02).to(torch.bfloat16)
        core.lm_head_argmax(h, w, max_logit=False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            core.lm_head_argmax(h, w, max_logit=False)
        e1.record()
        torch.cuda.synchronize()
        rate = 2.0 * rows * V * Dm * 5 / (e0.elapsed_time(e1) * 1e-3)
        dense = 2.0 * GEMM_PARAMS_8B / rate
        del h, w
        grid = [(B, P, T) for B in (32, 64) for P in (1024, 2048, 4096) for T in (4, 8, 16, 24, 32, 48, 64)]
        pages = max(B * -(-(P + T) // cfg.page_size) for B, P, T in grid)
        kk = [torch.randn(pages, cfg.Hkv, cfg.page_size, cfg.d, device=dev).to(torch.bfloat16)
              for _ in range(layers_distinct)]
        vv = [torch.randn(pages, cfg.Hkv, cfg.page_size, cfg.d, device=dev).to(torch.bfloat16)
              for _ in range(layers_distinct)]
        self.ctx.register_kv(1, [kk[l % layers_distinct] for l in range(cfg.L)],
                             [vv[l % layers_distinct] for l in range(cfg.L)])
        t = self.ctx.calibrate(cfg.Hq, grid, reps=3, dense_s_per_token=dense)
        self.ctx.register_kv(1, [], [])
        del kk, vv
        torch.cuda.empty_cache()
        self.info["calibration"] = {"gemm_TFLOPs": round(rate / 1e12, 1), "dense_s_per_token": dense,
                                    "gemm_params": GEMM_PARAMS_8B, "grid": {"B": [32, 64], "P": [1024, 2048, 4096],
                                                                            "T": [4, 8, 16, 24, 32, 48, 64]},
                                    "attention_ms": [round(x * 1e3, 3) for x in t]}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _relaunch(n):
    """`python bench.py --gpus N` outside torchrun: re-exec under torch.distributed.run with N
    ranks on this node (127.0.0.1 rendezvous); rank 0 prints the line. Returns the exit code."""
    import socket
    import subprocess
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def _device(local):
    """One process per GPU; when ranks outnumber the visible GPUs (a 1-GPU test box) ranks share
    devices round-robin."""
    n = max(1, torch.cuda.device_count())
    return torch.device("cuda", local % n)


def _pg_init(world, dev):
    """Control-plane process group for the bench's barriers and max-over-ranks timing (gloo: CPU
    scalars, works when ranks share a device). The data path has no collective; reallocation's KV
    transfers run in the library (NCCL) or over peer memory, not through this group."""
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")


def _allreduce(x, op="max"):
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, device_index: int, period_s: float = 0.02):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.mem, self.power = [], []
        self.period = period_s
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception as e:  # pragma: no cover - only on boxes without NVML
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.mem.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_MEM))
                self.power.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, v in self.REASONS.items():
                    if r & v and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._ok:
            self.t.join()

    def summary(self):
        if not self._ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "mem_mhz": statistics.median(self.mem) if self.mem else None,
                "power_w_median": round(statistics.median(self.power), 1) if self.power else None}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs"), d.get("bf16_tflops"), d.get("bf16_tflops_sustained"), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


def attention_algorithmic(b):
    """per layer, bytes = sum_b 4*Hkv*d*(P+T) + 4*Hq*d*T + 8*T + 4*ceil((P+T)/64);
    flops = 4*Hq*d*sum_i (P + |anc(i)|)."""
    Hq, Hkv, d = b["Hq"], b["Hkv"], b["d"]
    P = b["prefix_len"].astype(np.int64)
    T = b["T"].astype(np.int64)
    by = int(np.sum(4 * Hkv * d * (P + T) + 4 * Hq * d * T + 8 * T + 4 * ((P + T + 63) // 64)))
    anc = np.zeros(len(b["parent"]), dtype=np.int64)     # |ancestors-or-self| = depth + 1
    for i in range(b["B"]):
        s, e = b["tree_off"][i], b["tree_off"][i + 1]
        for x in range(s, e):
            pa = b["parent"][x]
            anc[x] = 1 if pa < 0 else anc[s + pa] + 1
    fl = 0
    for i in range(b["B"]):
        s, e = b["tree_off"][i], b["tree_off"][i + 1]
        fl += 4 * Hq * d * int(np.sum(P[i] + anc[s:e]))
    return by, fl


def _oracle_sample(job):
    """One whole sample of the workload through the CPU oracle (test infrastructure), in its own
    process with one BLAS/OpenMP thread: the sample's shape (P, tree) is the GPU run's, its
    q/K/V/logits are drawn from the same seeded recipe (synth). Timed: attention over
    `layers_run` of the L layers (extrapolated to L), acceptance and compaction in full. Returns
    (tokens committed, seconds)."""
    import threadpoolctl
    threadpoolctl.threadpool_limits(1)
    torch.set_num_threads(1)
    from oracle import accept as OAcc
    from oracle import attention as OA
    from oracle import compact as OC
    from oracle import tree as OT
    from synth import VerifyConfig, make_verify_batch
    cfg = VerifyConfig(**{**job["cfg"], "B": 1, "prefix": ("fixed", int(job["P"])), "seed": int(job["seed"])})
    L = cfg.L
    lr = max(1, min(L, int(job["layers_run"])))
    # only the layers that are run are drawn (bounded memory at 70B / 8K shapes)
    b = make_verify_batch(cfg, device="cpu", layers=lr,
                          parents=[np.asarray(job["parent"], np.int32)] if job["parent"] is not None else None)
    T = int(b["T"][0])
    masks, _, _ = OT.batch_masks(b["parent"], b["tree_off"])
    lg = b["logits"].contiguous().view(torch.int16).numpy().view(np.uint16)
    kc = [b["k_cache"][l].double().numpy() for l in range(lr)]
    vc = [b["v_cache"][l].double().numpy() for l in range(lr)]
    q = [b["q"][l].double().numpy() for l in range(lr)]
    dp = b["draft_probs"].float().numpy() if cfg.mode == "mss" else None
    om = {"greedy": OAcc.GREEDY, "delta": OAcc.DELTA, "mss": OAcc.MSS}[cfg.mode]
    t0 = time.perf_counter()
    for l in range(lr):
        OA.tree_verify_attention(q[l], kc[l], vc[l], b["block_table"], b["prefix_len"], b["tree_off"], masks,
                                 cfg.Hkv, cfg.page_size, b["sm_scale"])
    t_attn = (time.perf_counter() - t0) * L / lr
    t1 = time.perf_counter()
    acc, path, _, _ = OAcc.tree_accept(om, lg, b["parent"], b["token"], b["tree_off"], b["gid"], cfg.V, draft_probs=dp,
                                       temperature=cfg.temperature, seed=11, step=0)
    t_acc = time.perf_counter() - t1
    t2 = time.perf_counter()
    OC.kv_compact(kc + vc, b["block_table"], b["prefix_len"], acc, path, cfg.page_size)
    t_cmp = (time.perf_counter() - t2) * L / lr
    return int(acc[0]) + 1, t_attn + t_acc + t_cmp, T


def oracle_throughput(cfg, prefix_len, parents, n_procs, rounds=1, layers_run=None, seed0=50000, warmup_rounds=0):
    """The oracle on `n_procs` host cores at once (one process per core, one thread each): every
    process runs `rounds` whole samples of the workload (shapes taken from the GPU batch in
    order, values redrawn from the same recipe). Aggregate rate = sum over processes of
    tokens / busy seconds (the processes run concurrently). Returns (rate, samples, seconds,
    layers_run)."""
    import multiprocessing as mp
    L = cfg.L
    if layers_run is None:
        # bound the fp64 attention: the mean sample's cost scales with P; ~2 s of attention per
        # sample at the configs' shapes
        pm = float(np.mean(prefix_len))
        per_layer = 1.2e-9 * cfg.Hq * cfg.d * pm * 20       # measured order of the einsum oracle (s)
        layers_run = int(max(1, min(L, 2.0 / max(per_layer, 1e-6))))
    base = {k: v for k, v in cfg.__dict__.items()}
    jobs = []
    for r in range(warmup_rounds + rounds):
        for w in range(n_procs):
            i = (r * n_procs + w) % len(prefix_len)
            jobs.append(dict(cfg=base, P=int(prefix_len[i]), parent=None if parents is None else parents[i],
                             seed=seed0 + r * n_procs + w, layers_run=layers_run))
    ctx = mp.get_context("spawn")
    env_keep = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
    os.environ.update(OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
    try:
        with ctx.Pool(n_procs) as pool:
            res = pool.map(_oracle_sample, jobs, chunksize=1)
    finally:
        for k, v in env_keep.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    per_proc = {}
    res = res[warmup_rounds * n_procs:]
    for j, (tok, sec, _) in enumerate(res):
        w = j % n_procs
        a = per_proc.setdefault(w, [0, 0.0])
        a[0] += tok
        a[1] += sec
    rate = sum(t / s for t, s in per_proc.values())
    return rate, len(res), sum(s for _, s in per_proc.values()), layers_run


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_cpu_baseline(cfg, b, parents=None):
    """cpu_baseline: the oracle on ALL host cores (one process each) plus a 1-core run, on
    bounded samples of the workload (the GPU batch's sample shapes)."""
    n = host_cores()
    P = np.asarray(b["prefix_len"])
    t0 = time.perf_counter()
    rate_n, ns_n, sec_n, lr = oracle_throughput(cfg, P, parents, n)
    rate_1, ns_1, sec_1, _ = oracle_throughput(cfg, P, parents, 1, layers_run=lr)
    wall = time.perf_counter() - t0
    return dict(value=round(rate_n, 4), unit=UNIT, cores=n, kind="oracle", value_1core=round(rate_1, 4),
                sample=f"{ns_n} whole samples on {n} cores at once (one process and one BLAS thread each) + "
                       f"{ns_1} on 1 core; sample shapes = the GPU batch's first samples (P, tree), values redrawn "
                       f"from the same synth recipe; attention and compaction timed on {lr} of {cfg.L} layers and "
                       f"scaled to {cfg.L}, accept in full; numpy fp64 + C; {sec_n:.1f} core-s + {sec_1:.1f} s "
                       f"timed, {wall:.0f} s wall with data generation")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default 50; c4: 400)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3s",
                    help="default c3s = BASELINE configs[2] (the largest single-GPU config) as the method runs it")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=20,
                    help="pipelined end-to-end steps (the first upload and the last step's kernels are not overlapped)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-n", type=int, default=None,
                    help="c3s: every tree = S(n) for this n under the prior F (profiling runs: the calibrated "
                         "shapes without the calibration launches)")
    ap.add_argument("--no-lm-variant", action="store_true",
                    help="sampling configs: skip the f2 variant (the LM head in the step) reported beside the line")
    ap.add_argument("--no-calibrate", action="store_true",
                    help="c3s: keep the prior F / t_sd instead of profiling + rs_calibrate at startup")
    ap.add_argument("--realloc", default="on", choices=["on", "off"], help="c4: sample reallocation")
    ap.add_argument("--cooldown", type=int, default=32, help="c4: steps between reallocation checks (P:300)")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="c4: KV migration over peer memory (one push kernel, CUDA IPC) or NCCL send/recv")
    ap.add_argument("--migration", default="blocking", choices=["blocking", "two-stage"],
                    help="c4: stop-the-world rs_migrate_samples or the two-stage migration (f1, P:303-318)")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 400 if args.config == "c4" else 50
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch(args.gpus))
    world, rank, local = _dist()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    assert args.warmup >= 3, "W >= 3 warm-up steps"
    if args.impl == "reference":
        return run_reference(args, world, rank)
    if args.config == "c4":
        return run_c4(args, world, rank, local)
    return run_ours(args, world, rank, local)


def _pack_draft_rows(b, dev):
    """MSS draft rows of the nodes WITH children only, plus the node -> row map (Z29:
    a leaf's draft row is never read, so it is neither stored nor uploaded)."""
    par, off = np.asarray(b["parent"]), np.asarray(b["tree_off"])
    has = np.zeros(len(par), bool)
    for s_ in range(len(off) - 1):
        has[par[off[s_] + 1:off[s_ + 1]] + off[s_]] = True
    idx = np.nonzero(has)[0]
    row = np.full(len(par), -1, np.int32)
    row[idx] = np.arange(len(idx), dtype=np.int32)
    dq = b["draft_probs"].index_select(0, torch.as_tensor(idx, device=b["draft_probs"].device)).contiguous()
    return dq, torch.as_tensor(row, device=dev), has


def run_ours(args, world, rank, local):
    from paper_2512_04752_b200 import core
    from paper_2512_04752_b200.step import VerifyStep
    from synth import CONFIGS, make_lm_head_inputs, make_verify_batch

    dev = _device(local)
    torch.cuda.set_device(dev)
    _pg_init(world, dev)
    lm = LM_HEAD.get(args.config)
    n_buf = None
    if args.config == "c5":
        # configs[4]: B = 128 sample-sharded over the ranks (static split, no exchange)
        assert 128 % world == 0, "c5 splits 128 samples evenly over the GPUs"
        cfg = type(CONFIGS["c5g8"])(**{**CONFIGS["c5g8"].__dict__, "name": "c5", "B": 128 // world})
        pages = cfg.B * -(-(cfg.prefix[1] + cfg.tree[1]) // cfg.page_size)
        per_layer = 2 * pages * cfg.Hkv * cfg.page_size * cfg.d * 2
        n_buf = cfg.L if cfg.L * per_layer <= 100e9 else 16
    else:
        cfg = CONFIGS[lm[0] if lm else args.config]
    cfg = type(cfg)(**{**cfg.__dict__, "seed": cfg.seed + 1000 * rank})   # disjoint samples per rank
    strat = None
    if cfg.tree[0] == "strategy":
        strat = Strategy(cfg, core, dev, calibrate=not (args.no_calibrate or args.force_n), force_n=args.force_n)
        b = make_verify_batch(cfg, device=dev, gen_device=dev, parents=strat.parents)
    else:
        b = make_verify_batch(cfg, device=dev, gen_device=dev, with_logits=lm is None, layers=n_buf)
    if n_buf is not None and n_buf < cfg.L:
        b["L_logical"] = cfg.L
    mode = {"greedy": core.GREEDY, "delta": core.SAMPLE_DELTA, "mss": core.SAMPLE_MSS}[cfg.mode]
    has_kids = None
    if mode == core.SAMPLE_MSS and b.get("draft_probs") is not None:
        b["draft_probs"], b["draft_row"], has_kids = _pack_draft_rows(b, dev)
    lm_in = None
    if lm is not None:
        lm_in = make_lm_head_inputs(b, Dm=lm[1], seed=7 + 1000 * rank, device=dev, gen_device=dev)
        b["hidden"], b["lm_weight"] = lm_in["hidden"], lm_in["weight"]
    step = VerifyStep(b, mode=mode, temperature=cfg.temperature,
                      lm_head=None if lm is None else (lm_in["hidden"], lm_in["weight"]))
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for w in range(args.warmup):
        step.device_step(seed=7, step=w)
    barrier()
    res = step.results()
    tokens_per_step = int(np.sum(res["accepted_len"]) + b["B"])
    accepted_drafts = int(np.sum(res["accepted_len"]))
    info = step.plan.info()

    # ---------------- device-timed region: exactly K steps ----------------
    # events between the graph parts of every timed step: [start, after mask, after attention,
    # after accept, after compact]
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # mask, L x attention (split-KV merge fused), accept (f2: LM-head GEMM + finalize + walk), compact
    launches_per_step = 1 + step.L + (1 if lm is None else 3) + (0 if step.fused_commit else 1)
    # The step's device work is captured once into CUDA graphs (mask | L x attention | accept +
    # compact); every timed step replays them (the launches are still our kernels, counted below).
    g_mask, g_attn, g_acc, g_cmp = step.capture_parts(seed=11, step=0)
    for w in range(args.warmup):
        g_mask.replay(); g_attn.replay(); g_acc.replay()
        if g_cmp is not None:
            g_cmp.replay()
    sampler = ClockSampler(local)
    barrier()
    with sampler:
        start.record(stream)
        sel_s = 0.0
        for k in range(args.steps):
            if strat is not None:
                # a0 (host) for the next step, while the GPU runs the queued graphs
                t0 = time.perf_counter()
                strat.select()
                sel_s += time.perf_counter() - t0
            g_mask.replay()
            ev[k][0].record(stream)
            g_attn.replay()
            ev[k][1].record(stream)
            g_acc.replay()
            ev[k][2].record(stream)
            if g_cmp is not None:
                g_cmp.replay()
            ev[k][3].record(stream)
        end.record(stream)
        torch.cuda.synchronize()
    barrier()
    elapsed_ms = start.elapsed_time(end)
    attn_ms = sum(e[0].elapsed_time(e[1]) for e in ev) / args.steps
    acc_ms = sum(e[1].elapsed_time(e[2]) for e in ev) / args.steps
    cmp_ms = sum(e[2].elapsed_time(e[3]) for e in ev) / args.steps
    if world > 1:
        elapsed_ms = _allreduce(elapsed_ms, "max")
    ms_per_step = elapsed_ms / args.steps
    value = tokens_per_step * world * args.steps / (elapsed_ms / 1e3)

    # ---------------- roofline of the dominant kernel (attention) ----------------
    hbm, tc_burst, tc_sus, peak_src = _peaks()
    # tensor peak: the sustained bf16 figure for a kernel that runs for a long stretch inside the
    # step (attention: L launches back to back, >= 10 ms per step), the burst one for a short
    # kernel (B200_PROFILING.md); which one is used is reported, with the burst fraction beside it
    long_run = attn_ms >= 10.0
    tc_peak, tc_kind = (tc_sus, "sustained") if (tc_sus and long_run) else (tc_burst, "burst")
    host_meta = {k: b[k] for k in ("Hq", "Hkv", "d", "prefix_len", "T", "parent", "tree_off", "B")}
    by, fl = attention_algorithmic(host_meta)
    attn_launch_ms = attn_ms / step.L
    achieved_gbs = by / (attn_launch_ms * 1e-3) / 1e9
    achieved_tf = fl / (attn_launch_ms * 1e-3) / 1e12
    t_hbm = by / (hbm * 1e9)
    t_tc = fl / (tc_peak * 1e12)
    bound = "hbm" if t_hbm >= t_tc else "tensor"
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("dram_bytes_per_launch")
    if bound == "hbm":
        roof = {"bound": "hbm", "achieved": round(achieved_gbs, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved_gbs / hbm, 4), "traffic": traffic}
    else:
        roof = {"bound": "tensor", "achieved": round(achieved_tf, 1), "peak": tc_peak, "unit": "TFLOP/s",
                "frac": round(achieved_tf / tc_peak, 4), "traffic": traffic, "peak_kind": tc_kind,
                "frac_of_burst_peak": round(achieved_tf / tc_burst, 4)}
    roof.update({"kernel": "tree_attn_kernel", "peak_source": peak_src,
                 "algorithmic_bytes_per_launch": by, "algorithmic_flops_per_launch": fl,
                 "launch_ms": round(attn_launch_ms, 5), "attention_share_of_step": round(attn_ms / ms_per_step, 4),
                 "tensor_frac": round(achieved_tf / tc_peak, 4), "tensor_peak_kind": tc_kind})

    # ---------------- per-kernel breakdown (HBM-bound rows against the same peak) ----------------
    path_np, acc_np = res["path"], res["accepted_len"]
    moves = int(sum(int(np.sum(path_np[i, 1:acc_np[i] + 1] != np.arange(1, acc_np[i] + 1))) for i in range(b["B"])))
    esz = 2 if lm is not None or b["logits"].dtype == torch.bfloat16 else 4
    qsz = (b["draft_probs"].element_size() if mode == core.SAMPLE_MSS else 0)
    # visited rows: logits, plus (MSS) the draft row of every visited node that has children
    q_rows = 0
    if has_kids is not None:
        off_np = np.asarray(b["tree_off"])
        q_rows = int(sum(int(has_kids[off_np[i] + path_np[i, :acc_np[i] + 1]].sum()) for i in range(b["B"])))
    acc_bytes = tokens_per_step * cfg.V * esz + q_rows * cfg.V * qsz
    cmp_bytes = 2 * moves * step.L * 4 * cfg.Hkv * cfg.d
    kernels = {
        "attention": {"ms_per_step": round(attn_ms, 4), "launches": step.L, "bytes": by * step.L,
                      "GBps": round(by * step.L / (attn_ms * 1e-3) / 1e9, 1)},
        "accept": {"ms_per_step": round(acc_ms, 4), "launches": 1, "bytes": int(acc_bytes),
                   "GBps": round(acc_bytes / (acc_ms * 1e-3) / 1e9, 1), "frac_hbm": round(acc_bytes / (acc_ms * 1e-3) / 1e9 / hbm, 4),
                   "note": "latency-bound sequential walk: bytes = visited rows x V x dtype"},
        "compact": {"ms_per_step": round(cmp_ms, 4), "launches": 1, "bytes": int(cmp_bytes), "moves": moves,
                    "GBps": round(cmp_bytes / (cmp_ms * 1e-3) / 1e9, 1), "frac_hbm": round(cmp_bytes / (cmp_ms * 1e-3) / 1e9 / hbm, 4)},
        "mask": {"ms_per_step": round(ms_per_step - attn_ms - acc_ms - cmp_ms, 4), "launches": 1,
                 "note": "remainder of the step (mask kernel + graph launch gaps)"},
    }
    if step.fused_commit:
        # one launch commits the K/V in its tail (rs_tree_accept_compact): accept + compact together
        tot = acc_bytes + cmp_bytes
        kernels["accept"] = {"ms_per_step": round(acc_ms + cmp_ms, 4), "launches": 1, "bytes": int(tot),
                             "GBps": round(tot / ((acc_ms + cmp_ms) * 1e-3) / 1e9, 1),
                             "frac_hbm": round(tot / ((acc_ms + cmp_ms) * 1e-3) / 1e9 / hbm, 4),
                             "note": "rs_tree_accept_compact: the walk (bytes = visited rows x V x dtype) with the "
                                     "KV commit fused into each sample's tail"}
        kernels["compact"] = {"fused_into": "accept", "bytes": int(cmp_bytes), "moves": moves}
    if lm is not None:
        lm_flops = 2.0 * b["NT"] * cfg.V * lm[1]
        kernels.pop("accept")
        kernels["lm_head_accept"] = {
            "ms_per_step": round(acc_ms, 4), "launches": 3, "flops": lm_flops,
            "TFLOPs": round(lm_flops / (acc_ms * 1e-3) / 1e12, 1),
            "frac_tensor": round(lm_flops / (acc_ms * 1e-3) / 1e12 / tc_burst, 4), "peak_tflops": tc_burst,
            "peak_kind": "burst (one ~1 ms launch per step)",
            "bound": "tensor", "logits_bytes_not_written": int(b["NT"]) * cfg.V * 2,
            "note": "f2: rs_lm_head_argmax (tcgen05 GEMM [NT x Dm] x [V x Dm]^T, arg-max in the epilogue) "
                    "+ finalize + " + ("rs_tree_accept_greedy_tokens_compact (the walk with the KV commit)"
                                      if step.fused_commit else "rs_tree_accept_greedy_tokens walk")}

    # ---------------- f3: GPU verification-tree construction (timed alone, outside the step) ----------------
    if strat is not None:
        sel_n = strat.res["n"]
        cands = strat.cands
        cpar = torch.as_tensor(np.concatenate([p for p, _ in cands]), dtype=torch.int32, device=dev)
        co = torch.as_tensor(np.concatenate([o for _, o in cands]), dtype=torch.float64, device=dev)
        ctok = torch.randint(0, cfg.V, (cpar.numel(),), dtype=torch.int32, device=dev)
        coff = torch.as_tensor(np.concatenate([[0], np.cumsum([len(p) for p, _ in cands])]), dtype=torch.int32,
                               device=dev)
        rtok = torch.zeros(cfg.B, dtype=torch.int32, device=dev)
        kx = torch.tensor(strat.knots[0], dtype=torch.float64, device=dev)
        ky = torch.tensor(strat.knots[1], dtype=torch.float64, device=dev)
        ts_out = core.tree_select(cpar, co, ctok, coff, rtok, sel_n, kx, ky)
        g_ts = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_ts):
            core.tree_select(cpar, co, ctok, coff, rtok, sel_n, kx, ky, stream=torch.cuda.current_stream(), out=ts_out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g_ts.replay()
        e0.record()
        for _ in range(20):
            g_ts.replay()
        e1.record()
        torch.cuda.synchronize()
        same = bool(torch.equal(ts_out[0].cpu(), torch.as_tensor(b["parent"])))
        kernels["tree_select"] = {"us_per_call": round(e0.elapsed_time(e1) * 1e3 / 20, 2), "launches": 1,
                                  "candidates": int(cpar.numel()), "n": sel_n,
                                  "parents_equal_host_selection": same,
                                  "note": "f3 (SURVEY 8(f)): rs_tree_select timed alone (CUDA graph, 20 calls), "
                                          "not part of the step"}

    # ---------------- end-to-end through the public API with host buffers ----------------
    e2e = run_e2e(step, b, args.e2e_steps, tokens_per_step, world, dev, barrier, mode, cfg.temperature)
    lm_variant = None
    if mode == core.SAMPLE_MSS and lm is None and not args.no_lm_variant:
        lm_variant = run_lm_sampling_variant(args, cfg, b, dev, barrier, world, stream)

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"{args.config}: {WORKLOAD_DESC.get(args.config, args.config)}",
                   "B": cfg.B, "Hq": cfg.Hq, "Hkv": cfg.Hkv, "d": cfg.d, "L": cfg.L, "V": cfg.V,
                   "prefix": list(cfg.prefix), "tree": list(cfg.tree), "accept_mode": cfg.mode,
                   "tokens_per_step": tokens_per_step, "accepted_drafts_per_step": accepted_drafts,
                   "verified_tokens_per_step": int(b["NT"]),
                   "l2": "inputs larger than L2: %.1f GB of distinct per-layer KV resident" %
                         (2 * b["k_cache"].numel() * 2 / 1e9),
                   "parallelism": f"dp{world} (independent sample-sharded instances, no collective)",
                   **({"layer_buffers": n_buf} if n_buf is not None and n_buf < cfg.L else {}),
                   "attn_plan": info,
                   **({"lm_head": {"hidden": lm[1], "fused_argmax": True, "weight_GB": round(cfg.V * lm[1] * 2 / 1e9, 2)}}
                      if lm is not None else {}),
                   **({"select_strategy": {"n": strat.res["n"], "T": strat.res["n"] + 1, "depth": strat.res["depth"],
                                           "width": strat.res["width"], "pred_al": round(strat.res["al"], 2),
                                           "pred_t_sd_ms": round(strat.res["t_sd"] * 1e3, 3),
                                           "host_ms_per_call": round(sel_s / args.steps * 1e3, 4),
                                           "in_timed_loop": True, "strategy_state": strat.info}}
                      if strat is not None else {})},
        "clocks": sampler.summary(),
        "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "roofline": roof,
        "kernels": kernels,
    }
    if lm_variant is not None:
        line["lm_head_variant"] = lm_variant
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = run_cpu_baseline(cfg, b, parents=None if strat is None else strat.parents)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def c4_samples(world, rank, per_rank=256, seed=4):
    """Config 4 workload: per_rank x world samples, round-robin over the instances;
    prompt ~ LogNormal(ln 256, 0.784) in [32, 2048], response LMSYS-shaped capped at 2048
    (P:349). Drawn from one global RNG so every world size sees the same population."""
    from synth import lmsys_response_lengths
    rng = np.random.default_rng(seed)
    n = per_rank * world
    prompt = np.clip(np.rint(rng.lognormal(math.log(256.0), 0.784, size=n)), 32, 2048).astype(np.int32)
    resp = lmsys_response_lengths(rng, n)
    return [(g, int(prompt[g]), int(resp[g])) for g in range(n) if g % world == rank]


def raw_p2p_gbps(world, rank, dev, nbytes=1 << 30):
    """Reference for the migration bandwidth: a raw 1 GiB NCCL send 0 -> 1 on its own NCCL group,
    device-timed on the receiver. Only when ranks own distinct GPUs (NCCL refuses two ranks on
    one device); otherwise None with the reason."""
    import torch.distributed as dist
    if world < 2:
        return None
    if torch.cuda.device_count() < world:
        return {"GBps": None, "why": f"{world} ranks share {torch.cuda.device_count()} GPU(s): no NVLink pair to measure"}
    g = dist.new_group(backend="nccl")
    buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    ms = []
    for it in range(4):
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if rank == 0:
            dist.send(buf, 1, group=g)
        elif rank == 1:
            dist.recv(buf, 0, group=g)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    t = _allreduce(min(ms[1:]) if rank == 1 else 0.0, "max")
    del buf
    return {"GBps": round(nbytes / t / 1e6, 1), "bytes": nbytes, "what": "NCCL send/recv rank 0 -> 1, min of 3"}


def run_c4(args, world, rank, local):
    """BASELINE configs[3]: the verify loop of one generation instance per GPU over a long-tailed
    sample set; samples finish and leave, so loads diverge across instances; with --realloc on
    the instances rebalance every `cooldown` steps (threshold = knee of the measured
    throughput-vs-samples curve) and migrate KV over NCCL. A step is one verify step of
    every instance (host planning + one H2D of metadata + kernels + one D2H of results)."""
    from paper_2512_04752_b200 import core
    from paper_2512_04752_b200.instance import GenerationInstance
    from paper_2512_04752_b200.realloc import Rebalancer

    dev = _device(local)
    torch.cuda.set_device(dev)
    _pg_init(world, dev)
    samples = c4_samples(world, rank)
    L, Hq, Hkv, d, T = 32, 32, 8, 128, 16
    need = sum((p + r + T + 63) // 64 for _, p, r in samples)
    num_pages = int(need * 1.6) + 256
    inst = GenerationInstance(samples, Hq=Hq, Hkv=Hkv, d=d, L=L, V=128256, T=T, p_accept=0.8, num_pages=num_pages,
                              max_pages=72, max_batch=int(len(samples) * 1.5), seed=100 + rank, device=dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # threshold: knee of this instance's throughput-vs-samples curve (measured, not committed),
    # taken on rank 0 and broadcast so every instance plans with the same value
    counts = [8, 16, 32, 64, 96, 128, 192, 256]
    tput = []
    for n in counts:
        inst.step(seed=1, limit=n, commit=False)
        t0 = time.perf_counter()
        tok = sum(inst.step(seed=2 + k, limit=n, commit=False) for k in range(3))
        tput.append(tok / (time.perf_counter() - t0))
    thr = core.knee_threshold(counts, tput, 0.10)
    if world > 1:
        t = torch.tensor([thr], dtype=torch.int64)
        torch.distributed.broadcast(t, 0)
        thr = int(t.item())
    realloc = args.realloc == "on" and world > 1
    reb = Rebalancer(thr, cooldown=args.cooldown) if realloc else None
    # KV transport: peer memory (rs_peer_push into the destination's pages over CUDA IPC / NVLink;
    # works when ranks share a GPU) or NCCL send/recv through a staging buffer (one GPU per rank)
    if realloc and args.transport == "peer":
        comm = inst.connect_peers(rank)
        staging = scratch = None
    else:
        comm = core.Comm(rank, world) if realloc else None
        staging = torch.empty(4 << 30, dtype=torch.uint8, device=dev) if realloc else None
        scratch = torch.empty(3 * 512 + 512 * 72, dtype=torch.int32, device=dev) if realloc else None
    stalls, pushes = [], []
    raw = raw_p2p_gbps(world, rank, dev) if realloc else None

    def one_step(k, timing=False):
        mig = (0, 0, 0, 0.0)
        tok0 = inst.tokens
        if realloc:
            t0 = time.perf_counter()
            if args.migration == "two-stage":   # (its overlap step is a verify step of this loop)
                sent, recv, moved, tm = inst.rebalance_two_stage(reb, comm, staging, scratch, overlap_steps=1,
                                                                 seed=11)
                if tm:
                    stalls.append(tm["stage2_stall_ms"])
            else:
                inst.last_push = None
                sent, recv, moved = inst.rebalance(reb, comm, staging, scratch)
                if inst.last_push:
                    pushes.append(inst.last_push)
            mig = (sent, recv, moved, time.perf_counter() - t0)
        inst.step(seed=11, timing=timing)
        return inst.tokens - tok0, mig

    for w in range(args.warmup):
        one_step(w)
    barrier()
    hbm, _, _, peak_src = _peaks()
    sampler = ClockSampler(local)
    loads, attn_ms, attn_bytes = [], 0.0, 0.0
    tokens = 0
    migrations = []
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        start.record()
        for k in range(args.steps):
            loads.append(inst.load)
            c, mig = one_step(k, timing=True)
            tokens += c
            if mig[0] or mig[1]:
                migrations.append(mig)
            if inst.last_B:
                attn_ms += inst.last_attn_ms
                P = inst.last_prefix.astype(np.float64)
                attn_bytes += L * float(4 * Hkv * d * np.sum(P + T) + 4 * Hq * d * T * inst.last_B + 8 * T * inst.last_B
                                        + 4 * np.sum(np.ceil((P + T) / 64)))
        end.record()
        torch.cuda.synchronize()
    barrier()
    ms = start.elapsed_time(end)
    tok_all, ms_max = tokens, ms
    if world > 1:
        tok_all = int(_allreduce(tokens, "sum"))
        ms_max = _allreduce(ms, "max")
    value = tok_all / (ms_max / 1e3)
    gbs = attn_bytes / (attn_ms * 1e-3) / 1e9 if attn_ms > 0 else 0.0
    mig_bytes = sum(m[2] for m in migrations)
    push_b, push_ms = float(sum(p[0] for p in pushes)), float(sum(p[1] for p in pushes))
    if world > 1:   # push kernels run on the source ranks: totals over every rank
        push_b, push_ms = _allreduce(push_b, "sum"), _allreduce(push_ms, "sum")
    mig_s = sum(m[3] for m in migrations)
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"c4: {WORKLOAD_DESC['c4']}", "samples_per_instance": len(samples),
                   "Hq": Hq, "Hkv": Hkv, "d": d, "L": L, "V": 128256, "tree": ["fixed", T], "accept_mode": "greedy",
                   "realloc": "on" if realloc else "off", "cooldown": args.cooldown, "threshold": thr,
                   "migration": args.migration, "transport": args.transport if realloc else None,
                   "gpus_visible": torch.cuda.device_count(),
                   "knee_profile": {"counts": counts, "tokens_per_s": [round(x, 1) for x in tput]},
                   "load_first_last": [loads[0] if loads else 0, loads[-1] if loads else 0],
                   "finished_samples_rank0": inst.finished, "tokens_rank0": tokens,
                   "l2": "inputs larger than L2: %.1f GB of per-layer KV pools resident" % (
                       2 * (L + 1) * num_pages * Hkv * 64 * d * 2 / 1e9),
                   "parallelism": f"dp{world} (sample-sharded instances; collective only for reallocation)"},
        "clocks": sampler.summary(),
        "e2e": {"value": round(value, 1), "unit": UNIT,
                "h2d_bytes_per_step": int(4 * (len(samples) * (2 + 2 * T + 72) + 1) + 8 * len(samples)),
                "d2h_bytes_per_step": int(8 * len(samples)),
                "note": "the loop is host-driven end to end: every step uploads its metadata and reads back "
                        "accepted_len/new_len; Q and logits are produced on the device upstream (bounds above "
                        "are for the first step's batch)"},
        "gpu_launches": int(args.steps * (L + 3)),
        "roofline": {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(gbs / hbm, 4), "traffic": None, "kernel": "tree_attn_kernel",
                     "peak_source": peak_src, "attention_share_of_step": round(attn_ms / ms, 4)},
        "migration": {"events": len(migrations), "samples_moved_rank0": sum(m[0] + m[1] for m in migrations),
                      "bytes_rank0": int(mig_bytes), "seconds_rank0": round(mig_s, 4),
                      "GBps_rank0": round(mig_bytes / mig_s / 1e9, 2) if mig_s > 0 else None,
                      "note": "GBps_rank0 = KV bytes / host time of the whole reallocation (plan, "
                              "handshake, transfer) on rank 0",
                      "push_kernel_all_ranks": ({"bytes": int(push_b), "ms": round(push_ms, 3),
                                                 "GBps": round(push_b / push_ms / 1e6, 1)} if push_ms > 0 else None),
                      "raw_p2p_reference": raw,
                      **({"two_stage_stall_ms_rank0": [round(x, 3) for x in stalls]} if stalls else {})},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.destroy()
    if world > 1:
        torch.distributed.destroy_process_group()


def run_lm_sampling_variant(args, cfg, b, dev, barrier, world, stream, Dm=4096):
    """f2 for the sampling configs, reported beside the line (the
    hidden-state path is the realistic end-to-end): the same batch (trees, prefixes, KV, Q) with
    the LM head in the step — rs_lm_head_logits (tcgen05 GEMM, bf16 logits from its epilogue)
    then rs_tree_accept_compact — on synthetic final hidden states whose draft rows are noisy
    targets (synth.make_lm_head_sampling_inputs); end to end it uploads hidden states instead
    of logits. Device-timed like the main line (events between graph parts), then e2e."""
    from paper_2512_04752_b200 import core
    from paper_2512_04752_b200.step import VerifyStep
    from synth import make_lm_head_sampling_inputs
    li = make_lm_head_sampling_inputs(b, Dm=Dm, seed=17, device=dev, gen_device=dev)
    bl = dict(b)
    bl["token"] = li["token"]
    bl["draft_probs"] = li["draft_probs"]
    bl.pop("logits", None)
    bl["draft_probs"], bl["draft_row"], _ = _pack_draft_rows(bl, dev)
    del li["draft_probs"]
    st = VerifyStep(bl, mode=core.SAMPLE_MSS, temperature=cfg.temperature, lm_head=(li["hidden"], li["weight"]))
    K = min(args.steps, 20)
    for w in range(args.warmup):
        st.device_step(seed=7, step=w)
    barrier()
    res = st.results()
    tps = int(np.sum(res["accepted_len"]) + b["B"])
    g_mask, g_attn, g_acc, _ = st.capture_parts(seed=11, step=0)
    g_lm = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_lm):
        st.lm_head_step(torch.cuda.current_stream())
    for w in range(args.warmup):
        g_mask.replay(); g_attn.replay(); g_acc.replay()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    s0.record(stream)
    for k in range(K):
        g_mask.replay()
        ev[k][0].record(stream)
        g_attn.replay()
        ev[k][1].record(stream)
        g_acc.replay()
        ev[k][2].record(stream)
    s1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = s0.elapsed_time(s1)
    if world > 1:
        ms = _allreduce(ms, "max")
    acc_ms = sum(e[1].elapsed_time(e[2]) for e in ev) / K
    # the LM head alone (its share of the accept part), 10 replays
    l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g_lm.replay()
    l0.record(stream)
    for _ in range(10):
        g_lm.replay()
    l1.record(stream)
    torch.cuda.synchronize()
    lm_ms = l0.elapsed_time(l1) / 10
    flops = 2.0 * int(b["NT"]) * int(b["V"]) * Dm
    _, tc_burst, _, _ = _peaks()
    e2e = run_e2e(st, bl, args.e2e_steps, tps, world, dev, barrier, core.SAMPLE_MSS, cfg.temperature)
    return {"workload": "the line's batch with the LM head in the step (f2): final hidden states [NT, %d] -> "
                        "rs_lm_head_logits -> MSS acceptance + commit; draft = noisy target (synthetic)" % Dm,
            "value": round(tps * world * K / (ms / 1e3), 1), "unit": UNIT, "ms_per_step": round(ms / K, 4),
            "steps": K, "tokens_per_step": tps,
            "accept_part_ms": round(acc_ms, 4),
            "lm_head": {"ms_alone": round(lm_ms, 4), "flops": flops, "TFLOPs": round(flops / (lm_ms * 1e-3) / 1e12, 1),
                        "frac_burst_bf16": round(flops / (lm_ms * 1e-3) / 1e12 / tc_burst, 4),
                        "logits_bytes_written": int(b["NT"]) * int(b["V"]) * 2},
            "e2e": e2e}


def run_e2e(step, b, n_steps, tokens_per_step, world, dev, barrier, mode, temperature):
    """Same metric end to end through the public API with HOST buffers: every step copies its
    inputs (Q of every layer, logits, draft probabilities for MSS, tree metadata) from pinned
    host memory and reads the results (accepted_len, path, bonus, new_len) back. Two input
    buffer sets on a copy stream let step k+1's upload overlap step k's kernels (the
    double-buffered pipelining a serving loop uses); the timed region spans the first upload to
    the last download."""
    from paper_2512_04752_b200.step import VerifyStep
    compute = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    # a second step object with its own input buffers (KV caches and metadata layout shared)
    # per-step inputs: Q of every layer, then logits (or, f2, the nodes' final hidden states; the
    # LM-head weight is model state, resident like the KV cache), then MSS draft probabilities
    b2 = dict(b)
    b2["q"] = torch.empty_like(step.q)
    lm = step.hidden is not None
    if lm:
        b2["hidden"] = torch.empty_like(step.hidden)
    else:
        b2["logits"] = torch.empty_like(step.logits)
    if step.draft is not None:
        b2["draft_probs"] = torch.empty_like(step.draft)
    if step.draft_row is not None:
        b2["draft_row"] = torch.empty_like(step.draft_row)   # per-step metadata: its own buffer
    step2 = VerifyStep(b2, mode=mode, temperature=temperature,
                       lm_head=(b2["hidden"], step.lm_w) if lm else None)
    steps = [step, step2]
    q_reps = -(-step.L // step.q.shape[0])    # pooled layer buffers: upload Q once per logical layer
    ins = [[s.q] * q_reps + [s.hidden if lm else s.logits] for s in steps]
    h_q = torch.empty(step.q.shape, dtype=step.q.dtype, pin_memory=True).copy_(step.q)
    h_ins = [h_q] * q_reps + [torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t) for t in ins[0][q_reps:]]
    metas = [[s.parent, s.token, s.tree_off, s.prefix_len, s.block_table, s.gid] +
             ([s.draft_row] if s.draft_row is not None else []) for s in steps]
    h_meta = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t) for t in metas[0]]
    h_draft = None
    if step.draft is not None:
        h_draft = torch.empty(step.draft.shape, dtype=step.draft.dtype, pin_memory=True).copy_(step.draft)
    outs = [[s.acc, s.path, s.bonus, s.new_len] for s in steps]
    h_outs = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in outs[0]]
    h2d = sum(t.numel() * t.element_size() for t in h_ins + h_meta)
    if h_draft is not None:
        h2d += h_draft.numel() * h_draft.element_size()
    d2h = sum(t.numel() * t.element_size() for t in h_outs)
    copied = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(compute)
    copy.wait_stream(compute)
    for k in range(n_steps):
        i = k % 2
        st = steps[i]
        with torch.cuda.stream(copy):
            if k >= 2:
                copy.wait_event(done[i])          # buffer i free again (its step finished)
            for t, h in zip(ins[i], h_ins):
                t.copy_(h, non_blocking=True)
            for t, h in zip(metas[i], h_meta):
                t.copy_(h, non_blocking=True)
            if h_draft is not None:
                st.draft.copy_(h_draft, non_blocking=True)
            copied[i].record(copy)
        compute.wait_event(copied[i])
        st.device_step(seed=11, step=k, stream=compute)
        for t, h in zip(outs[i], h_outs):
            h.copy_(t, non_blocking=True)
        done[i].record(compute)
    e.record(compute)
    torch.cuda.synchronize()
    barrier()
    ms = s.elapsed_time(e)
    if world > 1:
        ms = _allreduce(ms, "max")
    return {"value": round(tokens_per_step * world * n_steps / (ms / 1e3), 1), "unit": UNIT,
            "inputs": "Q (all layers) + " + ("final hidden states (f2)" if lm else "logits") +
                      (" + draft probabilities" if step.draft is not None else "") + " + tree metadata",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": n_steps,
            "ms_per_step": round(ms / n_steps, 3),
            "pipelining": "double-buffered inputs: upload of step k+1 overlaps kernels of step k"}


def run_reference(args, world, rank):
    """Reference arm: the CPU oracle as it stands (no reference implementation exists for this
    paper: /root/reference holds only the paper text), on all host cores (one process per core).
    Each step = one whole sample per core of the workload (shapes as the GPU arm draws them,
    values from the same recipe), W warm-up steps untimed. Rank 0 only."""
    if rank != 0:
        return
    from synth import CONFIGS, VerifyConfig, draw_prefix_lengths
    parents = None
    if args.config == "c4":
        # c4's verify step on samples of its population: 8B shapes, prompt + partial response
        # lengths of the long tail (lognormal around 600 tokens), 16-node tree, greedy
        cfg = VerifyConfig("c4", B=256, Hq=32, Hkv=8, d=128, V=128256, L=32, prefix=("lognormal", 600, 0.784, 32, 4096),
                           tree=("fixed", 16), mode="greedy", seed=4)
        P = draw_prefix_lengths(np.random.default_rng(cfg.seed), cfg)
    else:
        cfg = CONFIGS[LM_HEAD[args.config][0] if args.config in LM_HEAD else args.config]
        P = draw_prefix_lengths(np.random.default_rng(cfg.seed), cfg)
        if cfg.tree[0] == "strategy":
            # c3s: the batch's n from the oracle's select_strategy over the batch's candidate trees
            # (same draws as strategy_trees), each sample's tree from the oracle's S(n)
            from oracle import strategy as OS
            from synth import make_candidate_tree
            rng = np.random.default_rng(cfg.seed + 77)
            cands = [make_candidate_tree(rng, int(cfg.tree[1])) for _ in range(cfg.B)]
            c = STRATEGY_COST
            cost = OS.CostModel(c["c_draft"], c["b0"], c["b1"], c["b2"], c["b3"], c["k_sat"], c["seq_bucket"],
                                c["draft_bucket"])
            n = OS.select_strategy(cands, P, STRATEGY_KX, STRATEGY_KY, cost, n_min=3, n_max=63, patience=2)["n"]
            parents = [OS.verification_tree(p_, o_, np.zeros(len(p_), np.int32), 0, n, STRATEGY_KX, STRATEGY_KY)[0]
                       for p_, o_ in cands]
    ncores = host_cores()
    t0 = time.perf_counter()
    rate, nsamp, busy, lr = oracle_throughput(cfg, P, parents, ncores, rounds=args.steps, warmup_rounds=args.warmup)
    wall = time.perf_counter() - t0
    ms_step = 1e3 * busy / max(1, nsamp) * 1.0       # per-core seconds per sample = one step on each core
    line = {"impl": "reference", "metric": METRIC, "value": round(rate, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: {WORKLOAD_DESC.get(args.config, args.config)}",
                       "step": f"one whole sample of the workload per host core ({ncores} processes at once)"},
            "cpu_baseline": {"value": round(rate, 3), "unit": UNIT, "cores": ncores, "kind": "oracle",
                             "sample": f"{nsamp} whole samples ({args.steps} steps x {ncores} cores, {args.warmup} "
                                       f"warm-up steps untimed); attention and compaction timed on {lr} of "
                                       f"{cfg.L} layers and scaled to {cfg.L}; accept in full; numpy fp64 + C, one thread per "
                                       f"process; {wall:.0f} s wall"},
            "e2e": {"value": round(rate, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
