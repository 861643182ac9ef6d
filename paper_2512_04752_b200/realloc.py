"""Sample reallocation across generation instances (§6.1-6.2): the control
plane around the library's planner (rs_plan_reallocation / rs_choose_samples, host C++) and its
data plane (rs_migrate_samples, NCCL). One process per GPU = one instance.

Every `cooldown` steps each rank contributes its load; all ranks compute the same plan
from the same all-gathered loads (the planner is deterministic), each source picks its samples
(shorter sequence first, then lower average accepted tokens), and every transfer runs as
one collective call between its source and destination. Sample metadata (gid, length, average
accepted) moves over the torch.distributed group; KV bytes move over NCCL in the library.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import core


@dataclass
class SampleMeta:
    gid: int
    seq_len: int
    avg_accepted: float
    remaining: int = 0      # sample state that travels with it (response tokens still to
    steps: int = 0          # generate, verify steps so far, accepted drafts so far)
    accepted: int = 0


@dataclass
class Transfer:
    src: int
    dst: int
    count: int
    samples: list = field(default_factory=list)   # SampleMeta chosen by the source


class Rebalancer:
    def __init__(self, threshold: int, cooldown: int = 32, pg=None):
        self.threshold = int(threshold)
        self.cooldown = int(cooldown)
        self.pg = pg
        self.steps_since = 0

    @staticmethod
    def threshold_from_profile(counts, tput, frac: float = 0.10) -> int:
        """Knee of the instance's throughput-vs-samples roofline (reading Z13)."""
        return core.knee_threshold(counts, tput, frac)

    def gather_loads(self, local_load: int) -> list[int]:
        world = dist.get_world_size(self.pg)
        t = torch.tensor([int(local_load)], dtype=torch.int64)
        if dist.get_backend(self.pg) == "nccl":
            t = t.cuda()
        out = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(out, t, group=self.pg)
        return [int(x.item()) for x in out]

    def should_trigger(self, loads) -> bool:
        """P:300 trigger (rs_realloc_should_trigger, host C++)."""
        return core.realloc_should_trigger(loads, self.threshold, self.steps_since, self.cooldown)

    def plan(self, local_load: int, force: bool = False) -> list[Transfer]:
        """Collective: identical plan on every rank (empty when not triggered)."""
        self.steps_since += 1
        loads = self.gather_loads(local_load)
        if not force and not self.should_trigger(loads):
            return []
        self.steps_since = 0
        return [Transfer(s, d, c) for s, d, c in core.plan_reallocation(loads, self.threshold)]

    def choose(self, transfers: list[Transfer], local_samples: list[SampleMeta]) -> list[Transfer]:
        """Collective: each source picks its samples; the choice is broadcast so the destination
        knows the gids, lengths and statistics it is about to receive."""
        rank = dist.get_rank(self.pg)
        for tr in transfers:
            payload = [None]
            if rank == tr.src:
                gid = np.array([s.gid for s in local_samples], np.int64)
                sl = np.array([s.seq_len for s in local_samples], np.int32)
                aa = np.array([s.avg_accepted for s in local_samples], np.float64)
                # never more than the source has eligible (the caller may filter its samples,
                # e.g. two-stage migration keeps only those that outlive the overlap): a short
                # or empty payload is broadcast instead of failing here while the other ranks
                # wait in the collective below; the destination takes what it receives
                k = min(int(tr.count), len(local_samples))
                chosen = set(core.choose_samples(gid, sl, aa, k)) if k > 0 else set()
                payload = [[s for s in local_samples if s.gid in chosen]]
                payload[0].sort(key=lambda s: (s.seq_len, s.avg_accepted, s.gid))
            src_global = dist.get_global_rank(self.pg, tr.src) if self.pg is not None else tr.src
            dist.broadcast_object_list(payload, src=src_global, group=self.pg)
            tr.samples = payload[0]
        return transfers

    def share(self, tr: Transfer, payload):
        """Collective: the source's payload for transfer tr (any picklable object), on every rank."""
        return self.share_from(tr.src, payload)

    def share_from(self, rank: int, payload):
        """Collective: `rank`'s payload (any picklable object), on every rank."""
        obj = [payload]
        src_global = dist.get_global_rank(self.pg, rank) if self.pg is not None else rank
        dist.broadcast_object_list(obj, src=src_global, group=self.pg)
        return obj[0]


def execute(transfers: list[Transfer], comm: "core.Comm", llm_layers, ssm_layers, page_size: int,
            pool: "core.PagePool", block_table_of, max_pages: int, staging, scratch, stream=None):
    """Data plane: run each transfer through rs_migrate_samples (both ends call it; other ranks
    skip). block_table_of(gids) -> device int32 [n, max_pages] rows of the source's samples.
    Returns {gid: new block-table row} for the samples this rank received."""
    received = {}
    for tr in transfers:
        if comm.rank not in (tr.src, tr.dst):
            continue
        gids = [s.gid for s in tr.samples]
        lens = [s.seq_len for s in tr.samples]
        src_bt = block_table_of(gids) if comm.rank == tr.src else None
        rows = core.migrate_samples(comm, tr.src, tr.dst, llm_layers, ssm_layers, page_size,
                                    pool if comm.rank == tr.dst else None, gids, lens, src_bt, max_pages,
                                    staging, scratch, stream)
        if rows is not None:
            received.update({g: rows[i] for i, g in enumerate(gids)})
    return received
