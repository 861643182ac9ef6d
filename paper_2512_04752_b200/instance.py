"""One generation instance running the speculative verify loop over a long-tailed sample set
(BASELINE configs[3]). One process per GPU = one instance.

Per step:
    host: live samples -> page reservations for the tree slots, block tables, lengths, the
          tree tokens of this step, the attention schedule (rs_attn_plan_create)
    device: one H2D of the packed metadata, rs_tree_build_mask, rs_tree_verify_attention_layers
          (L LLM layers), rs_tree_accept_compact (acceptance + the commit of the LLM layers and the
          SSM layer in one launch), one D2H of (accepted_len, new_len)
    host: lengths advance by a_b + 1; a sample whose response is complete leaves and its pages
          return to the pool (the long tail of P:95-101 shrinks the batch).
Every `cooldown` steps the instances rebalance (realloc.Rebalancer: all-gathered loads,
the Eq. 6 greedy plan, sample choice) and move the chosen samples' KV with rs_migrate_samples
(NCCL send/recv).

Synthetic content: Q and the logits are drawn once at the maximum batch size
and addressed by batch position (their values only steer acceptance); every step draws new
tree tokens on the host so that a node's argmax token is one of its children's tokens with
probability p_accept (greedy acceptance is then random per step). KV pages hold N(0, 1)
values; prompts are prefilled upstream (their pages are simply reserved).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import core
from .realloc import Rebalancer, SampleMeta

PAGE = 64


@dataclass
class Sample:
    gid: int
    length: int            # committed tokens with K/V in the cache (P_b)
    remaining: int         # response tokens still to generate
    pages: np.ndarray      # page ids (logical page j -> pages[j])
    steps: int = 0
    accepted: int = 0      # accepted draft tokens so far
    bt_row: np.ndarray = None   # block-table row [max_pages] (tail padded with the last page)

    def set_pages(self, pages, max_pages):
        self.pages = pages
        row = np.empty(max_pages, np.int32)
        row[:len(pages)] = pages
        row[len(pages):] = pages[-1]
        self.bt_row = row

    @property
    def avg_accepted(self) -> float:
        return self.accepted / self.steps if self.steps else 0.0


class GenerationInstance:
    def __init__(self, samples, *, Hq=32, Hkv=8, d=128, L=32, V=128256, T=16, p_accept=0.8,
                 num_pages=8192, max_pages=72, max_batch=None, seed=0, device="cuda", branching=(4, 3, 2, 2, 1)):
        """samples: iterable of (gid, prompt_len, response_len)."""
        from synth.workloads import random_tree_parents
        self.dev = torch.device(device)
        self.Hq, self.Hkv, self.d, self.L, self.V, self.T = Hq, Hkv, d, L, V, T
        self.p_accept = p_accept
        self.max_pages = max_pages
        self.rng = np.random.default_rng(seed)
        gen = torch.Generator(device=self.dev).manual_seed(seed)
        self.pool = core.PagePool(num_pages)
        self.samples: list[Sample] = []
        for gid, p0, r in samples:
            pg = self.pool.alloc(self._pages_for(int(p0) + T))
            if pg is None:
                raise MemoryError("page pool too small for the initial samples")
            smp = Sample(int(gid), int(p0), int(r), pg)
            smp.set_pages(pg, max_pages)
            self.samples.append(smp)
        self.max_batch = int(max_batch or max(len(self.samples), 1))
        # one tree shape for every sample (BFS, node 0 = root); children lists for the tokens
        self.parent = random_tree_parents(np.random.default_rng(seed + 7), T, branching)
        self.kids = [np.nonzero(self.parent == c)[0] for c in range(T)]
        # KV stores: L LLM layers + 1 SSM layer, per-layer page pools [pages, Hkv, 64, d]
        def pool_tensor():
            t = torch.empty((num_pages, Hkv, PAGE, d), dtype=torch.bfloat16, device=self.dev)
            return t.normal_(generator=gen)
        self.k_llm = [pool_tensor() for _ in range(L)]
        self.v_llm = [pool_tensor() for _ in range(L)]
        self.k_ssm, self.v_ssm = [pool_tensor()], [pool_tensor()]
        # synthetic Q and logits at the maximum batch, addressed by batch position
        NTmax = self.max_batch * T
        self.q = torch.randn((L, NTmax, Hq, d), generator=gen, device=self.dev).to(torch.bfloat16)
        logits = torch.randn((NTmax, V), generator=gen, device=self.dev)
        self.spike = self.rng.integers(0, V, size=NTmax).astype(np.int32)   # argmax token of each row
        logits[torch.arange(NTmax, device=self.dev), torch.from_numpy(self.spike).long().to(self.dev)] += 12.0
        self.logits = logits.to(torch.bfloat16)
        del logits
        self.out = torch.empty((L, NTmax, Hq, d), dtype=torch.bfloat16, device=self.dev)
        self._ptrs = (core.ptr_array([self.q[l] for l in range(L)]), core.ptr_array(self.k_llm),
                      core.ptr_array(self.v_llm), core.ptr_array([self.out[l] for l in range(L)]))
        self._kv_ptrs = (core._layer_ptrs(self.k_llm + self.k_ssm), core._layer_ptrs(self.v_llm + self.v_ssm))
        # packed per-step metadata: prefix_len [B] | tree_off [B+1] | parent [NT] | token [NT] |
        # block_table [B, max_pages]; one pinned host buffer, one H2D copy
        cap = self.max_batch * (2 + 2 * T + max_pages) + 1
        self.meta_h = torch.empty(cap, dtype=torch.int32).pin_memory()
        self.meta_d = torch.empty(cap, dtype=torch.int32, device=self.dev)
        self.gid_h = torch.empty(self.max_batch, dtype=torch.int64).pin_memory()
        self.gid_d = torch.empty(self.max_batch, dtype=torch.int64, device=self.dev)
        self.res_h = torch.empty(2 * self.max_batch, dtype=torch.int32).pin_memory()
        self.mask = torch.empty(NTmax, dtype=torch.int64, device=self.dev)
        self.depth = torch.empty(NTmax, dtype=torch.int32, device=self.dev)
        self.tflags = torch.empty(self.max_batch, dtype=torch.int32, device=self.dev)
        self.acc = torch.empty(self.max_batch, dtype=torch.int32, device=self.dev)
        self.path = torch.empty((self.max_batch, core.MAX_TREE), dtype=torch.int32, device=self.dev)
        self.bonus = torch.empty(self.max_batch, dtype=torch.int32, device=self.dev)
        self.aflags = torch.empty(self.max_batch, dtype=torch.int32, device=self.dev)
        self.res_d = torch.empty(2 * self.max_batch, dtype=torch.int32, device=self.dev)
        self.ws = core.alloc_workspace(1 << 20, self.dev)
        self.stream = torch.cuda.Stream(self.dev)
        self._ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        self._tok_next = self._tokens(self.max_batch)
        self.last_attn_ms = 0.0
        self.step_no = 0
        self.tokens = 0            # committed tokens (sum of a_b + 1)
        self.last_push = None      # (bytes, device ms) of the last peer-memory push this rank sourced
        self.finished = 0

    @staticmethod
    def _pages_for(n_tokens: int) -> int:
        return (n_tokens + PAGE - 1) // PAGE

    @property
    def load(self) -> int:
        return len(self.samples)

    # ------------------------------------------------------------------ host side of a step
    def _reserve_tree_slots(self):
        for s in self.samples:
            need = self._pages_for(s.length + self.T)
            if need > self.max_pages:
                raise RuntimeError(f"sample {s.gid}: {s.length} tokens exceed max_pages")
            if need > len(s.pages):
                extra = self.pool.alloc(need - len(s.pages))
                if extra is None:
                    raise MemoryError("page pool exhausted")
                s.set_pages(np.concatenate([s.pages, extra]), self.max_pages)

    def _tokens(self, B: int) -> np.ndarray:
        """Tree tokens of this step: random, except that with probability p_accept one child of
        each internal node carries its parent's argmax token (the row's spike)."""
        T = self.T
        tok = self.rng.integers(0, self.V, size=(B, T)).astype(np.int32)
        rows = np.arange(B) * T
        for c in range(T):
            kids = self.kids[c]
            if len(kids) == 0:
                continue
            hit = self.rng.random(B) < self.p_accept
            pick = kids[self.rng.integers(0, len(kids), size=B)]
            b = np.nonzero(hit)[0]
            tok[b, pick[b]] = self.spike[rows[b] + c]
        return tok.reshape(-1)

    def _pack_meta(self, B: int):
        T, mp = self.T, self.max_pages
        NT = B * T
        m = self.meta_h.numpy()
        o = 0
        pl = m[o:o + B]; o += B
        to = m[o:o + B + 1]; o += B + 1
        par = m[o:o + NT]; o += NT
        tok = m[o:o + NT]; o += NT
        bt = m[o:o + B * mp].reshape(B, mp); o += B * mp
        smp = self.samples
        pl[:] = np.fromiter((x.length for x in smp), np.int32, B)
        bt[:] = np.stack([x.bt_row for x in smp])
        self.gid_h.numpy()[:B] = np.fromiter((x.gid for x in smp), np.int64, B)
        to[:] = np.arange(B + 1, dtype=np.int32) * T
        par[:] = np.tile(self.parent, B)
        tok[:] = self._tok_next[:NT]
        return o, pl.copy(), to.copy()

    # ------------------------------------------------------------------ one verify step
    def step(self, seed: int = 0, limit: int | None = None, commit: bool = True, timing: bool = False):
        """Run one verify step over the live samples (the first `limit` of them); returns the
        committed tokens. commit=False leaves the host state untouched (profiling: the tree
        slots written by the compaction lie beyond the committed lengths). timing=True records
        the attention time of the step in self.last_attn_ms (CUDA events on the step's stream)."""
        all_samples = self.samples
        if limit is not None:
            self.samples = all_samples[:limit]
        try:
            return self._step(seed, commit, timing)
        finally:
            if limit is not None and not commit:
                self.samples = all_samples
            elif limit is not None:
                self.samples = self.samples + all_samples[limit:]

    def _step(self, seed, commit, timing):
        B = len(self.samples)
        if B == 0:
            return 0
        if B > self.max_batch:
            raise RuntimeError(f"batch {B} exceeds max_batch {self.max_batch}")
        T, mp, L = self.T, self.max_pages, self.L
        NT = B * T
        self._reserve_tree_slots()
        n, pl_h, to_h = self._pack_meta(B)
        plan = core.AttnPlan(pl_h, to_h, self.Hq, self.Hkv, self.d, PAGE)
        if plan.ws_bytes > self.ws.numel():
            self.ws = core.alloc_workspace(int(plan.ws_bytes * 1.25), self.dev)
        st = self.stream
        with torch.cuda.stream(st):
            self.meta_d[:n].copy_(self.meta_h[:n], non_blocking=True)
            self.gid_d[:B].copy_(self.gid_h[:B], non_blocking=True)
            md = self.meta_d
            o = 0
            pl = md[o:o + B]; o += B
            to = md[o:o + B + 1]; o += B + 1
            par = md[o:o + NT]; o += NT
            tok = md[o:o + NT]; o += NT
            bt = md[o:o + B * mp].view(B, mp)
            core.tree_build_mask(par, to, stream=st, out=(self.mask[:NT], self.depth[:NT], self.tflags[:B]))
            plan.upload(self.ws, stream=st)
            if timing:
                self._ev[0].record(st)
            qa, ka, va, oa = self._ptrs
            core.tree_verify_attention_layers(plan, L, qa, ka, va, self.k_llm[0].shape[0], bt, pl, to, self.mask[:NT],
                                              self.Hq, self.d, 1.0 / math.sqrt(self.d), oa, self.ws, stream=st)
            if timing:
                self._ev[1].record(st)
            # acceptance + the KV commit of the LLM and SSM layers in one launch
            core.tree_accept_compact(core.GREEDY, self.logits[:NT], par, tok, to, self.gid_d[:B],
                                     self.k_llm + self.k_ssm, self.v_llm + self.v_ssm, bt, pl, seed=seed,
                                     step=self.step_no, out=(self.acc[:B], self.path[:B], self.bonus[:B], self.aflags[:B]),
                                     new_len=self.res_d[B:2 * B], stream=st, layer_ptrs=self._kv_ptrs)
            self.res_d[:B].copy_(self.acc[:B])
            self.res_h[:2 * B].copy_(self.res_d[:2 * B], non_blocking=True)
        self._tok_next = self._tokens(self.max_batch)   # next step's tree tokens while the GPU works
        st.synchronize()
        if timing:
            self.last_attn_ms = self._ev[0].elapsed_time(self._ev[1])
        self.last_B, self.last_prefix = B, pl_h
        r = self.res_h.numpy()
        acc, new_len = r[:B], r[B:2 * B]
        if not commit:
            return int(np.sum(np.minimum(acc + 1, [s.remaining for s in self.samples])))
        committed = 0
        live = []
        for i, s in enumerate(self.samples):
            made = min(int(acc[i]) + 1, s.remaining)
            committed += made
            s.length = int(new_len[i])
            s.remaining -= made
            s.steps += 1
            s.accepted += int(acc[i])
            if s.remaining <= 0:
                self.pool.free(s.pages)
                self.finished += 1
            else:
                live.append(s)
        self.samples = live
        self.tokens += committed
        self.step_no += 1
        return committed

    # ------------------------------------------------------------------ reallocation
    def sample_meta(self):
        return [SampleMeta(s.gid, s.length, s.avg_accepted, s.remaining, s.steps, s.accepted) for s in self.samples]

    def _chunks(self, metas, cap_bytes):
        """Consecutive groups of the transfer whose packed KV (LLM + SSM) fits the staging buffer;
        both ends compute the same groups from the same broadcast list."""
        out, cur = [], []
        for m in metas:
            trial = cur + [m]
            lens = [x.seq_len for x in trial]
            need = 2 * (core.kv_pack_elems(self.L, self.Hkv, self.d, lens) + core.kv_pack_elems(1, self.Hkv, self.d, lens))
            if need > cap_bytes:
                if not cur:
                    raise RuntimeError(f"sample {m.gid} ({m.seq_len} tokens) does not fit the staging buffer")
                out.append(cur)
                cur = [m]
            else:
                cur = trial
        if cur:
            out.append(cur)
        return out

    def rebalance(self, rebalancer: Rebalancer, comm: "core.Comm", staging, scratch, force=False):
        """Collective over all instances (every rank calls it at the same step). Returns
        (#samples sent, #received, KV bytes moved by this rank). `comm` is the NCCL communicator
        (rs_migrate_samples: pack -> send/recv -> unpack through `staging`) or this instance's
        core.PeerStore (rs_peer_push straight into the destination's pages; staging unused)."""
        if isinstance(comm, core.PeerStore):
            return self._rebalance_peer(rebalancer, comm, force)
        transfers = rebalancer.plan(self.load, force=force)
        if not transfers:
            return 0, 0, 0
        transfers = rebalancer.choose(transfers, self.sample_meta())
        cap = staging.numel() * staging.element_size()
        by_gid = {s.gid: s for s in self.samples}
        sent_gids, received = set(), []
        sent = recv = moved = 0
        for tr in transfers:
            if comm.rank not in (tr.src, tr.dst):
                continue
            for chunk in self._chunks(tr.samples, cap):
                gids = [c.gid for c in chunk]
                lens = [c.seq_len for c in chunk]
                src_bt = None
                if comm.rank == tr.src:
                    rows = np.zeros((len(chunk), self.max_pages), np.int32)
                    for i, g in enumerate(gids):
                        pg = by_gid[g].pages
                        rows[i, :len(pg)] = pg
                        rows[i, len(pg):] = pg[-1]
                    with torch.cuda.stream(self.stream):   # allocated + copied on the stream that reads it
                        src_bt = torch.from_numpy(rows).to(self.dev)
                rows = core.migrate_samples(comm, tr.src, tr.dst, (self.k_llm, self.v_llm), (self.k_ssm, self.v_ssm),
                                            PAGE, self.pool if comm.rank == tr.dst else None, gids, lens, src_bt,
                                            self.max_pages, staging, scratch, self.stream)
                moved += 2 * (core.kv_pack_elems(self.L, self.Hkv, self.d, lens) +
                              core.kv_pack_elems(1, self.Hkv, self.d, lens))
                if comm.rank == tr.src:
                    for g in gids:
                        self.pool.free(by_gid.pop(g).pages)
                        sent_gids.add(g)
                        sent += 1
                if comm.rank == tr.dst:   # (src == dst only in the loopback test: moved in place)
                    for i, c in enumerate(chunk):
                        npg = self._pages_for(c.seq_len)
                        rcv = Sample(c.gid, c.seq_len, c.remaining, None, c.steps, c.accepted)
                        rcv.set_pages(rows[i, :npg].copy(), self.max_pages)
                        received.append(rcv)
                        recv += 1
        self.samples = [s for s in self.samples if s.gid not in sent_gids] + received
        return sent, recv, moved

    def rebalance_two_stage(self, rebalancer: Rebalancer, comm: "core.Comm", staging, scratch, overlap_steps=1,
                            seed=0, force=False):
        """Reallocation with the paper's two-stage migration (f1). Collective over all
        instances, like rebalance(). Stage 1 (rs_migrate_stage1) enqueues the chosen samples'
        verified KV on a side stream; every instance then runs `overlap_steps` verify steps — the
        migrating samples keep generating on their source, which only writes slots beyond the
        prefix in flight (Markov property); stage 2 (rs_migrate_stage2) moves the tokens
        committed meanwhile, SSM part first, and the samples change hands with their updated
        state. Only samples that cannot finish during the overlap are chosen. Returns
        (#sent, #received, KV bytes moved by this rank, timing dict in ms). With a core.PeerStore
        as `comm` both stages are rs_peer_push kernels on a side stream (staging unused)."""
        if isinstance(comm, core.PeerStore):
            return self._rebalance_two_stage_peer(rebalancer, comm, overlap_steps, seed, force)
        transfers = rebalancer.plan(self.load, force=force)
        if not transfers:
            return 0, 0, 0, {}
        guard = overlap_steps * self.T                 # a step commits at most T tokens per sample
        transfers = rebalancer.choose(transfers, [m for m in self.sample_meta() if m.remaining > guard])
        cap = staging.numel() * staging.element_size()
        side = torch.cuda.Stream(device=self.dev)
        ev = lambda: torch.cuda.Event(enable_timing=True)

        def src_rows(gids):
            # Allocated and copied ON the side stream that the pack kernels read it from: the copy
            # is ordered before them, and the caching allocator only reuses the block for later
            # side-stream work (core.TwoStageMigration also keeps it referenced until `done`).
            by_gid = {x.gid: x for x in self.samples}
            rows = np.zeros((len(gids), self.max_pages), np.int32)
            for i, g in enumerate(gids):
                pg = by_gid[g].pages
                rows[i, :len(pg)] = pg
                rows[i, len(pg):] = pg[-1]
            with torch.cuda.stream(side):
                return torch.from_numpy(rows).to(self.dev)

        jobs = []
        for tr in transfers:
            if comm.rank not in (tr.src, tr.dst) or not tr.samples:
                continue
            gids = [c.gid for c in tr.samples]
            len1 = [c.seq_len for c in tr.samples]
            reserve = [l + guard for l in len1]
            need = 2 * (core.kv_pack_elems(self.L, self.Hkv, self.d, reserve) +
                        core.kv_pack_elems(1, self.Hkv, self.d, reserve))
            if need > cap:
                raise RuntimeError(f"two-stage migration needs {need} staging bytes > {cap}")
            mig = core.TwoStageMigration(comm, tr.src, tr.dst, (self.k_llm, self.v_llm), (self.k_ssm, self.v_ssm),
                                         PAGE, self.pool if comm.rank == tr.dst else None, self.max_pages, staging,
                                         scratch, side)
            e = [ev() for _ in range(4)]
            e[0].record(side)
            mig.stage1(gids, len1, reserve, src_rows(gids) if comm.rank == tr.src else None)
            e[1].record(side)
            jobs.append((tr, mig, gids, e))
        for k in range(overlap_steps):                 # computation continues while stage 1 streams
            self.step(seed=seed + k)
        # the sources' updated sample state, on every rank (collective, in plan order)
        state = {}
        by_gid = {x.gid: x for x in self.samples}
        for tr in transfers:
            mine = None
            if comm.rank == tr.src:
                mine = [(g.gid, by_gid[g.gid].length, by_gid[g.gid].remaining, by_gid[g.gid].steps,
                         by_gid[g.gid].accepted) for g in tr.samples]
            state[id(tr)] = rebalancer.share(tr, mine)
        sent = recv = moved = 0
        sent_gids, received, timing = set(), [], {}
        for tr, mig, gids, e in jobs:
            upd = state[id(tr)]
            len2 = [u[1] for u in upd]
            e[2].record(side)
            mig.stage2(len2, src_rows(gids) if comm.rank == tr.src else None)
            e[3].record(side)
            side.synchronize()
            timing = {"stage1_ms": e[0].elapsed_time(e[1]), "stage2_stall_ms": e[2].elapsed_time(e[3]),
                      "delta_tokens": int(sum(len2) - sum(c.seq_len for c in tr.samples))}
            if comm.rank == tr.dst:
                timing["ssm_ready_ms"] = e[2].elapsed_time(mig.ssm_ready)
            moved += 2 * (core.kv_pack_elems(self.L, self.Hkv, self.d, len2) +
                          core.kv_pack_elems(1, self.Hkv, self.d, len2))
            if comm.rank == tr.src:
                self._migrated_from = {g: by_gid[g].pages.copy() for g in gids}   # (tests: old pages)
                for g in gids:
                    self.pool.free(by_gid[g].pages)
                    sent_gids.add(g)
                    sent += 1
            if comm.rank == tr.dst:
                rows = mig.dst_rows()
                for i, (g, length, rem, steps, acc) in enumerate(upd):
                    npg = self._pages_for(int(mig.capacity[i]))
                    rcv = Sample(g, length, rem, None, steps, acc)
                    rcv.set_pages(rows[i, :npg].copy(), self.max_pages)
                    received.append(rcv)
                    recv += 1
        self.samples = [x for x in self.samples if x.gid not in sent_gids] + received
        return sent, recv, moved, timing

    # ------------------------------------------------------------------ migration over peer memory
    def connect_peers(self, rank: int, pg=None) -> "core.PeerStore":
        """Register this instance's KV pools (LLM + SSM) for peer-memory migration and map every
        other instance's (collective over the torch.distributed group)."""
        store = core.PeerStore((self.k_llm, self.v_llm), (self.k_ssm, self.v_ssm), PAGE, rank)
        return core.peer_connect(store, pg)

    def _kv_bytes(self, lens) -> int:
        return 2 * (core.kv_pack_elems(self.L, self.Hkv, self.d, lens) + core.kv_pack_elems(1, self.Hkv, self.d, lens))

    def _src_rows(self, gids, stream):
        """Device block-table rows of this instance's samples `gids`, allocated and copied on the
        stream whose kernels read them."""
        by_gid = {x.gid: x for x in self.samples}
        rows = np.stack([by_gid[g].bt_row for g in gids]).astype(np.int32)
        with torch.cuda.stream(stream):
            return torch.from_numpy(rows).to(self.dev, non_blocking=False)

    def _to_dev(self, x, stream):
        with torch.cuda.stream(stream):
            return torch.from_numpy(np.ascontiguousarray(x, dtype=np.int32)).to(self.dev)

    def _rebalance_peer(self, rebalancer: Rebalancer, store: "core.PeerStore", force=False):
        """Stop-the-world reallocation with peer-memory migration. Per transfer (plan order, every
        rank takes part in the control-plane broadcasts): the destination reserves pages for the
        chosen samples all-or-nothing and broadcasts its rows (None = refused: the source
        keeps its samples); the source pushes every layer's KV into those pages with one kernel
        per model (SSM first) on the instance stream, records its event and broadcasts that it
        did; the destination's stream waits on the event, so its next step sees the pages."""
        transfers = rebalancer.plan(self.load, force=force)
        if not transfers:
            return 0, 0, 0
        transfers = rebalancer.choose(transfers, self.sample_meta())
        rank = store.rank
        sent = recv = moved = 0
        sent_gids, received, pushes = set(), [], []
        for tr in transfers:
            if not tr.samples:
                continue
            lens = [c.seq_len for c in tr.samples]
            gids = [c.gid for c in tr.samples]
            rows = self.pool.reserve(lens, PAGE, self.max_pages) if rank == tr.dst else None
            rows = rebalancer.share_from(tr.dst, rows)
            if rows is None:
                continue                                   # refused: nothing moves
            if rank == tr.src:
                st = self.stream
                sbt, dbt, ln = self._src_rows(gids, st), self._to_dev(rows, st), self._to_dev(lens, st)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                store.push(tr.dst, sbt, dbt, ln, stream=st)
                e1.record(st)
                pushes.append((self._kv_bytes(lens), e0, e1))
                store.signal(core.PEER_DONE, st)
                by_gid = {x.gid: x for x in self.samples}
                self._migrated = {g: (by_gid[g].bt_row.copy(), by_gid[g].length) for g in gids}   # (tests)
                for g in gids:
                    self.pool.free(by_gid[g].pages)        # reused only by later work on this stream
                    sent_gids.add(g)
                    sent += 1
                moved += self._kv_bytes(lens)
            rebalancer.share_from(tr.src, True)            # the source's signal is enqueued
            if rank == tr.dst:
                store.wait(tr.src, core.PEER_DONE, self.stream)
                for i, c in enumerate(tr.samples):
                    npg = self._pages_for(c.seq_len)
                    rcv = Sample(c.gid, c.seq_len, c.remaining, None, c.steps, c.accepted)
                    rcv.set_pages(np.asarray(rows[i, :npg]).copy(), self.max_pages)
                    received.append(rcv)
                    recv += 1
                moved += self._kv_bytes(lens)
        self.samples = [s for s in self.samples if s.gid not in sent_gids] + received
        if pushes:   # device time of this rank's push kernels (source side)
            pushes[-1][2].synchronize()
            self.last_push = (sum(p[0] for p in pushes), sum(p[1].elapsed_time(p[2]) for p in pushes))
        return sent, recv, moved

    def _rebalance_two_stage_peer(self, rebalancer: Rebalancer, store: "core.PeerStore", overlap_steps=1, seed=0,
                                  force=False):
        """Two-stage migration (f1) over peer memory. Stage 1: the destination reserves
        pages for the verified length plus the tokens the overlap can add, the source pushes the
        verified prefix on a side stream and every instance keeps verifying (the source writes
        only slots beyond the prefix in flight). Stage 2: the source shares the samples'
        updated state, the destination extends a row that outgrew its reservation, and the
        source pushes the tokens committed meanwhile, SSM part first (its event lets the
        destination resume drafting), then the LLM part; the destination's stream waits
        on the source's events."""
        transfers = rebalancer.plan(self.load, force=force)
        if not transfers:
            return 0, 0, 0, {}
        guard = overlap_steps * self.T
        transfers = rebalancer.choose(transfers, [m for m in self.sample_meta() if m.remaining > guard])
        rank = store.rank
        side = torch.cuda.Stream(device=self.dev)
        ev = lambda: torch.cuda.Event(enable_timing=True)
        jobs = []
        for tr in transfers:
            if not tr.samples:
                continue
            gids = [c.gid for c in tr.samples]
            len1 = [c.seq_len for c in tr.samples]
            reserve = [l + guard for l in len1]
            rows = self.pool.reserve(reserve, PAGE, self.max_pages) if rank == tr.dst else None
            rows = rebalancer.share_from(tr.dst, rows)
            if rows is None:
                continue
            e = [ev() for _ in range(4)]
            if rank == tr.src:
                side.wait_stream(self.stream)
                e[0].record(side)
                store.push(tr.dst, self._src_rows(gids, side), self._to_dev(rows, side), self._to_dev(len1, side),
                           stream=side)
                e[1].record(side)
            jobs.append((tr, gids, len1, np.asarray(rows).copy(), [self._pages_for(r) for r in reserve], e))
        for k in range(overlap_steps):                 # computation continues while stage 1 streams
            self.step(seed=seed + k)
        by_gid = {x.gid: x for x in self.samples}
        sent = recv = moved = 0
        sent_gids, received, timing = set(), [], {}
        for tr, gids, len1, rows, have, e in jobs:
            mine = None
            if rank == tr.src:
                mine = [(g, by_gid[g].length, by_gid[g].remaining, by_gid[g].steps, by_gid[g].accepted) for g in gids]
            upd = rebalancer.share(tr, mine)
            len2 = [u[1] for u in upd]
            if rank == tr.dst:                         # extend rows that outgrew the reservation
                need = [self._pages_for(l) for l in len2]
                extra = sum(max(0, n - h) for n, h in zip(need, have))
                pages = self.pool.alloc(extra) if extra else np.zeros(0, np.int32)
                if pages is None:
                    raise MemoryError("two-stage migration: destination pool exhausted at stage 2")
                o = 0
                for i, (n, h) in enumerate(zip(need, have)):
                    if n > h:
                        rows[i, h:n] = pages[o:o + n - h]
                        rows[i, n:] = rows[i, n - 1]
                        o += n - h
                        have[i] = n
            rows = rebalancer.share_from(tr.dst, rows if rank == tr.dst else None)
            delta = [b - a for a, b in zip(len1, len2)]
            if rank == tr.src:
                side.wait_stream(self.stream)          # the overlap steps' KV writes
                e[2].record(side)
                sbt, dbt = self._src_rows(gids, side), self._to_dev(rows, side)
                st_d, dl_d = self._to_dev(len1, side), self._to_dev(delta, side)
                store.push(tr.dst, sbt, dbt, dl_d, starts=st_d, parts=core.PEER_SSM, stream=side)
                store.signal(core.PEER_SSM_READY, side)
                store.push(tr.dst, sbt, dbt, dl_d, starts=st_d, parts=core.PEER_LLM, stream=side)
                store.signal(core.PEER_DONE, side)
                e[3].record(side)
                self.stream.wait_stream(side)          # pages are freed below: later work is ordered after
                self._migrated = {g: (by_gid[g].bt_row.copy(), by_gid[g].length) for g in gids}   # (tests)
                for g in gids:
                    self.pool.free(by_gid[g].pages)
                    sent_gids.add(g)
                    sent += 1
                moved += self._kv_bytes(len2)
            rebalancer.share_from(tr.src, True)
            if rank == tr.dst:
                t0 = ev()
                t1 = ev()
                t0.record(self.stream)
                store.wait(tr.src, core.PEER_SSM_READY, self.stream)
                store.wait(tr.src, core.PEER_DONE, self.stream)
                t1.record(self.stream)
                for i, (g, length, rem, steps, acc) in enumerate(upd):
                    rcv = Sample(g, length, rem, None, steps, acc)
                    rcv.set_pages(rows[i, :have[i]].copy(), self.max_pages)
                    received.append(rcv)
                    recv += 1
                moved += self._kv_bytes(len2)
            if rank == tr.src:
                side.synchronize()
                timing = {"stage1_ms": e[0].elapsed_time(e[1]), "stage2_stall_ms": e[2].elapsed_time(e[3]),
                          "delta_tokens": int(sum(delta))}
        self.samples = [x for x in self.samples if x.gid not in sent_gids] + received
        return sent, recv, moved, timing
