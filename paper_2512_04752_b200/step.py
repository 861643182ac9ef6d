"""One batched verification step through the C ABI (SURVEY.md §3 call stack (1)):

    rs_tree_build_mask -> rs_tree_verify_attention_layers (L layers) -> rs_tree_accept_compact

(rs_tree_accept_compact = rs_tree_accept + rs_kv_compact in one launch; `fused_commit=False`
issues the two calls separately.)

With `lm_head=(hidden, weight)` (f2) acceptance starts from the nodes' final hidden states:
greedy: rs_lm_head_argmax -> rs_tree_accept_greedy_tokens (the logits are never written);
sampling: rs_lm_head_logits (the bf16 logits from the GEMM epilogue) -> rs_tree_accept_compact.

Pure orchestration: buffers are torch tensors, every computation is a library call; arguments
are marshalled once so a step costs three ctypes calls. The device part can be captured into a
CUDA graph (one launch per step)."""
from __future__ import annotations

import torch

from . import core


class VerifyStep:
    def __init__(self, batch: dict, mode: int = core.GREEDY, temperature: float = 1.0, num_ctas: int = 0,
                 with_lse: bool = False, lm_head=None, fused_commit: bool = True):
        b = batch
        dev = b["q"].device
        self.b = b
        self.mode = mode
        self.temperature = temperature
        self.B, self.Hq, self.Hkv, self.d, self.ps = b["B"], b["Hq"], b["Hkv"], b["d"], b["page_size"]
        # b["L_logical"] > the number of layer buffers: a pool of distinct layer buffers (Q, K, V)
        # cycled so a deep model's step fits in memory (config 5 at 2 GPUs: SURVEY 8(d)); logical
        # layer l uses buffer l % pool, every launch still reads a full layer of K/V from HBM
        n_buf = b["q"].shape[0]
        self.L = int(b.get("L_logical", n_buf))
        self.layer_buf = [l % n_buf for l in range(self.L)]
        self.sm_scale = b["sm_scale"]

        def t32(x):
            return torch.as_tensor(x, dtype=torch.int32).to(dev) if not isinstance(x, torch.Tensor) else x.to(dev)
        self.parent = t32(b["parent"])
        self.token = t32(b["token"])
        self.tree_off = t32(b["tree_off"])
        self.prefix_len = t32(b["prefix_len"])
        self.block_table = t32(b["block_table"])
        self.gid = torch.as_tensor(b["gid"], dtype=torch.int64).to(dev)
        self.q = b["q"]
        self.k_layers = [b["k_cache"][i] for i in self.layer_buf]
        self.v_layers = [b["v_cache"][i] for i in self.layer_buf]
        self.logits = b.get("logits")
        self.hidden, self.lm_w = lm_head if lm_head is not None else (None, None)
        self.draft = b.get("draft_probs") if mode == core.SAMPLE_MSS else None
        # acceptance and the KV commit in one launch (not for the f2 token path, nor for more
        # layers than one launch's parameter block holds)
        self.lm_sampling = self.hidden is not None and mode != core.GREEDY
        self.fused_commit = bool(fused_commit) and self.L <= core.COMPACT_MAX_LAYERS
        self.layer_ptrs = (core._layer_ptrs(self.k_layers), core._layer_ptrs(self.v_layers))
        # MSS: optional row map (draft rows only for nodes with children, Z29)
        self.draft_row = b.get("draft_row") if mode == core.SAMPLE_MSS else None
        if self.draft_row is not None:
            self.draft_row = t32(self.draft_row)
            assert self.fused_commit, "a draft row map needs the fused acceptance call"
        NT = self.q.shape[1]
        self.mask = torch.empty(NT, dtype=torch.int64, device=dev)
        self.depth = torch.empty(NT, dtype=torch.int32, device=dev)
        self.tflags = torch.empty(self.B, dtype=torch.int32, device=dev)
        # host-side plan from this step's lengths (shared by all layers). early_prefix: the prefix
        # K/V (written by the previous step's compaction) may stream before the preceding grid
        # completes, because the mask kernel (a plain launch) always sits between the compaction
        # and the first attention layer, and attention layers write no K/V (header: PDL)
        self.plan = core.AttnPlan(b["prefix_len"], b["tree_off"], self.Hq, self.Hkv, self.d, self.ps,
                                  num_ctas=num_ctas, early_prefix=True)
        self.ws = core.alloc_workspace(self.plan.ws_bytes, dev)
        self.plan.upload(self.ws)
        self.attn_out = torch.empty((self.L, NT, self.Hq, self.d), dtype=torch.bfloat16, device=dev)
        self.lse = torch.empty((self.L, NT, self.Hq), dtype=torch.float32, device=dev) if with_lse else None
        self.acc = torch.empty(self.B, dtype=torch.int32, device=dev)
        self.path = torch.empty((self.B, core.MAX_TREE), dtype=torch.int32, device=dev)
        self.bonus = torch.empty(self.B, dtype=torch.int32, device=dev)
        self.flags = torch.empty(self.B, dtype=torch.int32, device=dev)
        self.new_len = torch.empty(self.B, dtype=torch.int32, device=dev)
        nws = core.accept_workspace_bytes(mode, self.B, b["V"]) if self.hidden is None else 0
        if self.lm_sampling:   # the LM head's logits (written by its epilogue every step)
            self.logits = torch.empty((NT, self.lm_w.shape[0]), dtype=torch.bfloat16, device=dev)
        elif self.hidden is not None:
            self.amax = torch.empty(NT, dtype=torch.int32, device=dev)
            self.lm_ws = torch.empty(max(core.lm_head_argmax_workspace_bytes(NT), 8), dtype=torch.uint8, device=dev)
        self.accept_ws = torch.empty(max(nws, 16), dtype=torch.uint8, device=dev)   # (0 bytes needed today)
        self.attn_call = core.AttentionLayersCall(
            self.plan, [self.q[i] for i in self.layer_buf], self.k_layers, self.v_layers, self.block_table,
            self.prefix_len, self.tree_off, self.mask, self.sm_scale, self.ws,
            [self.attn_out[l] for l in range(self.L)], None if self.lse is None else [self.lse[l] for l in range(self.L)])
        self.graph = None

    def mask_step(self, stream=None):
        core.tree_build_mask(self.parent, self.tree_off, stream=stream, out=(self.mask, self.depth, self.tflags))

    def attention_step(self, stream=None):
        self.attn_call(stream)

    def lm_head_step(self, stream=None):
        if self.lm_sampling:
            core.lm_head_logits(self.hidden, self.lm_w, out=self.logits, stream=stream)

    def accept_step(self, seed, step, stream=None):
        self.lm_head_step(stream)
        if self.hidden is not None and not self.lm_sampling:
            core.lm_head_argmax(self.hidden, self.lm_w, out=(self.amax, None), ws=self.lm_ws, stream=stream)
            core.tree_accept_greedy_tokens(self.amax, self.parent, self.token, self.tree_off,
                                           out=(self.acc, self.path, self.bonus, self.flags), stream=stream)
            return
        core.tree_accept(self.mode, self.logits, self.parent, self.token, self.tree_off, self.gid,
                         draft_probs=self.draft, temperature=self.temperature, seed=seed, step=step,
                         out=(self.acc, self.path, self.bonus, self.flags), stream=stream, ws=self.accept_ws)

    def compact_step(self, stream=None):
        core.kv_compact(self.k_layers, self.v_layers, self.block_table, self.prefix_len, self.acc, self.path,
                        self.ps, new_len=self.new_len, stream=stream)

    def accept_compact_step(self, seed, step, stream=None):
        if self.fused_commit and self.hidden is not None and not self.lm_sampling:
            # f2 greedy: the arg-max GEMM, then the walk with the KV commit in one launch
            core.lm_head_argmax(self.hidden, self.lm_w, out=(self.amax, None), ws=self.lm_ws, stream=stream)
            core.tree_accept_greedy_tokens_compact(self.amax, self.parent, self.token, self.tree_off, self.k_layers,
                                                   self.v_layers, self.block_table, self.prefix_len,
                                                   out=(self.acc, self.path, self.bonus, self.flags),
                                                   new_len=self.new_len, stream=stream, layer_ptrs=self.layer_ptrs)
            return
        if self.fused_commit:
            self.lm_head_step(stream)
            core.tree_accept_compact(self.mode, self.logits, self.parent, self.token, self.tree_off, self.gid,
                                     self.k_layers, self.v_layers, self.block_table, self.prefix_len,
                                     draft_probs=self.draft, temperature=self.temperature, seed=seed, step=step,
                                     out=(self.acc, self.path, self.bonus, self.flags), new_len=self.new_len,
                                     stream=stream, ws=self.accept_ws, layer_ptrs=self.layer_ptrs,
                                     draft_row=self.draft_row)
            return
        self.accept_step(seed, step, stream)
        self.compact_step(stream)

    def device_step(self, seed=0, step=0, stream=None):
        """Enqueue the whole step on `stream` (no host sync)."""
        self.mask_step(stream)
        self.attention_step(stream)
        self.accept_compact_step(seed, step, stream)

    def capture(self, seed=0, step=0, events=None):
        """Capture the device step into a CUDA graph (seed/step are baked in). `events`: optional
        (before_attention, after_attention) torch events recorded inside the graph."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.device_step(seed, step, stream=s)   # warm-up (lazy init outside capture)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            cs = torch.cuda.current_stream()
            self.mask_step(cs)
            if events is not None:
                events[0].record(cs)
            self.attention_step(cs)
            if events is not None:
                events[1].record(cs)
            self.accept_compact_step(seed, step, cs)
        self.graph = g
        return g

    def replay(self):
        self.graph.replay()

    def capture_parts(self, seed=0, step=0):
        """Four CUDA graphs (mask | L x attention | accept | compact) so a caller can time each
        part with events between replays. With the fused commit the third graph is accept +
        compact (one launch) and the fourth is None."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self.device_step(seed, step, stream=s)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        parts = []
        fns = [lambda st: self.mask_step(st), lambda st: self.attention_step(st)]
        if self.fused_commit:
            fns.append(lambda st: self.accept_compact_step(seed, step, st))
        else:
            fns += [lambda st: self.accept_step(seed, step, st), lambda st: self.compact_step(st)]
        for fn in fns:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn(torch.cuda.current_stream())
            parts.append(g)
        if self.fused_commit:
            parts.append(None)
        self.parts = parts
        return parts

    def results(self):
        return dict(accepted_len=self.acc.cpu().numpy(), path=self.path.cpu().numpy(),
                    bonus=self.bonus.cpu().numpy(), flags=self.flags.cpu().numpy(),
                    new_len=self.new_len.cpu().numpy())

    def run(self, seed=0, step=0):
        self.device_step(seed, step)
        return self.results()
