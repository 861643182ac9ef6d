"""Thin Python binding over librlhfspec_core.so (ctypes). Argument marshalling only: every step
of the hot path runs in the library's CUDA kernels / C++ host code. There is no fallback — if
the library is missing, importing this module raises.

Names follow the C ABI in include/rlhfspec_core.h (without the `rs_` prefix)."""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RS_CORE_LIB") or os.path.join(_HERE, "librlhfspec_core.so")   # RS_CORE_LIB: profiling variants
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2512_04752_b200.build` "
                      "(the CUDA path has no fallback)")
_lib = ctypes.CDLL(LIB_PATH)

GREEDY, SAMPLE_DELTA, SAMPLE_MSS = 0, 1, 2
DTYPE_BF16, DTYPE_F32 = 0, 1
FLAG_MALFORMED, FLAG_NONFINITE = 1, 2
MAX_TREE = 64
COMPACT_MAX_LAYERS = 256   # rs_tree_accept_compact: layers one launch commits

_P = ctypes.c_void_p
_i32, _i64, _u64, _f32, _f64, _sz = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float,
                                     ctypes.c_double, ctypes.c_size_t)


def _sig(name, restype, *argtypes):
    fn = getattr(_lib, name)
    fn.restype = restype
    fn.argtypes = list(argtypes)
    return fn


_lib.rs_last_error.restype = ctypes.c_char_p
_lib.rs_version.restype = ctypes.c_char_p
_sig("rs_tree_build_mask", _i32, _P, _P, _i32, _P, _P, _P, _P)
_sig("rs_attn_plan_create", _i32, _P, _P, _i32, _i32, _i32, _i32, _i32, _i32, ctypes.POINTER(_P))
_sig("rs_attn_plan_workspace_bytes", _sz, _P)
_sig("rs_attn_plan_upload", _i32, _P, _P, _sz, _P)
_sig("rs_attn_plan_info", _i32, _P, ctypes.POINTER(_i32), ctypes.POINTER(_i32), ctypes.POINTER(_i32))
_sig("rs_attn_plan_destroy", None, _P)
_sig("rs_attn_plan_items", _i32, _P, _P, _P)
_sig("rs_attn_plan_set_early_prefix", _i32, _P, _i32)
_sig("rs_attn_set_trace", _i32, _P, _sz)
_sig("rs_tree_verify_attention", _i32, _P, _P, _P, _P, _i64, _P, _i32, _P, _P, _P, _i32, _i32, _i32,
     _i32, _i32, _f32, _P, _P, _P, _sz, _P)
_sig("rs_tree_verify_attention_layers", _i32, _P, _i32, _P, _P, _P, _i64, _P, _i32, _P, _P, _P, _i32, _i32,
     _i32, _i32, _i32, _f32, _P, _P, _P, _sz, _P)
_sig("rs_tree_accept", _i32, _i32, _P, _i32, _P, _P, _P, _P, _P, _i32, _i32, _f32, _u64, _u64, _P, _P,
     _P, _P, _P, _sz, _P)
_sig("rs_tree_accept_workspace_bytes", _sz, _i32, _i32, _i32)
_sig("rs_tree_accept_ex", _i32, _i32, _P, _i32, _P, _i32, _P, _P, _P, _P, _i32, _i32, _f32, _u64, _u64, _P, _P,
     _P, _P, _P, _sz, _P)
_sig("rs_philox4x32_10", _i32, _P, _i64, _P, _P, _P)
_sig("rs_exp_spec", _i32, _P, _i64, _P, _P)
_sig("rs_kv_compact", _i32, _P, _P, _i32, _i64, _i32, _i32, _i32, _P, _i32, _P, _P, _P, _i32, _P, _P, _P)
_sig("rs_tree_accept_compact", _i32, _i32, _P, _i32, _P, _i32, _P, _P, _P, _P, _P, _i32, _i32, _f32, _u64, _u64,
     _P, _P, _P, _P, _P, _sz, _P, _P, _i32, _i32, _i32, _i32, _P, _i32, _P, _P, _P, _P)


class RSError(RuntimeError):
    pass


def _check(status: int, what: str):
    if status != 0:
        raise RSError(f"{what} failed (status {status}): {_lib.rs_last_error().decode()}")


def version() -> str:
    return _lib.rs_version().decode()


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _host_i32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


# ------------------------------------------------------------------ a1
def tree_build_mask(parent: torch.Tensor, tree_off: torch.Tensor, stream=None, out=None):
    B = tree_off.numel() - 1
    NT = parent.numel()
    if out is None:
        out = (torch.empty(NT, dtype=torch.int64, device=parent.device),
               torch.empty(NT, dtype=torch.int32, device=parent.device),
               torch.empty(B, dtype=torch.int32, device=parent.device))
    mask, depth, flags = out
    _check(_lib.rs_tree_build_mask(_ptr(parent), _ptr(tree_off), B, _ptr(mask), _ptr(depth), _ptr(flags),
                                   _stream(stream)), "rs_tree_build_mask")
    return mask, depth, flags


# ------------------------------------------------------------------ f3
_sig("rs_tree_select", _i32, _P, _P, _P, _P, _P, _i32, _i32, _P, _P, _i32, _P, _P, _P, _P, _P, _P)
FLAG_INSUFFICIENT = 4


def tree_select(cand_parent, cand_o, cand_token, cand_off, root_token, n, knots_x, knots_y, stream=None, out=None):
    """Verification trees (root + S(n)) for every sample, built on the device. Returns
    (parent, token, mask, depth, flags); tree b occupies rows b*(n+1) .. b*(n+1)+n."""
    B = cand_off.numel() - 1
    dev = cand_parent.device
    NT = B * (n + 1)
    if out is None:
        out = (torch.empty(NT, dtype=torch.int32, device=dev), torch.empty(NT, dtype=torch.int32, device=dev),
               torch.empty(NT, dtype=torch.int64, device=dev), torch.empty(NT, dtype=torch.int32, device=dev),
               torch.empty(B, dtype=torch.int32, device=dev))
    par, tok, mask, dep, flags = out
    _check(_lib.rs_tree_select(_ptr(cand_parent), _ptr(cand_o), _ptr(cand_token), _ptr(cand_off), _ptr(root_token),
                               B, int(n), _ptr(knots_x), _ptr(knots_y), knots_x.numel(), _ptr(par), _ptr(tok),
                               _ptr(mask), _ptr(dep), _ptr(flags), _stream(stream)), "rs_tree_select")
    return par, tok, mask, dep, flags


# ------------------------------------------------------------------ a2
class AttnPlan:
    """Host schedule for one verify step (lengths of this step), shared by every layer."""

    def __init__(self, prefix_len_host, tree_off_host, Hq, Hkv, head_dim, page_size=64, num_ctas=0,
                 early_prefix=False):
        self._pl = _host_i32(prefix_len_host)
        self._to = _host_i32(tree_off_host)
        self.B, self.Hq, self.Hkv, self.head_dim, self.page_size = len(self._pl), Hq, Hkv, head_dim, page_size
        h = _P()
        _check(_lib.rs_attn_plan_create(_ptr(self._pl), _ptr(self._to), self.B, Hq, Hkv, head_dim, page_size,
                                        num_ctas, ctypes.byref(h)), "rs_attn_plan_create")
        self.handle = h
        self.ws_bytes = int(_lib.rs_attn_plan_workspace_bytes(h))
        if early_prefix:
            _check(_lib.rs_attn_plan_set_early_prefix(h, 1), "rs_attn_plan_set_early_prefix")

    def info(self):
        a, b, c = _i32(), _i32(), _i32()
        _check(_lib.rs_attn_plan_info(self.handle, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)),
               "rs_attn_plan_info")
        return dict(num_ctas=a.value, num_items=b.value, num_split_units=c.value)

    def schedule(self):
        """(cta_off [num_ctas+1], items [num_items, 12]) as numpy arrays (fields: rs_attn_plan_items)."""
        inf = self.info()
        cta = np.zeros(inf["num_ctas"] + 1, dtype=np.int32)
        items = np.zeros((inf["num_items"], 12), dtype=np.int32)
        _check(_lib.rs_attn_plan_items(self.handle, _ptr(cta), _ptr(items)), "rs_attn_plan_items")
        return cta, items

    def upload(self, ws: torch.Tensor, stream=None):
        _check(_lib.rs_attn_plan_upload(self.handle, _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)),
               "rs_attn_plan_upload")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            _lib.rs_attn_plan_destroy(h)
            self.handle = None


def attn_set_trace(buf):
    """Profiling: per-(CTA, block, event) clock64 timestamps of every attention launch (None = off)."""
    _check(_lib.rs_attn_set_trace(_ptr(buf), 0 if buf is None else buf.numel() * buf.element_size()),
           "rs_attn_set_trace")


def alloc_workspace(nbytes: int, device="cuda") -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def tree_verify_attention(plan: AttnPlan, q, k_pages, v_pages, block_table, prefix_len, tree_off, tree_mask,
                          sm_scale, ws, out=None, lse=None, stream=None):
    NT, Hq, d = q.shape
    if out is None:
        out = torch.empty_like(q)
    _check(_lib.rs_tree_verify_attention(
        plan.handle, _ptr(q), _ptr(k_pages), _ptr(v_pages), k_pages.shape[0], _ptr(block_table),
        block_table.shape[1], _ptr(prefix_len), _ptr(tree_off), _ptr(tree_mask), plan.B, Hq, plan.Hkv, d,
        plan.page_size, float(sm_scale), _ptr(out), _ptr(lse), _ptr(ws), ws.numel() * ws.element_size(),
        _stream(stream)), "rs_tree_verify_attention")
    return out, lse


def ptr_array(tensors):
    """Host array of device pointers (for the *_layers entry points)."""
    return (_P * len(tensors))(*[t.data_ptr() for t in tensors])


class AttentionLayersCall:
    """Pre-marshalled rs_tree_verify_attention_layers call for fixed buffers (one ctypes call
    per step launches all L layers)."""

    def __init__(self, plan: AttnPlan, q_layers, k_layers, v_layers, block_table, prefix_len, tree_off, tree_mask,
                 sm_scale, ws, out_layers, lse_layers=None):
        L = len(q_layers)
        NT, Hq, d = q_layers[0].shape
        self._keep = (q_layers, k_layers, v_layers, out_layers, lse_layers, ws, block_table, prefix_len, tree_off,
                      tree_mask)
        self._arrays = (ptr_array(q_layers), ptr_array(k_layers), ptr_array(v_layers), ptr_array(out_layers),
                        ptr_array(lse_layers) if lse_layers is not None else None)
        qa, ka, va, oa, la = self._arrays
        self.args = [plan.handle, L, qa, ka, va, k_layers[0].shape[0], _ptr(block_table), block_table.shape[1],
                     _ptr(prefix_len), _ptr(tree_off), _ptr(tree_mask), plan.B, Hq, plan.Hkv, d, plan.page_size,
                     float(sm_scale), oa, la, _ptr(ws), ws.numel() * ws.element_size()]
        self.plan = plan

    def __call__(self, stream=None):
        _check(_lib.rs_tree_verify_attention_layers(*self.args, _stream(stream)), "rs_tree_verify_attention_layers")


def tree_verify_attention_layers(plan: AttnPlan, L, q_ptrs, k_ptrs, v_ptrs, num_pages, block_table, prefix_len,
                                 tree_off, tree_mask, Hq, head_dim, sm_scale, out_ptrs, ws, lse_ptrs=None,
                                 stream=None):
    """All L layers through rs_tree_verify_attention_layers with pre-built pointer arrays
    (ptr_array of the per-layer Q / K / V / O tensors), for loops whose batch changes every
    step (the Q/O rows of this step are the first tree_off[B] rows of each layer tensor)."""
    _check(_lib.rs_tree_verify_attention_layers(
        plan.handle, L, q_ptrs, k_ptrs, v_ptrs, int(num_pages), _ptr(block_table), block_table.shape[1],
        _ptr(prefix_len), _ptr(tree_off), _ptr(tree_mask), plan.B, Hq, plan.Hkv, head_dim, plan.page_size,
        float(sm_scale), out_ptrs, lse_ptrs, _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)),
        "rs_tree_verify_attention_layers")


# ------------------------------------------------------------------ a3
def accept_workspace_bytes(mode, B, V) -> int:
    return int(_lib.rs_tree_accept_workspace_bytes(int(mode), int(B), int(V)))


def tree_accept(mode, logits, parent, token, tree_off, gid, draft_probs=None, temperature=1.0, seed=0, step=0,
                out=None, stream=None, ws=None):
    """ws: device workspace of >= accept_workspace_bytes(mode, B, V) bytes (allocated here if None)."""
    NT, V = logits.shape
    B = tree_off.numel() - 1
    need = accept_workspace_bytes(mode, B, V)
    if ws is None and need:
        ws = torch.empty(need, dtype=torch.uint8, device=logits.device)
    dt = DTYPE_BF16 if logits.dtype == torch.bfloat16 else DTYPE_F32
    dev = logits.device
    if out is None:
        out = (torch.empty(B, dtype=torch.int32, device=dev), torch.empty((B, MAX_TREE), dtype=torch.int32, device=dev),
               torch.empty(B, dtype=torch.int32, device=dev), torch.empty(B, dtype=torch.int32, device=dev))
    acc, path, bonus, flags = out
    qdt = DTYPE_BF16 if (draft_probs is not None and draft_probs.dtype == torch.bfloat16) else DTYPE_F32
    _check(_lib.rs_tree_accept_ex(int(mode), _ptr(logits), dt, _ptr(draft_probs), qdt, _ptr(parent), _ptr(token),
                                  _ptr(tree_off), _ptr(gid), B, V, float(temperature), int(seed), int(step), _ptr(acc),
                                  _ptr(path), _ptr(bonus), _ptr(flags), _ptr(ws) if need else None,
                                  ws.numel() if need else 0, _stream(stream)), "rs_tree_accept_ex")
    return acc, path, bonus, flags


def tree_accept_compact(mode, logits, parent, token, tree_off, gid, k_layers, v_layers, block_table, prefix_len,
                        draft_probs=None, temperature=1.0, seed=0, step=0, out=None, new_len=None, moves=None,
                        stream=None, ws=None, layer_ptrs=None, draft_row=None):
    """rs_tree_accept_ex + rs_kv_compact in one launch (the sample's cluster commits its path's
    K/V when its walk ends). layer_ptrs: optional pre-built (k, v) ctypes pointer arrays.
    draft_row (MSS): optional int32 [NT] row of draft_probs per node (-1: no children)."""
    NT, V = logits.shape
    B = tree_off.numel() - 1
    need = accept_workspace_bytes(mode, B, V)
    if ws is None and need:
        ws = torch.empty(need, dtype=torch.uint8, device=logits.device)
    dt = DTYPE_BF16 if logits.dtype == torch.bfloat16 else DTYPE_F32
    dev = logits.device
    if out is None:
        out = (torch.empty(B, dtype=torch.int32, device=dev), torch.empty((B, MAX_TREE), dtype=torch.int32, device=dev),
               torch.empty(B, dtype=torch.int32, device=dev), torch.empty(B, dtype=torch.int32, device=dev))
    if new_len is None:
        new_len = torch.empty(B, dtype=torch.int32, device=dev)
    acc, path, bonus, flags = out
    qdt = DTYPE_BF16 if (draft_probs is not None and draft_probs.dtype == torch.bfloat16) else DTYPE_F32
    L = len(k_layers)
    _, Hkv, ps, d = k_layers[0].shape
    kp, vp = layer_ptrs if layer_ptrs is not None else (_layer_ptrs(k_layers), _layer_ptrs(v_layers))
    _check(_lib.rs_tree_accept_compact(int(mode), _ptr(logits), dt, _ptr(draft_probs), qdt, _ptr(draft_row),
                                       _ptr(parent), _ptr(token),
                                       _ptr(tree_off), _ptr(gid), B, V, float(temperature), int(seed), int(step),
                                       _ptr(acc), _ptr(path), _ptr(bonus), _ptr(flags), _ptr(ws) if need else None,
                                       ws.numel() if need else 0, kp, vp, L, Hkv, d, ps, _ptr(block_table),
                                       block_table.shape[1], _ptr(prefix_len), _ptr(new_len), _ptr(moves),
                                       _stream(stream)), "rs_tree_accept_compact")
    return acc, path, bonus, flags, new_len, moves


def philox4x32_10(ctr: torch.Tensor, key, stream=None):
    out = torch.empty_like(ctr)
    k = np.asarray(key, dtype=np.uint32)
    _check(_lib.rs_philox4x32_10(_ptr(ctr), ctr.shape[0], _ptr(k), _ptr(out), _stream(stream)), "rs_philox4x32_10")
    return out


def exp_spec(x: torch.Tensor, stream=None):
    y = torch.empty_like(x)
    _check(_lib.rs_exp_spec(_ptr(x), x.numel(), _ptr(y), _stream(stream)), "rs_exp_spec")
    return y


# ------------------------------------------------------------------ a4
def _layer_ptrs(layers):
    arr = (_P * len(layers))(*[t.data_ptr() for t in layers])
    return arr


def kv_compact(k_layers, v_layers, block_table, prefix_len, accepted_len, path, page_size=64, moves=None,
               new_len=None, stream=None):
    L = len(k_layers)
    num_pages, Hkv, ps, d = k_layers[0].shape
    B = prefix_len.numel()
    if new_len is None:
        new_len = torch.empty(B, dtype=torch.int32, device=prefix_len.device)
    kp, vp = _layer_ptrs(k_layers), _layer_ptrs(v_layers)
    _check(_lib.rs_kv_compact(kp, vp, L, num_pages, Hkv, d, ps, _ptr(block_table), block_table.shape[1],
                              _ptr(prefix_len), _ptr(accepted_len), _ptr(path), B, _ptr(new_len), _ptr(moves),
                              _stream(stream)), "rs_kv_compact")
    return new_len, moves


# ------------------------------------------------------------------ a0 (host C++)
class CostModelC(ctypes.Structure):
    _fields_ = [("c_draft", _f64), ("b0", _f64), ("b1", _f64), ("b2", _f64), ("b3", _f64), ("k_sat", _f64),
                ("seq_bucket", _i32), ("draft_bucket", _i32)]


class StrategyC(ctypes.Structure):
    _fields_ = [("n", _i32), ("depth", _i32), ("width", _i32), ("n_stop", _i32), ("cache_hit", _i32),
                ("cache_entries", _i32), ("al", _f64), ("t_sd", _f64), ("objective", _f64)]


_sig("rs_selector_create", _i32, ctypes.POINTER(CostModelC), _P, _P, _i32, ctypes.POINTER(_P))
_sig("rs_selector_destroy", None, _P)
_sig("rs_select_strategy", _i32, _P, _P, _P, _P, _P, _i32, _i32, _i32, _i32, ctypes.POINTER(StrategyC), _P)
_sig("rs_cost_model_fit", _i32, _P, _P, _P, _i32, ctypes.POINTER(CostModelC))


def _cost_c(cost) -> CostModelC:
    """cost: any object with c_draft, b0..b3, k_sat, seq_bucket, draft_bucket attributes."""
    return CostModelC(float(cost.c_draft), float(cost.b0), float(cost.b1), float(cost.b2), float(cost.b3),
                      float(cost.k_sat), int(cost.seq_bucket), int(cost.draft_bucket))


class Selector:
    """Drafting-strategy selector with its bucket cache of t_sd predictions."""

    def __init__(self, cost, knots_x, knots_y):
        self._kx = np.ascontiguousarray(knots_x, dtype=np.float64)
        self._ky = np.ascontiguousarray(knots_y, dtype=np.float64)
        self._h = _P()
        _check(_lib.rs_selector_create(ctypes.byref(_cost_c(cost)), _ptr(self._kx), _ptr(self._ky), len(self._kx),
                                       ctypes.byref(self._h)), "rs_selector_create")

    def select(self, trees, prefix_len, n_min=2, n_max=48, patience=2, return_selected=False):
        """trees: per sample (parent int array, o float array) of the candidate tree."""
        B = len(trees)
        off = np.zeros(B + 1, dtype=np.int32)
        for b, (p, _) in enumerate(trees):
            off[b + 1] = off[b] + len(p)
        parent = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int32) for p, _ in trees]) if B else
                                      np.zeros(0, np.int32), dtype=np.int32)
        o = np.ascontiguousarray(np.concatenate([np.asarray(q, np.float64) for _, q in trees]) if B else
                                 np.zeros(0), dtype=np.float64)
        pl = _host_i32(prefix_len)
        sel = np.full((max(B, 1), n_max), -1, dtype=np.int32)
        out = StrategyC()
        _check(_lib.rs_select_strategy(self._h, _ptr(parent), _ptr(o), _ptr(off), _ptr(pl), B, n_min, n_max,
                                       patience, ctypes.byref(out), _ptr(sel)), "rs_select_strategy")
        res = {k: getattr(out, k) for k, _ in StrategyC._fields_}
        if return_selected:
            res["selected"] = sel[:B]
        return res

    def select_flat(self, parent, o, off, prefix_len, n_min=2, n_max=48, patience=2, selected=None):
        """The same call on pre-flattened host arrays (int32 parent [N], float64 o [N], int32 off
        [B+1], int32 prefix_len [B]); `selected` (int32 [B, n_max]) is filled when given."""
        B = len(off) - 1
        out = StrategyC()
        _check(_lib.rs_select_strategy(self._h, _ptr(parent), _ptr(o), _ptr(off), _ptr(prefix_len), B, n_min, n_max,
                                       patience, ctypes.byref(out), _ptr(selected)), "rs_select_strategy")
        return {k: getattr(out, k) for k, _ in StrategyC._fields_}

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.rs_selector_destroy(self._h)
            self._h = None


def cost_model_fit(n_seq, n_draft, t_sec, cost):
    """Least-squares b0..b3 (c_draft and k_sat kept); returns a CostModelC."""
    a = [np.ascontiguousarray(x, dtype=np.float64) for x in (n_seq, n_draft, t_sec)]
    c = _cost_c(cost)
    _check(_lib.rs_cost_model_fit(_ptr(a[0]), _ptr(a[1]), _ptr(a[2]), len(a[0]), ctypes.byref(c)),
           "rs_cost_model_fit")
    return c


# ------------------------------------------------------------------ a6 (host C++)
_sig("rs_knee_threshold", _i32, _P, _P, _i32, _f64, ctypes.POINTER(_i32))
_sig("rs_plan_reallocation", _i32, _P, _i32, _i32, _P, _P, _P, ctypes.POINTER(_i32))
_sig("rs_choose_samples", _i32, _P, _P, _P, _i32, _i32, _P)
_sig("rs_realloc_should_trigger", _i32, _P, _i32, _i32, _i32, _i32, ctypes.POINTER(_i32))


_sig("rs_acceptance_fit", _i32, _P, _P, _i64, _i32, _P, _P, ctypes.POINTER(_i32))


_sig("rs_draft_logits", _i32, _P, _P, _P, _i32, _P)


def draft_logits(parent, o, off):
    """dl of every candidate (flat host arrays as Selector.select_flat)."""
    dl = np.zeros(len(parent))
    _check(_lib.rs_draft_logits(_ptr(np.ascontiguousarray(parent, np.int32)), _ptr(np.ascontiguousarray(o, np.float64)),
                                _ptr(np.ascontiguousarray(off, np.int32)), len(off) - 1, _ptr(dl)), "rs_draft_logits")
    return dl


def acceptance_fit(dl, accepted, n_buckets=20):
    """F's knots from (dl, accepted) observations (rs_acceptance_fit). Returns (knots_x, knots_y)."""
    x = np.ascontiguousarray(dl, dtype=np.float64)
    y = np.ascontiguousarray(accepted, dtype=np.float64)
    kx, ky = np.zeros(n_buckets), np.zeros(n_buckets)
    m = _i32()
    _check(_lib.rs_acceptance_fit(_ptr(x), _ptr(y), len(x), int(n_buckets), _ptr(kx), _ptr(ky), ctypes.byref(m)),
           "rs_acceptance_fit")
    return kx[:m.value].copy(), ky[:m.value].copy()


def knee_threshold(counts, tput, frac=0.1) -> int:
    c = np.ascontiguousarray(counts, dtype=np.float64)
    t = np.ascontiguousarray(tput, dtype=np.float64)
    thr = _i32()
    _check(_lib.rs_knee_threshold(_ptr(c), _ptr(t), len(c), float(frac), ctypes.byref(thr)), "rs_knee_threshold")
    return thr.value


def realloc_should_trigger(loads, threshold, steps_since_last, cooldown):
    ld = _host_i32(loads)
    t = _i32()
    _check(_lib.rs_realloc_should_trigger(_ptr(ld), len(ld), int(threshold), int(steps_since_last), int(cooldown),
                                          ctypes.byref(t)), "rs_realloc_should_trigger")
    return bool(t.value)


def plan_reallocation(loads, threshold):
    ld = _host_i32(loads)
    G = len(ld)
    s, d, c = (np.zeros(max(G, 1), np.int32) for _ in range(3))
    m = _i32()
    _check(_lib.rs_plan_reallocation(_ptr(ld), G, int(threshold), _ptr(s), _ptr(d), _ptr(c), ctypes.byref(m)),
           "rs_plan_reallocation")
    return [(int(s[i]), int(d[i]), int(c[i])) for i in range(m.value)]


def choose_samples(gid, seq_len, avg_accepted, k):
    g = np.ascontiguousarray(gid, dtype=np.int64)
    sl = _host_i32(seq_len)
    aa = np.ascontiguousarray(avg_accepted, dtype=np.float64)
    out = np.zeros(max(k, 1), np.int64)
    _check(_lib.rs_choose_samples(_ptr(g), _ptr(sl), _ptr(aa), len(g), int(k), _ptr(out)), "rs_choose_samples")
    return [int(x) for x in out[:k]]


# ------------------------------------------------------------------ a5
_lib.rs_kv_pack_elems.restype = _i64
_lib.rs_kv_pack_elems.argtypes = [_i32, _i32, _i32, _P, _i32]
_sig("rs_kv_pack", _i32, _P, _P, _i32, _i32, _i32, _i32, _P, _i32, _P, _P, _i32, _P, _i64, _P)
_sig("rs_kv_unpack", _i32, _P, _P, _i32, _i32, _i32, _i32, _P, _i32, _P, _P, _i32, _P, _i64, _P)
_sig("rs_page_pool_create", _i32, _i32, ctypes.POINTER(_P))
_sig("rs_page_pool_destroy", None, _P)
_sig("rs_page_pool_free_count", _i32, _P)
_sig("rs_page_pool_alloc", _i32, _P, _i32, _P)
_sig("rs_page_pool_free", _i32, _P, _P, _i32)
_sig("rs_migrate_reserve", _i32, _P, _P, _i32, _i32, _i32, _P)
_sig("rs_comm_unique_id", _i32, _P)
_sig("rs_comm_create", _i32, _P, _i32, _i32, ctypes.POINTER(_P))
_sig("rs_comm_destroy", _i32, _P)


class KVDescC(ctypes.Structure):
    _fields_ = [("k_ssm", _P), ("v_ssm", _P), ("L_ssm", _i32), ("Hkv_ssm", _i32), ("d_ssm", _i32),
                ("k_llm", _P), ("v_llm", _P), ("L_llm", _i32), ("Hkv_llm", _i32), ("d_llm", _i32),
                ("page_size", _i32)]


_sig("rs_migrate_samples", _i32, _P, _i32, _i32, ctypes.POINTER(KVDescC), _P, _P, _P, _i32, _P, _i32, _P, _P, _sz,
     _P, _P)


def kv_pack_elems(L, Hkv, head_dim, lens) -> int:
    ln = _host_i32(lens)
    return int(_lib.rs_kv_pack_elems(L, Hkv, head_dim, _ptr(ln), len(ln)))


def kv_pack(k_layers, v_layers, block_table, sample_rows, lens, buf, offset_elems=0, stream=None):
    """Gather the samples' K/V of one model (per-layer page pools [pages, Hkv, ps, d]) into buf."""
    _, Hkv, ps, d = k_layers[0].shape
    _check(_lib.rs_kv_pack(_layer_ptrs(k_layers), _layer_ptrs(v_layers), len(k_layers), Hkv, d, ps,
                           _ptr(block_table), block_table.shape[1], _ptr(sample_rows), _ptr(lens), lens.numel(),
                           _ptr(buf), int(offset_elems), _stream(stream)), "rs_kv_pack")
    return buf


def kv_unpack(k_layers, v_layers, block_table, sample_rows, lens, buf, offset_elems=0, stream=None):
    _, Hkv, ps, d = k_layers[0].shape
    _check(_lib.rs_kv_unpack(_layer_ptrs(k_layers), _layer_ptrs(v_layers), len(k_layers), Hkv, d, ps,
                             _ptr(block_table), block_table.shape[1], _ptr(sample_rows), _ptr(lens), lens.numel(),
                             _ptr(buf), int(offset_elems), _stream(stream)), "rs_kv_unpack")


class PagePool:
    """Host page allocator of one instance's KV store (all-or-nothing reservations)."""

    def __init__(self, num_pages: int):
        self._h = _P()
        _check(_lib.rs_page_pool_create(int(num_pages), ctypes.byref(self._h)), "rs_page_pool_create")

    @property
    def handle(self):
        return self._h

    def free_count(self) -> int:
        return int(_lib.rs_page_pool_free_count(self._h))

    def alloc(self, n: int):
        out = np.zeros(max(n, 1), np.int32)
        st = _lib.rs_page_pool_alloc(self._h, int(n), _ptr(out))
        if st == 6:   # RS_ERR_NO_MEMORY
            return None
        _check(st, "rs_page_pool_alloc")
        return out[:n]

    def free(self, pages):
        p = _host_i32(pages)
        _check(_lib.rs_page_pool_free(self._h, _ptr(p), len(p)), "rs_page_pool_free")

    def reserve(self, lens, page_size, max_pages):
        ln = _host_i32(lens)
        rows = np.zeros((max(len(ln), 1), max_pages), np.int32)
        st = _lib.rs_migrate_reserve(self._h, _ptr(ln), len(ln), int(page_size), int(max_pages), _ptr(rows))
        if st == 6:
            return None
        _check(st, "rs_migrate_reserve")
        return rows[:len(ln)]

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.rs_page_pool_destroy(self._h)
            self._h = None


class Comm:
    """NCCL communicator between generation instances; the unique id travels over the
    torch.distributed group `pg` (any backend) from rank 0."""

    def __init__(self, rank: int, world: int, pg=None):
        import torch.distributed as dist
        uid = np.zeros(128, np.uint8)
        if rank == 0:
            _check(_lib.rs_comm_unique_id(_ptr(uid)), "rs_comm_unique_id")
        if world > 1:
            t = torch.from_numpy(uid.astype(np.int64))
            dist.broadcast(t, 0, group=pg)
            uid = np.ascontiguousarray(t.numpy().astype(np.uint8))
        self._h = _P()
        _check(_lib.rs_comm_create(_ptr(uid), int(rank), int(world), ctypes.byref(self._h)), "rs_comm_create")
        self.rank, self.world = rank, world

    def destroy(self):
        if getattr(self, "_h", None):
            _lib.rs_comm_destroy(self._h)
            self._h = None


def migrate_samples(comm: Comm, src_rank, dst_rank, llm_layers, ssm_layers, page_size, pool: PagePool | None,
                    gids, lens, src_block_table, max_pages, staging, scratch, stream=None):
    """Collective over (src, dst). llm_layers/ssm_layers: (k_layers, v_layers) lists or None.
    Returns the destination block-table rows (dst) or None (src); raises RSError on refusal."""
    def _model(m):
        if not m:
            return None, None, 0, 1, 8
        k, v = m
        return _layer_ptrs(k), _layer_ptrs(v), len(k), k[0].shape[1], k[0].shape[3]
    ks, vs, Ls, Hs, ds = _model(ssm_layers)
    kl, vl, Ll, Hl, dl = _model(llm_layers)
    desc = KVDescC(ctypes.cast(ks, _P) if ks else None, ctypes.cast(vs, _P) if vs else None, Ls, Hs, ds,
                   ctypes.cast(kl, _P), ctypes.cast(vl, _P), Ll, Hl, dl, int(page_size))
    n = len(lens)
    g = np.ascontiguousarray(gids, dtype=np.int64)
    ln = _host_i32(lens)
    rows = np.zeros((max(n, 1), max_pages), np.int32)
    _check(_lib.rs_migrate_samples(comm._h, int(src_rank), int(dst_rank), ctypes.byref(desc),
                                   pool.handle if pool is not None else None, _ptr(g), _ptr(ln), n,
                                   _ptr(src_block_table), int(max_pages), _ptr(rows), _ptr(staging),
                                   staging.numel() * staging.element_size(), _ptr(scratch), _stream(stream)),
           "rs_migrate_samples")
    return rows[:n] if comm.rank == dst_rank else None


# ------------------------------------------------------------------ f2
_sig("rs_lm_head_argmax_workspace_bytes", _sz, _i32)
_sig("rs_lm_head_argmax", _i32, _P, _P, _i32, _i32, _i32, _P, _P, _P, _sz, _P)
_sig("rs_tree_accept_greedy_tokens", _i32, _P, _P, _P, _P, _i32, _P, _P, _P, _P, _P)


def lm_head_argmax_workspace_bytes(rows) -> int:
    return int(_lib.rs_lm_head_argmax_workspace_bytes(int(rows)))


_sig("rs_lm_head_logits", _i32, _P, _P, _i32, _i32, _i32, _P, _P)


def lm_head_logits(hidden, weight, out=None, stream=None):
    """bf16 logits [rows, V] of the LM head (f2 for the sampling modes): rs_lm_head_logits."""
    rows, Dm = hidden.shape
    V = weight.shape[0]
    if out is None:
        out = torch.empty((rows, V), dtype=torch.bfloat16, device=hidden.device)
    _check(_lib.rs_lm_head_logits(_ptr(hidden), _ptr(weight), rows, V, Dm, _ptr(out), _stream(stream)),
           "rs_lm_head_logits")
    return out


def lm_head_argmax(hidden, weight, out=None, max_logit=True, ws=None, stream=None):
    """Per-row arg-max of hidden @ weight^T (bf16 in, fp32 accumulate), computed in the GEMM
    epilogue; returns (argmax_token int32 [rows], max_logit fp32 [rows] or None)."""
    rows, Dm = hidden.shape
    V = weight.shape[0]
    dev = hidden.device
    if out is None:
        out = (torch.empty(rows, dtype=torch.int32, device=dev),
               torch.empty(rows, dtype=torch.float32, device=dev) if max_logit else None)
    tok, mx = out
    need = lm_head_argmax_workspace_bytes(rows)
    if ws is None:
        ws = torch.empty(max(need, 8), dtype=torch.uint8, device=dev)
    _check(_lib.rs_lm_head_argmax(_ptr(hidden), _ptr(weight), rows, V, Dm, _ptr(tok), _ptr(mx), _ptr(ws),
                                  ws.numel(), _stream(stream)), "rs_lm_head_argmax")
    return tok, mx


_sig("rs_tree_accept_greedy_tokens_compact", _i32, _P, _P, _P, _P, _i32, _P, _P, _P, _P, _P, _P, _i32, _i32,
     _i32, _i32, _P, _i32, _P, _P, _P, _P)


def tree_accept_greedy_tokens_compact(argmax_token, parent, token, tree_off, k_layers, v_layers, block_table,
                                      prefix_len, out=None, new_len=None, moves=None, stream=None, layer_ptrs=None):
    """The f2 walk on per-node arg-max tokens with the KV commit in one launch."""
    B = tree_off.numel() - 1
    dev = argmax_token.device
    if out is None:
        out = (torch.empty(B, dtype=torch.int32, device=dev), torch.empty((B, MAX_TREE), dtype=torch.int32, device=dev),
               torch.empty(B, dtype=torch.int32, device=dev), torch.empty(B, dtype=torch.int32, device=dev))
    if new_len is None:
        new_len = torch.empty(B, dtype=torch.int32, device=dev)
    acc, path, bonus, flags = out
    L = len(k_layers)
    _, Hkv, ps, d = k_layers[0].shape
    kp, vp = layer_ptrs if layer_ptrs is not None else (_layer_ptrs(k_layers), _layer_ptrs(v_layers))
    _check(_lib.rs_tree_accept_greedy_tokens_compact(_ptr(argmax_token), _ptr(parent), _ptr(token), _ptr(tree_off), B,
                                                     _ptr(acc), _ptr(path), _ptr(bonus), _ptr(flags), kp, vp, L, Hkv,
                                                     d, ps, _ptr(block_table), block_table.shape[1], _ptr(prefix_len),
                                                     _ptr(new_len), _ptr(moves), _stream(stream)),
           "rs_tree_accept_greedy_tokens_compact")
    return acc, path, bonus, flags, new_len, moves


def tree_accept_greedy_tokens(argmax_token, parent, token, tree_off, out=None, stream=None):
    B = tree_off.numel() - 1
    dev = parent.device
    if out is None:
        out = (torch.empty(B, dtype=torch.int32, device=dev), torch.empty((B, MAX_TREE), dtype=torch.int32, device=dev),
               torch.empty(B, dtype=torch.int32, device=dev), torch.empty(B, dtype=torch.int32, device=dev))
    acc, path, bonus, flags = out
    _check(_lib.rs_tree_accept_greedy_tokens(_ptr(argmax_token), _ptr(parent), _ptr(token), _ptr(tree_off), B,
                                             _ptr(acc), _ptr(path), _ptr(bonus), _ptr(flags), _stream(stream)),
           "rs_tree_accept_greedy_tokens")
    return acc, path, bonus, flags


# ------------------------------------------------------------------ f1 (two-stage migration)
_sig("rs_kv_pack_range", _i32, _P, _P, _i32, _i32, _i32, _i32, _P, _i32, _P, _P, _P, _i32, _P, _i64, _P)
_sig("rs_kv_unpack_range", _i32, _P, _P, _i32, _i32, _i32, _i32, _P, _i32, _P, _P, _P, _i32, _P, _i64, _P)
_sig("rs_migrate_stage1", _i32, _P, _i32, _i32, ctypes.POINTER(KVDescC), _P, _P, _P, _P, _i32, _P, _i32, _P, _P, _sz,
     _P, _P)
_sig("rs_migrate_stage2", _i32, _P, _i32, _i32, ctypes.POINTER(KVDescC), _P, _P, _P, _i32, _P, _i32, _P, _P, _P, _sz,
     _P, _P, _P)


def kv_pack_range(k_layers, v_layers, block_table, sample_rows, starts, lens, buf, offset_elems=0, stream=None):
    _, Hkv, ps, d = k_layers[0].shape
    _check(_lib.rs_kv_pack_range(_layer_ptrs(k_layers), _layer_ptrs(v_layers), len(k_layers), Hkv, d, ps,
                                 _ptr(block_table), block_table.shape[1], _ptr(sample_rows), _ptr(starts), _ptr(lens),
                                 lens.numel(), _ptr(buf), int(offset_elems), _stream(stream)), "rs_kv_pack_range")
    return buf


def kv_unpack_range(k_layers, v_layers, block_table, sample_rows, starts, lens, buf, offset_elems=0, stream=None):
    _, Hkv, ps, d = k_layers[0].shape
    _check(_lib.rs_kv_unpack_range(_layer_ptrs(k_layers), _layer_ptrs(v_layers), len(k_layers), Hkv, d, ps,
                                   _ptr(block_table), block_table.shape[1], _ptr(sample_rows), _ptr(starts),
                                   _ptr(lens), lens.numel(), _ptr(buf), int(offset_elems), _stream(stream)),
           "rs_kv_unpack_range")


def _kv_desc(llm_layers, ssm_layers, page_size):
    keep = []

    def _model(m):
        if not m:
            return None, None, 0, 1, 8
        k, v = m
        kp, vp = _layer_ptrs(k), _layer_ptrs(v)
        keep.extend([kp, vp])
        return kp, vp, len(k), k[0].shape[1], k[0].shape[3]
    ks, vs, Ls, Hs, ds = _model(ssm_layers)
    kl, vl, Ll, Hl, dl = _model(llm_layers)
    desc = KVDescC(ctypes.cast(ks, _P) if ks else None, ctypes.cast(vs, _P) if vs else None, Ls, Hs, ds,
                   ctypes.cast(kl, _P), ctypes.cast(vl, _P), Ll, Hl, dl, int(page_size))
    return desc, keep


class TwoStageMigration:
    """f1: stage1() enqueues the verified prefix [0, lens) on `stream` and returns
    while the instances keep computing; stage2(new_lens) moves [lens, new_lens) with the SSM part
    first (`ssm_ready` event recorded on the destination) and the LLM part behind it. Both ranks
    of the pair drive the same object calls; the staging / scratch buffers stay referenced here
    until the stream is done."""

    def __init__(self, comm: Comm, src_rank, dst_rank, llm_layers, ssm_layers, page_size, pool: PagePool | None,
                 max_pages, staging, scratch, stream):
        self.comm, self.src, self.dst = comm, int(src_rank), int(dst_rank)
        self.desc, self._keep = _kv_desc(llm_layers, ssm_layers, page_size)
        self.pool, self.max_pages, self.staging, self.scratch, self.stream = pool, int(max_pages), staging, scratch, stream
        self.ps = int(page_size)
        self.rows = None
        self.capacity = None
        self.ssm_ready = torch.cuda.Event(enable_timing=True)
        self.done = torch.cuda.Event(enable_timing=True)
        self.ssm_ready.record(stream)      # torch creates the CUDA event lazily, on first record
        self.done.record(stream)

    def stage1(self, gids, lens, reserve_lens, src_block_table):
        n = len(lens)
        self.n = n
        self.lens1 = _host_i32(lens)
        g = np.ascontiguousarray(gids, dtype=np.int64)
        rsv = _host_i32(reserve_lens)
        self.rows = np.zeros((max(n, 1), self.max_pages), np.int32)
        _check(_lib.rs_migrate_stage1(self.comm._h, self.src, self.dst, ctypes.byref(self.desc),
                                      self.pool.handle if self.pool is not None else None, _ptr(g), _ptr(self.lens1),
                                      _ptr(rsv), n, _ptr(src_block_table), self.max_pages, _ptr(self.rows),
                                      _ptr(self.staging), self.staging.numel() * self.staging.element_size(),
                                      _ptr(self.scratch), _stream(self.stream)), "rs_migrate_stage1")
        self.capacity = np.ascontiguousarray(rsv.copy())
        self._keep_bt1 = self._hold(src_block_table)
        self.done.record(self.stream)

    def stage2(self, new_lens, src_block_table):
        starts = self.lens1
        delta = _host_i32(np.asarray(new_lens) - starts)
        _check(_lib.rs_migrate_stage2(self.comm._h, self.src, self.dst, ctypes.byref(self.desc),
                                      self.pool.handle if self.pool is not None else None, _ptr(starts), _ptr(delta),
                                      self.n, _ptr(src_block_table), self.max_pages, _ptr(self.rows),
                                      _ptr(self.capacity), _ptr(self.staging),
                                      self.staging.numel() * self.staging.element_size(), _ptr(self.scratch),
                                      ctypes.c_void_p(self.ssm_ready.cuda_event) if self.comm.rank == self.dst else None,
                                      _stream(self.stream)), "rs_migrate_stage2")
        self._keep_bt2 = self._hold(src_block_table)
        self.done.record(self.stream)

    def _hold(self, t):
        """Keep a caller's device tensor alive (and out of the caching allocator's reuse on other
        streams) until this migration's stream has passed the kernels that read it."""
        if isinstance(t, torch.Tensor) and t.is_cuda and self.stream is not None:
            t.record_stream(self.stream)
        return t

    def dst_rows(self):
        return self.rows[:self.n] if self.comm.rank == self.dst else None


# ------------------------------------------------------------------ a5 over peer memory
_sig("rs_peer_create", _i32, ctypes.POINTER(KVDescC), _i32, ctypes.POINTER(_P))
_sig("rs_peer_blob_bytes", _sz, _P)
_sig("rs_peer_export", _i32, _P, _P, _sz)
_sig("rs_peer_import", _i32, _P, _P, _sz)
_sig("rs_peer_push", _i32, _P, _i32, _P, _P, _i32, _P, _P, _i32, _i32, _P)
_sig("rs_peer_signal", _i32, _P, _i32, _P)
_sig("rs_peer_wait", _i32, _P, _i32, _i32, _P)
_sig("rs_peer_destroy", None, _P)

PEER_SSM, PEER_LLM = 1, 2
PEER_DONE, PEER_SSM_READY = 0, 1


class PeerStore:
    """This rank's KV store registered for peer-memory migration (rs_peer_*). export() gives the
    host blob other ranks import(); push() copies sample token ranges into a peer's reserved
    pages (one kernel per model); signal()/wait() carry completion as an inter-process event."""

    def __init__(self, llm_layers, ssm_layers, page_size, rank: int):
        self.desc, self._keep = _kv_desc(llm_layers, ssm_layers, page_size)
        self._h = _P()
        _check(_lib.rs_peer_create(ctypes.byref(self.desc), int(rank), ctypes.byref(self._h)), "rs_peer_create")
        self.rank = int(rank)
        self._hold = []

    def export(self) -> bytes:
        n = int(_lib.rs_peer_blob_bytes(self._h))
        buf = np.zeros(n, np.uint8)
        _check(_lib.rs_peer_export(self._h, _ptr(buf), n), "rs_peer_export")
        return buf.tobytes()

    def import_(self, blob: bytes):
        buf = np.frombuffer(blob, np.uint8).copy()
        _check(_lib.rs_peer_import(self._h, _ptr(buf), buf.size), "rs_peer_import")

    def push(self, dst_rank, src_block_table, dst_block_table, lens, starts=None, parts=PEER_SSM | PEER_LLM,
             stream=None):
        """src/dst_block_table: device int32 [n, max_pages]; lens/starts: device int32 [n]. The
        tensors are kept referenced on `stream` until it passes the kernels."""
        n = int(lens.numel())
        _check(_lib.rs_peer_push(self._h, int(dst_rank), _ptr(src_block_table), _ptr(dst_block_table),
                                 int(src_block_table.shape[1]), _ptr(starts) if starts is not None else None,
                                 _ptr(lens), n, int(parts), _stream(stream)), "rs_peer_push")
        if stream is not None:
            for t in (src_block_table, dst_block_table, lens, starts):
                if isinstance(t, torch.Tensor):
                    t.record_stream(stream)

    def signal(self, which=PEER_DONE, stream=None):
        _check(_lib.rs_peer_signal(self._h, int(which), _stream(stream)), "rs_peer_signal")

    def wait(self, src_rank, which=PEER_DONE, stream=None):
        _check(_lib.rs_peer_wait(self._h, int(src_rank), int(which), _stream(stream)), "rs_peer_wait")

    def destroy(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.rs_peer_destroy(self._h)
            self._h = None

    def __del__(self):
        self.destroy()


def peer_connect(store: PeerStore, pg=None):
    """Collective over the torch.distributed group: every rank exports its blob, all-gathers
    the others' and imports them (its own too: pid-local, raw pointers)."""
    import torch.distributed as dist
    blob = store.export()
    world = dist.get_world_size(pg)
    blobs = [None] * world
    dist.all_gather_object(blobs, blob, group=pg)
    for b in blobs:
        store.import_(b)
    return store


# ------------------------------------------------------------------ rs_ctx / rs_calibrate
class CtxDescC(ctypes.Structure):
    _fields_ = [("rank", _i32), ("world", _i32), ("page_size", _i32)]


class CalibDescC(ctypes.Structure):
    _fields_ = [("Hq", _i32), ("n_points", _i32), ("B", _P), ("P", _P), ("T", _P), ("reps", _i32), ("q", _P),
                ("out", _P), ("qo_elems", _sz), ("ws", _P), ("ws_bytes", _sz), ("dense_s_per_token", _f64),
                ("stream", _P)]


_sig("rs_ctx_create", _i32, ctypes.POINTER(CtxDescC), ctypes.POINTER(_P))
_sig("rs_ctx_destroy", _i32, _P)
_sig("rs_ctx_register_kv", _i32, _P, _i32, _i32, _P, _P, _i32, _i32, _i32)
_sig("rs_ctx_set_strategy", _i32, _P, ctypes.POINTER(CostModelC), _P, _P, _i32)
_sig("rs_ctx_get_strategy", _i32, _P, ctypes.POINTER(CostModelC), _P, _P, ctypes.POINTER(_i32))
_sig("rs_ctx_selector", _P, _P)
_sig("rs_ctx_fit_acceptance", _i32, _P, _P, _P, _i64, _i32)
_sig("rs_calibrate_workspace_bytes", _sz, _P, ctypes.POINTER(CalibDescC))
_sig("rs_calibrate", _i32, _P, ctypes.POINTER(CalibDescC), _P)


class Ctx:
    """One instance's rs_ctx: KV registrations + the strategy state (F, t_sd) and its selector."""

    def __init__(self, rank=0, world=1, page_size=64):
        self._h = _P()
        _check(_lib.rs_ctx_create(ctypes.byref(CtxDescC(rank, world, page_size)), ctypes.byref(self._h)),
               "rs_ctx_create")
        self._keep = []

    def register_kv(self, model, k_layers, v_layers):
        if not k_layers:   # unregister
            _check(_lib.rs_ctx_register_kv(self._h, int(model), 0, None, None, 0, 1, 1), "rs_ctx_register_kv")
            return
        kp, vp = _layer_ptrs(k_layers), _layer_ptrs(v_layers)
        self._keep += [kp, vp, list(k_layers), list(v_layers)]
        num_pages, Hkv, _, d = k_layers[0].shape
        _check(_lib.rs_ctx_register_kv(self._h, int(model), len(k_layers), kp, vp, int(num_pages), int(Hkv), int(d)),
               "rs_ctx_register_kv")

    def set_strategy(self, cost=None, knots_x=None, knots_y=None):
        c = _cost_c(cost) if cost is not None else None
        kx = None if knots_x is None else np.ascontiguousarray(knots_x, dtype=np.float64)
        ky = None if knots_y is None else np.ascontiguousarray(knots_y, dtype=np.float64)
        _check(_lib.rs_ctx_set_strategy(self._h, ctypes.byref(c) if c is not None else None, _ptr(kx), _ptr(ky),
                                        0 if kx is None else len(kx)), "rs_ctx_set_strategy")

    def strategy(self):
        """(cost model dict, knots_x, knots_y) currently in the ctx."""
        c = CostModelC()
        m = _i32(64)
        kx, ky = np.zeros(64), np.zeros(64)
        _check(_lib.rs_ctx_get_strategy(self._h, ctypes.byref(c), _ptr(kx), _ptr(ky), ctypes.byref(m)),
               "rs_ctx_get_strategy")
        return {k: getattr(c, k) for k, _ in CostModelC._fields_}, kx[:m.value].copy(), ky[:m.value].copy()

    def fit_acceptance(self, dl, accepted, n_buckets=20):
        x = np.ascontiguousarray(dl, dtype=np.float64)
        y = np.ascontiguousarray(accepted, dtype=np.float64)
        _check(_lib.rs_ctx_fit_acceptance(self._h, _ptr(x), _ptr(y), len(x), int(n_buckets)),
               "rs_ctx_fit_acceptance")

    def calibrate(self, Hq, grid, reps=3, dense_s_per_token=0.0, stream=None):
        """grid: list of (B, P, T). Returns the measured attention seconds per point; the ctx's cost
        model is refitted (see rs_calibrate)."""
        g = np.ascontiguousarray(np.asarray(grid, dtype=np.int32).T)
        Bs, Ps, Ts = (np.ascontiguousarray(g[i]) for i in range(3))
        d = self._keep[-2][0].shape[3]
        elems = int(max(b * t for b, _, t in grid) * Hq * d)
        dev = self._keep[-2][0].device
        q = torch.randn(elems, device=dev).to(torch.bfloat16)
        out = torch.empty(elems, dtype=torch.bfloat16, device=dev)
        desc = CalibDescC(int(Hq), len(grid), _ptr(Bs), _ptr(Ps), _ptr(Ts), int(reps), _ptr(q), _ptr(out), elems,
                          None, 0, float(dense_s_per_token), _stream(stream))
        need = int(_lib.rs_calibrate_workspace_bytes(self._h, ctypes.byref(desc)))
        if need == 0:
            raise RSError(8, "rs_calibrate_workspace_bytes: " + _lib.rs_last_error().decode())
        ws = torch.empty(need, dtype=torch.uint8, device=dev)
        desc.ws, desc.ws_bytes = _ptr(ws), need
        t = np.zeros(len(grid))
        _check(_lib.rs_calibrate(self._h, ctypes.byref(desc), _ptr(t)), "rs_calibrate")
        return t

    def select(self, parent, o, off, prefix_len, n_min=2, n_max=48, patience=2, selected=None):
        """rs_select_strategy with the ctx's selector (flat host arrays, see Selector.select_flat)."""
        h = _lib.rs_ctx_selector(self._h)
        if not h:
            raise RSError(1, "rs_ctx: no acceptance fit set")
        B = len(off) - 1
        out = StrategyC()
        _check(_lib.rs_select_strategy(h, _ptr(parent), _ptr(o), _ptr(off), _ptr(prefix_len), B, n_min, n_max,
                                       patience, ctypes.byref(out), _ptr(selected)), "rs_select_strategy")
        return {k: getattr(out, k) for k, _ in StrategyC._fields_}

    def destroy(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.rs_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        self.destroy()
