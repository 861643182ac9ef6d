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
LIB_PATH = os.path.join(_HERE, "librlhfspec_core.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2512_04752_b200.build` "
                      "(the CUDA path has no fallback)")
_lib = ctypes.CDLL(LIB_PATH)

GREEDY, SAMPLE_DELTA, SAMPLE_MSS = 0, 1, 2
DTYPE_BF16, DTYPE_F32 = 0, 1
FLAG_MALFORMED, FLAG_NONFINITE = 1, 2
MAX_TREE = 64

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
_sig("rs_attn_set_trace", _i32, _P, _sz)
_sig("rs_tree_verify_attention", _i32, _P, _P, _P, _P, _i64, _P, _i32, _P, _P, _P, _i32, _i32, _i32,
     _i32, _i32, _f32, _P, _P, _P, _sz, _P)
_sig("rs_tree_verify_attention_layers", _i32, _P, _i32, _P, _P, _P, _i64, _P, _i32, _P, _P, _P, _i32, _i32,
     _i32, _i32, _i32, _f32, _P, _P, _P, _sz, _P)
_sig("rs_tree_accept", _i32, _i32, _P, _i32, _P, _P, _P, _P, _P, _i32, _i32, _f32, _u64, _u64, _P, _P,
     _P, _P, _P, _sz, _P)
_sig("rs_philox4x32_10", _i32, _P, _i64, _P, _P, _P)
_sig("rs_exp_spec", _i32, _P, _i64, _P, _P)
_sig("rs_kv_compact", _i32, _P, _P, _i32, _i64, _i32, _i32, _i32, _P, _i32, _P, _P, _P, _i32, _P, _P, _P)


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


# ------------------------------------------------------------------ a2
class AttnPlan:
    """Host schedule for one verify step (lengths of this step), shared by every layer."""

    def __init__(self, prefix_len_host, tree_off_host, Hq, Hkv, head_dim, page_size=64, num_ctas=0):
        self._pl = _host_i32(prefix_len_host)
        self._to = _host_i32(tree_off_host)
        self.B, self.Hq, self.Hkv, self.head_dim, self.page_size = len(self._pl), Hq, Hkv, head_dim, page_size
        h = _P()
        _check(_lib.rs_attn_plan_create(_ptr(self._pl), _ptr(self._to), self.B, Hq, Hkv, head_dim, page_size,
                                        num_ctas, ctypes.byref(h)), "rs_attn_plan_create")
        self.handle = h
        self.ws_bytes = int(_lib.rs_attn_plan_workspace_bytes(h))

    def info(self):
        a, b, c = _i32(), _i32(), _i32()
        _check(_lib.rs_attn_plan_info(self.handle, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)),
               "rs_attn_plan_info")
        return dict(num_ctas=a.value, num_items=b.value, num_split_units=c.value)

    def schedule(self):
        """(cta_off [num_ctas+1], items [num_items, 7]) as numpy arrays."""
        inf = self.info()
        cta = np.zeros(inf["num_ctas"] + 1, dtype=np.int32)
        items = np.zeros((inf["num_items"], 10), dtype=np.int32)
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


# ------------------------------------------------------------------ a3
def tree_accept(mode, logits, parent, token, tree_off, gid, draft_probs=None, temperature=1.0, seed=0, step=0,
                out=None, stream=None):
    NT, V = logits.shape
    B = tree_off.numel() - 1
    dt = DTYPE_BF16 if logits.dtype == torch.bfloat16 else DTYPE_F32
    dev = logits.device
    if out is None:
        out = (torch.empty(B, dtype=torch.int32, device=dev), torch.empty((B, MAX_TREE), dtype=torch.int32, device=dev),
               torch.empty(B, dtype=torch.int32, device=dev), torch.empty(B, dtype=torch.int32, device=dev))
    acc, path, bonus, flags = out
    _check(_lib.rs_tree_accept(int(mode), _ptr(logits), dt, _ptr(draft_probs), _ptr(parent), _ptr(token),
                               _ptr(tree_off), _ptr(gid), B, V, float(temperature), int(seed), int(step), _ptr(acc),
                               _ptr(path), _ptr(bonus), _ptr(flags), None, 0, _stream(stream)), "rs_tree_accept")
    return acc, path, bonus, flags


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
