"""Oracle: tree acceptance — ctypes wrapper over oracle/accept_ref.c (test infrastructure only).

The arithmetic lives in accept_ref.c (plain sequential C, see its header for the rule and the
paper passages). This module only compiles it (gcc, -ffp-contract=off, no fast-math)
and marshals numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "accept_ref.c")
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle_accept.so")
_lib = None

GREEDY, DELTA, MSS = 0, 1, 2
FLAG_MALFORMED, FLAG_NONFINITE = 1, 2
MAX_TREE = 64


def build(force: bool = False) -> str:
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        _lib.oracle_philox4x32_10.argtypes = [P, P, P]
        _lib.oracle_exp_spec.argtypes = [ctypes.c_float]
        _lib.oracle_exp_spec.restype = ctypes.c_float
        _lib.oracle_exp_spec_array.argtypes = [P, P, ctypes.c_int64]
        _lib.oracle_row_weights.argtypes = [P, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                            ctypes.c_float, P, P]
        _lib.oracle_tree_accept.argtypes = [ctypes.c_int, P, ctypes.c_int, P, P, P, P, P,
                                            ctypes.c_int, ctypes.c_int, ctypes.c_float,
                                            ctypes.c_uint64, ctypes.c_uint64, P, P, P, P]
        _lib.oracle_tree_accept_rows.argtypes = [ctypes.c_int, P, ctypes.c_int, P, P, P, P, P, P,
                                                 ctypes.c_int, ctypes.c_int, ctypes.c_float,
                                                 ctypes.c_uint64, ctypes.c_uint64, P, P, P, P]
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def philox4x32_10(ctr, key):
    ctr = np.ascontiguousarray(ctr, dtype=np.uint32)
    key = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    _load().oracle_philox4x32_10(_ptr(ctr), _ptr(key), _ptr(out))
    return out


def exp_spec(x: float) -> np.float32:
    return np.float32(_load().oracle_exp_spec(ctypes.c_float(float(x))))


def exp_spec_array(x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.empty_like(x)
    _load().oracle_exp_spec_array(_ptr(x), _ptr(y), x.size)
    return y


def row_weights(logits_row, inv_tau=1.0):
    """Integer weights of one target row (bf16 given as uint16 view, or float32)."""
    arr = np.ascontiguousarray(logits_row)
    is_bf16 = 1 if arr.dtype == np.uint16 else 0
    if not is_bf16:
        arr = arr.astype(np.float32)
    V = arr.shape[-1]
    w = np.zeros(V, dtype=np.uint64)
    Z = np.zeros(1, dtype=np.uint64)
    rc = _load().oracle_row_weights(_ptr(arr), is_bf16, 0, V, ctypes.c_float(inv_tau), _ptr(w), _ptr(Z))
    if rc != 0:
        return None, None
    return w, int(Z[0])


def tree_accept(mode, logits, parent, token, tree_off, gid, V, draft_probs=None,
                temperature=1.0, seed=0, step=0, draft_row=None):
    """logits: [NT, V] as np.uint16 (bf16 bits) or np.float32. Returns
    (accepted_len[B], path[B,64], bonus[B], flags[B]). MSS: draft_probs [R, V]; draft_row
    (optional, int32 [NT]) = the row of node i's draft distribution (None: row i); only nodes
    with children are read (reading Z29)."""
    lg = np.ascontiguousarray(logits)
    is_bf16 = 1 if lg.dtype == np.uint16 else 0
    if not is_bf16:
        lg = lg.astype(np.float32)
    B = len(tree_off) - 1
    par = np.ascontiguousarray(parent, dtype=np.int32)
    tok = np.ascontiguousarray(token, dtype=np.int32)
    off = np.ascontiguousarray(tree_off, dtype=np.int32)
    g = np.ascontiguousarray(gid, dtype=np.int64)
    dp = None
    if mode == MSS:
        dp = np.ascontiguousarray(draft_probs, dtype=np.float32)
    acc = np.zeros(B, dtype=np.int32)
    path = np.zeros((B, MAX_TREE), dtype=np.int32)
    bonus = np.zeros(B, dtype=np.int32)
    flags = np.zeros(B, dtype=np.int32)
    dr = None if draft_row is None else np.ascontiguousarray(draft_row, dtype=np.int32)
    _load().oracle_tree_accept_rows(int(mode), _ptr(lg), is_bf16, _ptr(dp) if dp is not None else None,
                                    _ptr(dr) if dr is not None else None,
                                    _ptr(par), _ptr(tok), _ptr(off), _ptr(g), B, int(V),
                                    ctypes.c_float(temperature), ctypes.c_uint64(seed),
                                    ctypes.c_uint64(step), _ptr(acc), _ptr(path), _ptr(bonus), _ptr(flags))
    return acc, path, bonus, flags
