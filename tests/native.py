"""Test-only native helpers (tests/csrc/*.cu), built in-tree by nvcc for sm_100a. Not part of the
product library; only GPU tests load them."""
import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD = os.path.join(HERE, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build(force=False):
    os.makedirs(BUILD, exist_ok=True)
    out = {}
    for name in ("pdl_writer",):
        src = os.path.join(HERE, "csrc", name + ".cu")
        lib = os.path.join(BUILD, f"lib{name}.so")
        if force or not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src):
            tmp = lib + f".{os.getpid()}.tmp"
            subprocess.check_call([NVCC, "-O2", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                                   "-Xcompiler", "-fPIC", "-shared", "-o", tmp, src])
            os.replace(tmp, lib)
        out[name] = lib
    return out


def pdl_writer():
    lib = ctypes.CDLL(build()["pdl_writer"])
    P = ctypes.c_void_p
    lib.pdl_test_write_rows.argtypes = [P, P, P, ctypes.c_int, ctypes.c_int, P, P, ctypes.c_ulonglong, P]
    lib.pdl_test_write_rows.restype = ctypes.c_int
    return lib
