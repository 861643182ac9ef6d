"""rlhfspec_core on B200: the RLHFSpec (arXiv 2512.04752) verification hot path.

The compute lives in librlhfspec_core.so (CUDA sm_100a + C++), declared in
include/rlhfspec_core.h; `paper_2512_04752_b200.core` is its thin ctypes binding."""
__all__ = ["core", "build"]
