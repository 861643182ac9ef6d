"""Seeded synthetic input generators shared by the CUDA path's tests/bench and the CPU oracle.

This package holds NO arithmetic of the method (no attention, no acceptance rule, no
draft-logit products, no compaction): it only draws random inputs with the shapes and
structure of the paper's workloads.
"""
from .workloads import *  # noqa: F401,F403
