"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds input GENERATION only (ball sets, weights, rotation
matrices, grid descriptions).  It contains none of the correlation
arithmetic, so both `oracle/` and the CUDA path may consume its arrays
without sharing any of the method's code.
"""
from .configs import (  # noqa: F401
    Workload,
    CONFIG_NAMES,
    make_config,
    random_rotations,
    random_small_case,
)
