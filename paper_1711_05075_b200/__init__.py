"""paper_1711_05075_b200 -- B200-native analytic ball-set correlator.

Implements the data-parallel hot path of Behandish & Ilies, "Analytic Methods
for Geometric Modeling via Spherical Decomposition" (arXiv 1711.05075): the
correlation f_R(t) = int rho_A(x) rho_{RB}(x - t) dx of two weighted ball
sets over an N^3 translation grid for a batch of rotations, through the
Fourier domain or by exact pair-lens spreading
(L343-L360), in hand-written sm_100a kernels behind the C ABI of
include/ballcorr.h.

`ballcorr` is the ctypes binding (argument marshalling only); `presets`
holds the per-workload parameters (band, period, mode) chosen by the parity
measurements recorded in DESIGN.md.
"""
from . import ballcorr  # noqa: F401  (raises ImportError if libballcorr.so is missing)
from .ballcorr import Correlator, BallCorrError  # noqa: F401
