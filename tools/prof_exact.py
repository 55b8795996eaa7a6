"""Profiling driver: exact mode on a workload (default single), two correlate calls of one
rotation (for ncu -k regex:exact)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import make_config  # noqa: E402
from paper_1711_05075_b200 import ballcorr  # noqa: E402
from paper_1711_05075_b200.presets import correlator_kwargs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "single"
w = make_config(name)
c = ballcorr.Correlator(**correlator_kwargs(name, w.N, w.h, w.t0, w.weights))
c.shape_upload(0, w.A_xyzr, w.A_w)
c.shape_upload(1, w.B_xyzr, w.B_w)
for _ in range(2):
    c.correlate_rotations(w.R[:1], "minmax")
print("ok")
