"""Profiling driver: the sweep workload, one warm-up batch then one batch of 8 rotations
(for ncu: `ncu --set full -k regex:... python tools/prof_sweep.py`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from synth import make_config  # noqa: E402
from paper_1711_05075_b200 import ballcorr  # noqa: E402
from paper_1711_05075_b200.presets import correlator_kwargs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "sweep"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 8
w = make_config(name, n_rot=2 * nb)
c = ballcorr.Correlator(**correlator_kwargs(name, w.N, w.h, w.t0, w.weights))
c.shape_upload(0, w.A_xyzr, w.A_w)
c.shape_upload(1, w.B_xyzr, w.B_w)
c.spectrum_A()
kind = "max_real" if w.weights == "complex" else "min_argmin"
out = torch.empty(nb * 16, dtype=torch.uint8, device="cuda")
for r0 in (0, nb):
    c.correlate_rotations(w.R[r0:r0 + nb], kind, out=out)
torch.cuda.synchronize()
print("ok", c.query("L_B"), c.query("fused_spread_z"))
