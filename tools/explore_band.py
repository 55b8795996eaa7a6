"""Band-error exploration: spectral f at several (Np, K) vs the GPU exact pair-lens f
(exact mode is pinned to the fp64 oracle by tests/test_gpu_exact.py)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from synth import make_config
from paper_1711_05075_b200 import ballcorr

name = sys.argv[1]
nrot = int(sys.argv[2])
combos = [tuple(float(v) for v in s.split(":")) for s in sys.argv[3:]]
w = make_config(name)
R = w.R[:nrot]
t = time.time()
ex = ballcorr.Correlator(N=w.N, h=w.h, t0=w.t0, mode="exact", precision="f32", weights=w.weights, max_batch=1)
ex.shape_upload(0, w.A_xyzr, w.A_w); ex.shape_upload(1, w.B_xyzr, w.B_w); ex.spectrum_A()
fe = ex.correlate_rotations(R, "full").astype(np.float64)
if w.weights == "complex":
    fe = fe[..., 0] + 1j * fe[..., 1]
print(f"{name}: exact {time.time()-t:.1f}s  max|f| {np.abs(fe).max():.6g}", flush=True)
ex.close()
for cmb in combos:
    Np, K = int(cmb[0]), int(cmb[1])
    rad = cmb[2] if len(cmb) > 2 else 0.0
    c = ballcorr.Correlator(N=w.N, h=w.h, t0=w.t0, Np=Np, K=K, weights=w.weights, max_batch=2, band_radius=rad)
    try:
        c.shape_upload(0, w.A_xyzr, w.A_w); c.shape_upload(1, w.B_xyzr, w.B_w); c.spectrum_A()
    except ballcorr.BallCorrError as e:
        print(Np, K, "ERR", e); continue
    fs = c.correlate_rotations(R, "full").astype(np.float64)
    if w.weights == "complex":
        fs = fs[..., 0] + 1j * fs[..., 1]
    errs = [np.abs(fs[r] - fe[r]).max() / np.abs(fe[r]).max() for r in range(nrot)]
    re_err = [np.abs(fs[r].real - fe[r].real).max() / np.abs(fe[r].real).max() for r in range(nrot)]
    best = [(fs[r].real.max(), fe[r].real.max(), int(np.argmax(fs[r].real)), int(np.argmax(fe[r].real))) for r in range(nrot)]
    print(f"Np={Np} K={K} R={rad} sigma_f={2*K/Np:.2f}: rel err {['%.2e' % e for e in errs]} re {['%.2e' % e for e in re_err]}  max {best[:2]}", flush=True)
    c.close()
