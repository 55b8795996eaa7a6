"""Dev timing of one config through the spectral path (stage times via library events)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from synth import make_config
from paper_1711_05075_b200 import ballcorr

name = sys.argv[1] if len(sys.argv) > 1 else "sweep"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 255
Np = int(sys.argv[3]) if len(sys.argv) > 3 else 256
nrot = int(sys.argv[4]) if len(sys.argv) > 4 else 16
w = make_config(name, n_rot=nrot)
c = ballcorr.Correlator(N=w.N, h=w.h, t0=w.t0, Np=Np, K=K, weights=w.weights)
t = time.time(); c.shape_upload(0, w.A_xyzr, w.A_w); c.shape_upload(1, w.B_xyzr, w.B_w); print("upload s", time.time() - t)
for k in ["P", "L_A", "c_A", "G_A", "tau_A", "L_B", "c_B", "G_B", "tau_B", "cut_B", "band_modes"]:
    print(k, c.query(k))
c.set_profiling(True)
torch.cuda.synchronize(); t = time.time(); c.spectrum_A(); torch.cuda.synchronize(); print("spectrum_A s", time.time() - t)
kind = "max_real" if w.weights == "complex" else "min_argmin"
out = torch.empty(nrot * 16, dtype=torch.uint8, device="cuda")
c.correlate_rotations(w.R, kind, out=out)
torch.cuda.synchronize()
c.reset_stage_times()
t = time.time()
c.correlate_rotations(w.R, kind, out=out)
torch.cuda.synchronize()
dt = time.time() - t
print(f"{nrot} rotations: {dt*1e3:.1f} ms wall, {dt/nrot*1e3:.3f} ms/rot, {w.N**3*nrot/dt:.3e} transl*rot/s")
for k, (ms, n) in c.stage_times().items():
    print(f"  {k:16s} {ms/nrot:8.3f} ms/rot  ({n} launches)")
print(np.frombuffer(out.cpu().numpy().tobytes(), dtype=ballcorr.EXTREMUM_DTYPE)[:4])
