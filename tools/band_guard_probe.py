"""Band-error guard vs the oracle: for a B and several bands K, the library's probe estimate
(bc_query("band_error")) beside the sampled error against the fp64 lens oracle."""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from synth import make_config
from paper_1711_05075_b200 import ballcorr
from paper_1711_05075_b200.presets import correlator_kwargs

E = np.array([[0.0, 0.0, 0.0, 0.02], [0.2, 0.0, 0.0, 0.02], [0.0, -0.2, 0.0, 0.005],
              [0.0, 0.0, 0.2, 0.01], [-0.1155, 0.1155, -0.1155, 0.02]])
w = make_config("sweep", n_rot=2)
cases = {"edge5": E, "edge4": E[[0, 1, 3, 4]], "sweepB": w.B_xyzr}
Ks = [int(k) for k in sys.argv[1].split(",")] if len(sys.argv) > 1 else [255, 319, 399, 499]
for name, B in cases.items():
    for K in Ks:
        try:
            c = ballcorr.Correlator(**correlator_kwargs("sweep", w.N, w.h, w.t0, "real", K=K, tolerance=1.0))
            c.shape_upload(0, w.A_xyzr, w.A_w)
            c.shape_upload(1, B)
            c.spectrum_A()
            t = time.time()
            c.correlate_rotations(w.R[:1], "min_argmin")
            tp = time.time() - t
            est = c.query("band_error")
            f = c.correlate_rotations(w.R[1:2], "full")[0].reshape(-1)
            rng = np.random.default_rng(5)
            idx = np.unique(np.concatenate([rng.choice(f.size, 300, replace=False), np.argpartition(np.abs(f), -150)[-150:]]))
            ref = oracle.correlate_points(w.A_xyzr, w.A_w, B, None, w.R[1], w.N, w.h, w.t0, idx)
            err = np.abs(f[idx] - ref).max() / np.abs(ref).max()
            print(f"{name} K={K} fold_fast={c.query('fold_fast')} probe_est={est:.3e} oracle_sampled={err:.3e} probe_s={tp:.2f}", flush=True)
            c.close()
        except Exception as e:
            print(name, K, "ERR", e, flush=True)
