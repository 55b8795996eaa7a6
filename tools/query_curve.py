"""Accuracy / latency of the time-critical query against m' (Fig. 9):
the spectral query (bc_evaluate_points_spectral, truncated Parseval in radial-shell order)
beside the exact pair-lens query (bc_evaluate_points), on a workload's shapes.

    python tools/query_curve.py [workload] > profiles/r2/query_curve_<workload>.json

Configurations: 64 (R, t) near each sampled rotation's grid maximum (overlap, where f is
large) -- the exact query is the reference.  Latency: CUDA events around one call on device
buffers, after warm-up (median of 20): one query, and 1,024 queries per call."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import make_config  # noqa: E402
from paper_1711_05075_b200 import ballcorr  # noqa: E402
from paper_1711_05075_b200.presets import correlator_kwargs  # noqa: E402


def timed(fn, reps=20):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main(name="sweep"):
    w = make_config(name, n_rot=8)
    c = ballcorr.Correlator(**correlator_kwargs(name, w.N, w.h, w.t0, w.weights))
    c.shape_upload(0, w.A_xyzr, w.A_w)
    c.shape_upload(1, w.B_xyzr, w.B_w)
    c.spectrum_A()
    kind = "max_real" if w.weights == "complex" else "max_argmax"
    best = c.correlate_rotations(w.R, kind)
    rng = np.random.default_rng(0)
    Rs, ts = [], []
    for r in range(8):
        m = np.array(np.unravel_index(int(best[r]["idx"]), (w.N,) * 3))
        for _ in range(8):
            Rs.append(w.R[r])
            ts.append(np.asarray(w.t0) + w.h * (m + rng.uniform(-3, 3, size=3)))
    R = np.array(Rs)
    t = np.array(ts)
    exact = c.evaluate_points(R, t)
    scale = np.abs(exact).max()
    K = int(c.query("K"))
    band = (2 * K + 1) ** 3
    dev = torch.device("cuda")
    R1, t1 = torch.tensor(R[:1], device=dev), torch.tensor(t[:1], device=dev)
    Rb = torch.tensor(np.resize(R, (1024, 3, 3)), device=dev)
    tb = torch.tensor(np.resize(t, (1024, 3)), device=dev)
    o1 = torch.empty(4, dtype=torch.float64, device=dev)
    ob = torch.empty(4096, dtype=torch.float64, device=dev)
    rows = []
    for lm in range(6, 23, 2):
        m = min(2 ** lm, band, 2 ** 22)
        got = c.evaluate_points_spectral(R, t, m)
        err = float(np.abs(got - exact).max() / scale)
        lat1 = timed(lambda: c.evaluate_points_spectral(R1, t1, m, out=o1[:(2 if c.complex else 1)]))
        latb = timed(lambda: c.evaluate_points_spectral(Rb, tb, m, out=ob[:(2048 if c.complex else 1024)]), reps=5)
        rows.append({"m_prime": m, "rel_max_err_vs_exact": err, "latency_1_query_ms": lat1,
                     "latency_per_query_batch1024_ms": latb / 1024})
        print(rows[-1], file=sys.stderr, flush=True)
    ex1 = timed(lambda: c.evaluate_points(R1, t1, out=o1[:(2 if c.complex else 1)]))
    exb = timed(lambda: c.evaluate_points(Rb, tb, out=ob[:(2048 if c.complex else 1024)]), reps=5)
    print(json.dumps({"workload": name, "n_A": len(w.A_xyzr), "n_B": len(w.B_xyzr), "K": K,
                      "configurations": "64 (R, t): 8 rotations x 8 translations within 3 cells of the rotation's "
                                        "grid maximum", "scale": "max |f_exact| over them",
                      "spectral": rows,
                      "exact_query": {"latency_1_query_ms": ex1, "latency_per_query_batch1024_ms": exb / 1024}},
                     indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
