"""Probe: capture one correlate_rotations call (device R and out) into a CUDA graph and compare
replay with eager calls (bitwise output, time per call).  python tools/graph_probe.py tiny"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth import make_config  # noqa: E402
from paper_1711_05075_b200 import ballcorr  # noqa: E402
from paper_1711_05075_b200.presets import correlator_kwargs  # noqa: E402

for name in sys.argv[1:]:
    w = make_config(name)
    c = ballcorr.Correlator(**correlator_kwargs(name, w.N, w.h, w.t0, w.weights))
    c.shape_upload(0, w.A_xyzr, w.A_w)
    c.shape_upload(1, w.B_xyzr, w.B_w)
    c.spectrum_A()
    kind = w.output if w.output != "max_real" else "max_real"
    R = torch.tensor(w.R[:1] if name in ("tiny", "single") else w.R[:16], dtype=torch.float64, device="cuda")
    _, shp, dt = c.out_shape(R.shape[0], kind)
    nbytes = int(np.prod(shp)) * np.dtype(dt).itemsize
    out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            c.correlate_rotations(R, kind, out=out, stream=s)
    torch.cuda.synchronize()
    ref = out.clone()
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=s):
            c.correlate_rotations(R, kind, out=out, stream=s)
    except Exception as e:  # noqa: BLE001
        print(name, "capture failed:", e)
        continue
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    same = torch.equal(out, ref)
    K = 200
    for mode in ("eager", "graph", "eager", "graph"):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(K):
                if mode == "graph":
                    g.replay()
                else:
                    c.correlate_rotations(R, kind, out=out, stream=s)
            e1.record(s)
        torch.cuda.synchronize()
        print(name, mode, "bitwise" if same else "DIFFERS", round(e0.elapsed_time(e1) / K, 4), "ms/call")
