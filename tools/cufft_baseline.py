"""cuFFT (through torch.fft) on the FFT shapes a library-FFT version of the sweep's
per-rotation path would run (north_star (c): cuFFT only if the hand-written FFTs lose):

* forward: B's spread grid at the fine spacing P/G, G = 1024 (the same oversampling as ours),
  as one 1024^3 FFT (real input, R2C), then the band crop |k_i| <= 255 is a gather;
  also the pruned alternative a library allows: the 256^3 box zero-padded along one axis at a
  time -- three batched 1D transforms of length 1024 over only the lines that carry data;
* inverse: the folded N_p^3 = 256^3 C2R.

Timed with CUDA events after warm-up; prints one JSON line.  Compare with bench.py's
per-rotation stage times (spread + z + y + fold + inverse = 0.67 ms)."""
import json

import torch


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    dev = torch.device("cuda")
    out = {}
    # full oversampled grid (what a spread-then-cuFFT NUFFT does)
    g = torch.randn(1024, 1024, 1024, device=dev)
    out["rfftn_1024^3_ms"] = timed(lambda: torch.fft.rfftn(g))
    del g
    torch.cuda.empty_cache()
    # pruned: z (R2C, 256^2 lines of 1024, keep 256 modes), y (C2C over the 256 x 256 live
    # lines, keep 511), x (C2C over 511 x 256 lines, keep 511)
    box = torch.randn(256, 256, 256, device=dev)

    def pruned():
        t1 = torch.fft.rfft(box, n=1024, dim=2)[:, :, :256]
        t2 = torch.fft.fft(t1, n=1024, dim=1)
        t2 = torch.cat([t2[:, :256], t2[:, -255:]], dim=1)
        t3 = torch.fft.fft(t2, n=1024, dim=0)
        return t3
    out["pruned_1d_passes_ms"] = timed(pruned)
    f = torch.randn(256, 256, 129, dtype=torch.complex64, device=dev)
    out["irfftn_256^3_ms"] = timed(lambda: torch.fft.irfftn(f, s=(256, 256, 256)))
    out["device"] = torch.cuda.get_device_name()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
