#!/usr/bin/env python
"""Benchmark of the hot path: f_R(t) over the 256^3 translation grid for a batch of
rotations of the "Rotational sweep" workload (BASELINE.json configs[3], the
config the north_star metric is quoted on), per-rotation (min, argmin).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One process per GPU (torchrun for N > 1, NCCL).  A step = one pass of the whole
path (spread -> box DFT -> spectral product/fold -> inverse FFT -> reduction) over
the rank's batch of rotations; each rank owns its own batch (weak scaling, no
data-path collective).  Rank 0 prints one JSON line.

`--impl reference` times the fp64 CPU oracle (oracle/, the only other place
this script executes it) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import make_config, random_rotations  # noqa: E402

WORKLOAD = "sweep"
METRIC = "translations*rotations/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rot-per-rank", type=int, default=512)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-slabs", type=int, default=32, help="x-slabs of the 256^3 grid in the oracle sample")
    return ap.parse_args()


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi sampling during the timed region (clock line of B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- algorithmic bytes

def stage_bytes(q, N, Np, K, complex_w):
    """Compulsory bytes per rotation of each kernel of the spectral path:
    its input read once plus its output written once."""
    M = 2 * K + 1
    Kz = M if complex_w else K + 1
    Fz = Np if complex_w else Np // 2 + 1
    L = int(q("L_B"))
    box = L ** 3 * (8 if complex_w else 4)
    T1 = L * L * Kz * 8
    T2 = L * M * Kz * 8
    Bh = M * M * Kz * 8
    F = Np * Np * Fz * 8
    X1 = N * Np * Fz * 8
    Y1 = N * N * Fz * 8
    return {
        "spread_z_B": T1,             # fused spread + z transform: write T1 (the box stays on chip)
        "fold_x_inv": T2 + Bh + X1,   # fused fold + inverse x: read T2 and A's band, write X1
        "fold_fast": T2 + Bh + X1,    # same, compile-time plan of the sweep's shape
        "pass_y_fast": T1 + T2,       # read T1, write T2 (compile-time plan)
        "spread_B": box,              # write the smoothed density box of R B
        "pass_z_B": box + T1,         # read box, write T1
        "pass_y_B": T1 + T2,          # read T1, write T2
        "fold_x": T2 + Bh + F,        # read T2 and A's band spectrum, write the folded product F
        "inv_x": F + X1,
        "inv_y": X1 + Y1,
        "inv_z_reduce": Y1,           # read Y1, write 16 B of keys
    }


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------------------- CPU oracle sample

def cpu_oracle_sample(w, R, slabs):
    """Oracle (fp64 C/OpenMP) on one rotation over `slabs` x-slabs of the grid."""
    import oracle
    oracle.build_oracle()
    N = w.N
    lo = (N // 2 - slabs // 2, 0, 0)
    hi = (N // 2 - slabs // 2 + slabs, N, N)
    t = time.perf_counter()
    oracle.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, R, N, w.h, w.t0, lo, hi)
    dt = time.perf_counter() - t
    n_t = slabs * N * N
    return {"value": n_t / dt, "unit": METRIC, "cores": oracle.oracle_threads(), "kind": "oracle",
            "sample": f"1 rotation x {slabs}x{N}x{N} translations (x-slabs {lo[0]}..{hi[0] - 1}) of the "
                      f"{WORKLOAD} workload, fp64, {dt:.2f} s"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    w = make_config(WORKLOAD, n_rot=max(args.steps + args.warmup, 1))
    for i in range(args.warmup):
        cpu_oracle_sample(w, w.R[i % w.n_rot], max(2, args.cpu_slabs // 4))
    vals, tot = [], 0.0
    last = None
    for i in range(args.steps):
        last = cpu_oracle_sample(w, w.R[(args.warmup + i) % w.n_rot], args.cpu_slabs)
        vals.append(last["value"])
    v = float(np.mean(vals))
    per_step_translations = args.cpu_slabs * w.N * w.N
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": METRIC, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_step_translations / v * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "N": w.N, "n_A": len(w.A_xyzr), "n_B": len(w.B_xyzr),
                   "translations_per_step": per_step_translations, "rotations_per_step": 1},
        "cpu_baseline": {"value": v, "unit": METRIC, "cores": last["cores"], "kind": "oracle", "sample": last["sample"]},
        "e2e": {"value": v, "unit": METRIC, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our path

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1711_05075_b200 import ballcorr
    from paper_1711_05075_b200.presets import correlator_kwargs

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    w = make_config(WORKLOAD, n_rot=args.rot_per_rank)
    R = w.R if rank == 0 else random_rotations(np.random.default_rng((0, rank)), args.rot_per_rank)
    n_rot = len(R)
    kw = correlator_kwargs(WORKLOAD, w.N, w.h, w.t0, w.weights)
    ctx = ballcorr.Correlator(device=local_rank, **kw)
    stream = torch.cuda.current_stream(dev)
    t = time.perf_counter()
    ctx.shape_upload(0, w.A_xyzr, w.A_w)
    ctx.shape_upload(1, w.B_xyzr, w.B_w)
    ctx.spectrum_A(stream=stream)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t

    kind = "min_argmin"
    R_dev = torch.tensor(R, dtype=torch.float64, device=dev)
    out = torch.empty(n_rot * 16, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        ctx.correlate_rotations(R_dev, kind, out=out, stream=stream)
    torch.cuda.synchronize()

    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    ctx.set_profiling(True)
    ctx.reset_stage_times()
    l0 = ctx.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        ctx.correlate_rotations(R_dev, kind, out=out, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    launches = ctx.launch_count() - l0
    stages = ctx.stage_times()
    ctx.set_profiling(False)
    clocks = sampler.stop()
    t_max = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms_max = float(t_max.item())
    res = np.frombuffer(out.cpu().numpy().tobytes(), dtype=ballcorr.EXTREMUM_DTYPE)

    units = n_rot * w.N ** 3 * args.steps * world
    value = units / (ms_max / 1e3)

    # gather the per-rotation (min, argmin) of all ranks (outside the timed region)
    best = None
    if world > 1:
        from paper_1711_05075_b200.sharding import gather_extrema, global_best
        vals, idxs = gather_extrema(res["val"], res["idx"], n_rot * world, device=dev)
        best = global_best(vals, idxs, "min")

    # e2e through the public API with host buffers (pinned), copies inside the timed region
    R_host = torch.tensor(R, dtype=torch.float64).pin_memory()
    out_host = torch.empty(n_rot * 16, dtype=torch.uint8).pin_memory()
    ctx.correlate_rotations(R_host, kind, out=out_host, stream=stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    h0 = torch.cuda.Event(enable_timing=True)
    h1 = torch.cuda.Event(enable_timing=True)
    h0.record(stream)
    for _ in range(args.e2e_steps):
        ctx.correlate_rotations(R_host, kind, out=out_host, stream=stream)
    h1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([h0.elapsed_time(h1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = n_rot * w.N ** 3 * args.e2e_steps * world / (float(e2e_ms.item()) / 1e3)

    if rank != 0:
        return
    # roofline of the dominant kernel (largest share of device time in the timed region)
    q = ctx.query
    sb = stage_bytes(q, w.N, kw["Np"], kw["K"], w.weights == "complex")
    peak, peak_kind = measured_peaks()
    dom = max(stages.items(), key=lambda kv: kv[1][0]) if stages else None
    roof = None
    if dom is not None and dom[0] in sb:
        name, (tot_ms, nl) = dom
        batch = int(q("batch"))
        per_launch_bytes = sb[name] * batch
        avg_s = tot_ms / nl / 1e3
        achieved = per_launch_bytes / avg_s / 1e9
        roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None, "peak_source": peak_kind,
                "alg_bytes_per_launch": per_launch_bytes, "avg_launch_ms": avg_s * 1e3,
                "share_of_step": tot_ms / ms}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_sample(w, R[0], args.cpu_slabs)
    line = {
        "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "N": w.N, "n_A": len(w.A_xyzr), "n_B": len(w.B_xyzr),
                   "rotations_per_rank_per_step": n_rot, "mode": kw["mode"], "Np": kw["Np"], "K": kw["K"],
                   "output": kind, "l2": "inputs larger than L2 (A spectrum %.0f MB)" % (
                       (2 * kw["K"] + 1) ** 2 * (kw["K"] + 1) * 8 / 1e6),
                   "setup_s": setup_s},
        "clocks": clocks,
        "gpu_launches": launches,
        "e2e": {"value": e2e_value, "unit": METRIC, "h2d_bytes_per_step": int(R.size * 8),
                "d2h_bytes_per_step": int(n_rot * 16)},
        "roofline": roof,
        "cpu_baseline": cpu,
        "stages_ms_per_step": {k: v[0] / args.steps for k, v in stages.items()},
        "result_sample": {"rot0_min": float(res[0]["val"]), "rot0_argmin": int(res[0]["idx"]),
                          "global_best": best},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl")
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
