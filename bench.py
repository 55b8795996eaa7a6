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
import math
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
    ap.add_argument("--workload", default=WORKLOAD, choices=["tiny", "single", "torus", "sweep", "docking"],
                    help="BASELINE.json config (the metric is quoted on the sweep; the others for reference)")
    ap.add_argument("--rot-per-rank", type=int, default=0, help="0 = the config's rotation count")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-slabs", type=int, default=0, help="x-slabs of the grid in the oracle sample (0 = per config)")
    ap.add_argument("--max-batch", type=int, default=0, help="rotations per launch (0 = library default)")
    ap.add_argument("--concurrency", type=int, default=0, help="batches in flight (0 = library default)")
    args = ap.parse_args()
    if args.cpu_slabs <= 0:
        args.cpu_slabs = CPU_SLABS[args.workload]
    return args


# oracle sample per config: ~10-30 s of fp64 CPU work on the box's cores
CPU_SLABS = {"tiny": 32, "single": 64, "torus": 8, "sweep": 32, "docking": 2}


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

def stage_work(q, N, Np, K, complex_w):
    """Algorithmic work per rotation of each kernel of the spectral path:
    compulsory bytes (input read once + output written once) and FP32 flops
    (5 n log2 n per complex n-point FFT, 6 per complex multiply, 2 per complex add,
    30 per window-profile evaluation of a spread cell)."""
    M = 2 * K + 1
    Kz = M if complex_w else K + 1
    Fz = Np if complex_w else Np // 2 + 1
    L, c = int(q("L_B")), int(q("c_B"))
    lg = math.log2
    fft = lambda n: 5.0 * n * lg(n)
    box = L ** 3 * (8 if complex_w else 4)
    T1 = L * L * Kz * 8
    T2 = L * M * Kz * 8
    Bh = M * M * Kz * 8
    F = Np * Np * Fz * 8
    X1 = N * Np * Fz * 8
    Y1 = N * N * Fz * 8
    axis = lambda lines: lines * c * (fft(L) + 6 * L)       # c coset transforms + coset twiddles
    tiles = q("live_tiles_B")
    spread_z_flops = 30 * q("spread_cells_B") + tiles * 8 * axis(1) + tiles * 16 * Kz * 8
    fold_flops = axis(M * Kz) + 8.0 * M * M * Kz + Np * Fz * fft(Np)
    return {
        "spread_z_B": (T1, spread_z_flops),            # fused spread + z transform: write T1
        "pass_y_fast": (T1 + T2, axis(L * Kz) + 6.0 * L * M * Kz),
        "fold_fast": (T2 + Bh + X1, fold_flops),       # read T2 and A's band, write X1
        "fold_x_inv": (T2 + Bh + X1, fold_flops),
        "spread_B": (box, 30 * q("spread_cells_B")),
        "pass_z_B": (box + T1, axis(L * L)),
        "pass_y_B": (T1 + T2, axis(L * Kz) + 6.0 * L * M * Kz),
        "fold_x": (T2 + Bh + F, axis(M * Kz) + 8.0 * M * M * Kz),
        "inv_x": (F + X1, Np * Fz * fft(Np)),
        "inv_y": (X1 + Y1, N * Fz * fft(Np)),
        "inv_z_reduce": (Y1, (N * N / 2) * fft(Np) + N ** 3),
    }


def alu_peak_tflops():
    """FP32 peak from the unit counts of B200_PROFILING.md: 148 SMs x 128 FP32 lanes x
    2 flop (FFMA) x 1.965 GHz (clocks.max.sm)."""
    return 148 * 128 * 2 * 1.965e9 / 1e12


STAGE_KERNEL = {"fold_fast": "fold_fast_kernel", "spread_z_B": "spread_z_kernel", "pass_y_fast": "pass_y_fast_kernel",
                "inv_y": "pass_kernel", "inv_z_reduce": "last_tma_kernel"}


def ncu_traffic(stage, rotations, workload="sweep"):
    """DRAM bytes per launch of `stage` from the committed ncu --set full capture of the sweep
    (profiles/r1/ncu_traffic.json, per rotation), or None."""
    if workload != "sweep":
        return None
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r1", "ncu_traffic.json")))
        return d["dram_bytes_per_rotation"][STAGE_KERNEL[stage]] * rotations
    except Exception:
        return None


def path_roofline(N, Np, K, complex_w, rot_per_s, peak):
    """SURVEY §8(d)'s two whole-path numbers.  R2 (method efficiency): the method's
    algorithmic bytes per rotation B_alg = 8 M_b 3 (write + read B's band spectrum, read A's)
    + 8 N_pb 2 (folded product write + read) + s N^3 2 (f write + read), M_b / N_pb the band /
    folded mode counts (halved for real weights), times rotations/s over the HBM peak.
    R1: the DRAM bytes ncu measured per rotation over every kernel of the step
    (profiles/r1/ncu_traffic.json) times rotations/s over the peak."""
    half = 1 if complex_w else 2
    M_b = (2 * K + 1) ** 3 / half
    N_pb = Np ** 3 / half
    s = 8 if complex_w else 4
    b_alg = 8 * M_b * 3 + 8 * N_pb * 2 + s * N ** 3 * 2
    out = {"B_alg_per_rot": b_alg, "R2_method_frac": b_alg * rot_per_s / 1e9 / peak}
    try:
        if (N, Np, K, complex_w) != (256, 256, 255, False):
            raise ValueError("the committed ncu capture is the sweep's")
        d = json.load(open(os.path.join(ROOT, "profiles", "r1", "ncu_traffic.json")))
        dram = sum(d["dram_bytes_per_rotation"].values())
        out.update({"dram_bytes_per_rot": dram, "R1_dram_frac": dram * rot_per_s / 1e9 / peak})
    except Exception:
        pass
    return out


def l2_note(w, kw):
    """Flush-or-larger-than-L2 statement of the timing rules (L2 = 126 MB)."""
    if kw["mode"] == "spectral":
        kz = kw["K"] + 1 if w.weights == "real" else 2 * kw["K"] + 1
        mb = (2 * kw["K"] + 1) ** 2 * kz * 8 / 1e6
        return "inputs larger than L2 (A spectrum %.0f MB)" % mb if mb > 126 else \
            "A spectrum %.0f MB fits L2 (re-read every rotation, no flush)" % mb
    return "exact mode: inputs (ball lists) L2-resident, no flush"


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
    slabs = min(slabs, N)
    lo = (N // 2 - slabs // 2, 0, 0)
    hi = (N // 2 - slabs // 2 + slabs, N, N)
    t = time.perf_counter()
    f = oracle.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, R, N, w.h, w.t0, lo, hi)
    dt = time.perf_counter() - t
    n_t = slabs * N * N
    return {"value": n_t / dt, "unit": METRIC, "cores": oracle.oracle_threads(), "kind": "oracle",
            "sample": f"1 rotation x {slabs}x{N}x{N} translations (x-slabs {lo[0]}..{hi[0] - 1}) of the "
                      f"{w.name} workload, fp64, {dt:.2f} s"}, (f[lo[0]:hi[0]], lo[0], hi[0])


def run_reference(args, rank, world):
    if rank != 0:
        return
    w = make_config(args.workload, n_rot=max(args.steps + args.warmup, 1))
    for i in range(args.warmup):
        cpu_oracle_sample(w, w.R[i % w.n_rot], max(2, args.cpu_slabs // 4))[0]
    vals, tot = [], 0.0
    last = None
    for i in range(args.steps):
        last = cpu_oracle_sample(w, w.R[(args.warmup + i) % w.n_rot], args.cpu_slabs)[0]
        vals.append(last["value"])
    v = float(np.mean(vals))
    per_step_translations = min(args.cpu_slabs, w.N) * w.N * w.N
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": METRIC, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_step_translations / v * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "N": w.N, "n_A": len(w.A_xyzr), "n_B": len(w.B_xyzr),
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
    w = make_config(args.workload, n_rot=args.rot_per_rank or None)
    R = w.R if rank == 0 else random_rotations(np.random.default_rng((0, rank)), w.n_rot)
    n_rot = len(R)
    kw = correlator_kwargs(w.name, w.N, w.h, w.t0, w.weights, max_batch=args.max_batch,
                           concurrency=args.concurrency)
    ctx = ballcorr.Correlator(device=local_rank, **kw)
    stream = torch.cuda.current_stream(dev)
    t = time.perf_counter()
    ctx.shape_upload(0, w.A_xyzr, w.A_w)
    ctx.shape_upload(1, w.B_xyzr, w.B_w)
    if world > 1:  # rank 0 computes A's spectrum, NCCL broadcasts it (north_star)
        from paper_1711_05075_b200.sharding import broadcast_spectrum_A
        broadcast_spectrum_A(ctx, src=0)
    else:
        ctx.spectrum_A(stream=stream)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t

    kind = w.output  # sweep: min_argmin; docking: max_real; the others: the full field
    _, oshape, odt = ctx.out_shape(n_rot, kind)
    out_bytes = int(np.prod(oshape)) * np.dtype(odt).itemsize
    R_dev = torch.tensor(R, dtype=torch.float64, device=dev)
    out = torch.empty(out_bytes, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        ctx.correlate_rotations(R_dev, kind, out=out, stream=stream)
    torch.cuda.synchronize()

    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
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
    clocks = sampler.stop()
    # per-stage device times: one more (untimed) step with the library's per-launch CUDA
    # events on; profiling serialises the batches (no concurrent slots), so shares refer to
    # this profiled step
    ctx.set_profiling(True)
    ctx.reset_stage_times()
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    ctx.correlate_rotations(R_dev, kind, out=out, stream=stream)
    p1.record(stream)
    torch.cuda.synchronize()
    prof_ms = p0.elapsed_time(p1)
    stages = ctx.stage_times()
    ctx.set_profiling(False)
    t_max = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms_max = float(t_max.item())
    res = np.frombuffer(out.cpu().numpy().tobytes(), dtype=ballcorr.EXTREMUM_DTYPE) if kind != "full" else None

    units = n_rot * w.N ** 3 * args.steps * world
    value = units / (ms_max / 1e3)

    # gather the per-rotation (min, argmin) of all ranks (outside the timed region)
    best = None
    if world > 1 and res is not None:
        from paper_1711_05075_b200.sharding import gather_extrema, global_best
        vals, idxs = gather_extrema(res["val"], res["idx"], n_rot * world, device=dev)
        best = global_best(vals, idxs, "min" if kind == "min_argmin" else "max")

    # e2e through the public API with host buffers (pinned), copies inside the timed region
    R_host = torch.tensor(R, dtype=torch.float64).pin_memory()
    out_host = torch.empty(out_bytes, dtype=torch.uint8).pin_memory()
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
    # roofline of the dominant kernel (largest share of device time in the timed region):
    # HBM-bound if its algorithmic flop/byte is below the FP32 ridge, else ALU-bound
    q = ctx.query
    spectral = kw["mode"] == "spectral"
    work = stage_work(q, w.N, kw["Np"], kw["K"], w.weights == "complex") if spectral else {}
    peak, peak_kind = measured_peaks()
    alu_peak = alu_peak_tflops()
    ridge = alu_peak * 1e12 / (peak * 1e9)
    batch = int(q("batch")) if spectral else 1
    per_stage = {}
    for name, (tot_ms, nl) in stages.items():
        if name not in work:
            continue
        by, fl = work[name]
        avg_s = tot_ms / nl / 1e3
        per_stage[name] = {"ms_per_rot": tot_ms / n_rot, "share": tot_ms / prof_ms,
                           "hbm_GBps": by * batch / avg_s / 1e9, "hbm_frac": by * batch / avg_s / 1e9 / peak,
                           "fp32_TFLOPs": fl * batch / avg_s / 1e12, "alu_frac": fl * batch / avg_s / 1e12 / alu_peak,
                           "flop_per_byte": fl / by}
    roof = None
    if per_stage:
        name = max(per_stage, key=lambda k: per_stage[k]["share"])
        st = per_stage[name]
        tot_ms, nl = stages[name]
        by, fl = work[name]
        alu = fl / by > ridge
        roof = {"bound": "alu" if alu else "hbm", "kernel": name,
                "achieved": st["fp32_TFLOPs"] if alu else st["hbm_GBps"],
                "peak": alu_peak if alu else peak, "unit": "TFLOP/s" if alu else "GB/s",
                "frac": st["alu_frac"] if alu else st["hbm_frac"], "traffic": ncu_traffic(name, batch, w.name),
                "traffic_source": "profiles/r1/ncu_traffic.json (ncu --set full, dram__bytes_read.sum + "
                                  "dram__bytes_write.sum per rotation x rotations per launch)",
                "peak_source": ("derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz" if alu else peak_kind),
                "alg_bytes_per_launch": by * batch, "alg_flops_per_launch": fl * batch,
                "avg_launch_ms": tot_ms / nl, "share_of_step": st["share"],
                "hbm_view": {"achieved_GBps": st["hbm_GBps"], "peak_GBps": peak, "frac": st["hbm_frac"]},
                "ridge_flop_per_byte": ridge}
    cpu = None
    rel_err = None
    if world == 1 and not args.no_cpu_baseline:
        cpu, (f_ref, x0, x1) = cpu_oracle_sample(w, R[0], args.cpu_slabs)
        # the metric's third part (BASELINE.json: "rel max error"): this GPU run's full f of the
        # same rotation (outside the timed region) against the oracle on the sampled slabs
        f_gpu = ctx.correlate_rotations(R[:1], "full")[0][x0:x1]
        if w.weights == "complex":
            f_gpu = f_gpu[..., 0] + 1j * f_gpu[..., 1]
        tol = 1e-9 if kw["precision"] == "f64" else 1e-4
        rel_err = {"value": float(np.abs(f_gpu - f_ref).max() / np.abs(f_ref).max()), "tolerance": tol,
                   "sample": "rotation 0, the cpu_baseline slabs (x %d..%d, %d translations), fp64 oracle"
                             % (x0, x1 - 1, f_ref.size)}
    line = {
        "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": kw["precision"], "data": "synthetic",
        "config": {"workload": w.name, "N": w.N, "n_A": len(w.A_xyzr), "n_B": len(w.B_xyzr),
                   "rotations_per_rank_per_step": n_rot, "mode": kw["mode"], "Np": kw["Np"], "K": kw["K"],
                   "output": kind, "l2": l2_note(w, kw),
                   "setup_s": setup_s,
                   "spectrum_A": "rank 0, NCCL broadcast" if world > 1 else "computed"},
        "clocks": clocks,
        "gpu_launches": launches,
        "e2e": {"value": e2e_value, "unit": METRIC, "h2d_bytes_per_step": int(R.size * 8),
                "d2h_bytes_per_step": out_bytes},
        "roofline": roof,
        "path_roofline": path_roofline(w.N, kw["Np"], kw["K"], w.weights == "complex",
                                       n_rot * args.steps / (ms_max / 1e3), peak) if spectral else None,
        "cpu_baseline": cpu,
        "rel_max_error": rel_err,
        "stages_ms_per_step": {k: v[0] for k, v in stages.items()},
        "profiled_step_ms": prof_ms,
        "stages": per_stage,
        "result_sample": None if res is None else {"rot0_val": float(res[0]["val"]), "rot0_idx": int(res[0]["idx"]),
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
