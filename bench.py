#!/usr/bin/env python
"""Benchmark of the hot path: f_R(t) over the 256^3 translation grid for a batch of
rotations of the "Rotational sweep" workload (BASELINE.json configs[3], the
config the north_star metric is quoted on), per-rotation (min, argmin).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One process per GPU (torchrun for N > 1, NCCL; `--gpus N` without a torchrun
environment re-launches itself under torch.distributed.run).  A step = one pass of
the whole path (spread -> box DFT -> spectral product/fold -> inverse FFT ->
reduction) over the config's 512 rotations, sharded over the ranks in contiguous
blocks (sharding.rotation_block; strong scaling), followed by the
all-gather of the per-rotation (min, argmin) records -- T includes it (SURVEY.md
§8(d)).  `--scaling weak` keeps the rank's block at the full rotation count instead.
Rank 0 prints one JSON line.  `--dry-run` runs the same launcher and protocol on CPU
(gloo, a stand-in correlator; tests/test_bench_launcher.py).

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
# bc_extremum (include/ballcorr.h): {double val; int64 idx}
REC_DTYPE = np.dtype([("val", np.float64), ("idx", np.int64)])


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
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's rotations sharded over the ranks (headline); weak: every rank "
                         "correlates its own full rotation set")
    ap.add_argument("--collectives", default="nccl", choices=["nccl", "p2p"],
                    help="strong scaling: nccl = NCCL broadcast of A's spectrum + all-gather of the records per "
                         "step; p2p = A's spectrum sharded by balls and reduced over peer memory inside the A'' "
                         "build, records stored into every rank's buffer by the reduction epilogue (no gather)")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay each step's kernels from a CUDA graph (auto: one GPU, <= 16 rotations per step)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU-only launcher/protocol check: gloo, stand-in correlator, no CUDA")
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
    """Algorithmic work per rotation of each kernel of the spectral path.

    Bytes: SURVEY.md §8(d)'s per-unit figures wherever the kernel carries a §8(d) step --
    the fold (a5: spectral product + fold) moves A's band spectrum (read once per rotation,
    8 M_b bytes, M_b = M^3 / 2 modes for real weights) and writes the folded product
    (8 N_pb, N_pb = Np^3 / 2); the last pass (a6 + a7) reads the folded/inverse-transformed
    rows and writes f or nothing (reductions).  Multi-pass FFT intermediates (T1, T2, X1, Y1)
    are implementation traffic, excluded by §8(d); they are listed separately as
    `impl_bytes` (compulsory read + write of each kernel's own input and output).
    Flops (FP32 view): 5 n log2 n per complex n-point FFT, 6 per complex multiply, 2 per
    complex add, 30 per window-profile evaluation of a spread cell."""
    M = 2 * K + 1
    Kz = M if complex_w else K + 1
    Fz = Np if complex_w else Np // 2 + 1
    half = 1 if complex_w else 2
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
    a5 = 8 * M ** 3 / half + 8 * Np ** 3 / half       # §8(d): A band read + folded product write
    axis = lambda lines: lines * c * (fft(L) + 6 * L)       # c coset transforms + coset twiddles
    tiles = q("live_tiles_B")
    spread_z_flops = 30 * q("spread_cells_B") + tiles * 8 * axis(1) + tiles * 16 * Kz * 8
    fold_flops = axis(M * Kz) + 8.0 * M * M * Kz + Np * Fz * fft(Np)
    # name: (§8(d) algorithmic bytes or None, implementation bytes, flops)
    return {
        "spread_z_B": (None, T1, spread_z_flops),          # fused spread + z transform: write T1
        "pass_y_fast": (None, T1 + T2, axis(L * Kz) + 6.0 * L * M * Kz),
        "fold_fast": (a5, T2 + Bh + X1, fold_flops),       # read T2 and A's band, write X1
        "fold_x_inv": (a5, T2 + Bh + X1, fold_flops),
        "spread_B": (None, box, 30 * q("spread_cells_B")),
        "pass_z_B": (None, box + T1, axis(L * L)),
        "pass_y_B": (None, T1 + T2, axis(L * Kz) + 6.0 * L * M * Kz),
        "fold_x": (a5, T2 + Bh + F, axis(M * Kz) + 8.0 * M * M * Kz),
        "inv_x": (None, F + X1, Np * Fz * fft(Np)),
        "inv_y": (None, X1 + Y1, N * Fz * fft(Np)),
        "inv_z_reduce": (None, Y1, (N * N / 2) * fft(Np) + N ** 3),
    }


def alu_peak_tflops():
    """FP32 peak from the unit counts of B200_PROFILING.md: 148 SMs x 128 FP32 lanes x
    2 flop (FFMA) x 1.965 GHz (clocks.max.sm)."""
    return 148 * 128 * 2 * 1.965e9 / 1e12


STAGE_KERNEL = {"fold_fast": "fold_fast_kernel", "spread_z_B": "spread_z_kernel", "pass_y_fast": "pass_y_fast_kernel",
                "inv_y": "pass_kernel", "inv_z_reduce": "last_tma_kernel"}


TRAFFIC_FILES = ("profiles/r2/ncu_traffic.json", "profiles/r1/ncu_traffic.json")


def _traffic_file():
    for rel in TRAFFIC_FILES:
        path = os.path.join(ROOT, rel)
        if os.path.exists(path):
            return rel, json.load(open(path))
    return None, None


def ncu_traffic(stage, rotations, workload="sweep"):
    """DRAM bytes per launch of `stage` (dram__bytes_read.sum + dram__bytes_write.sum) from the
    committed ncu --set full capture of the sweep at the bench's own rotations per launch
    (profiles/r2/ncu_traffic.json; per rotation x rotations per launch), or None."""
    if workload != "sweep":
        return None
    rel, d = _traffic_file()
    try:
        return d["dram_bytes_per_rotation"][STAGE_KERNEL[stage]] * rotations
    except Exception:
        return None


def smem_view(stage, rotations, avg_launch_s, sm_mhz, workload="sweep"):
    """Shared-memory crossbar view of the dominant kernel: ncu's shared wavefronts per rotation
    (profiles/r2/ncu_smem.json, from the committed --set full summary) x rotations per launch,
    over the live launch time, against 148 SM x 1 wavefront (128 B) per cycle at the clock
    sampled under load (B300_MICROARCH.md "LDS/STS": 128/N B/cyc/SM).  None off the sweep."""
    path = os.path.join(ROOT, "profiles/r2/ncu_smem.json")
    if workload != "sweep" or not os.path.exists(path) or not sm_mhz:
        return None
    try:
        k = json.load(open(path))["per_kernel"][STAGE_KERNEL[stage]]
    except Exception:
        return None
    wf = k["wavefronts_per_rotation"] * rotations
    peak = 148 * sm_mhz * 1e6
    return {"wavefronts_per_launch": wf, "Gwavefronts_per_s": wf / avg_launch_s / 1e9, "peak_Gwavefronts_per_s": peak / 1e9,
            "frac": wf / avg_launch_s / peak, "bank_conflict_share": k["bank_conflicts_per_rotation"] / k["wavefronts_per_rotation"],
            "source": "profiles/r2/ncu_smem.json (l1tex__data_pipe_lsu_wavefronts_mem_shared.sum); peak 148 SM x 1 "
                      "wavefront/cycle x the sampled SM clock"}


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
        rel, d = _traffic_file()
        dram = sum(d["dram_bytes_per_rotation"].values())
        out.update({"dram_bytes_per_rot": dram, "R1_dram_frac": dram * rot_per_s / 1e9 / peak, "dram_source": rel})
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

class _DryCorrelator:
    """--dry-run stand-in for ballcorr.Correlator (CPU, no CUDA): deterministic per-rotation
    extremum records (a function of the rotation matrix only), so that any sharding of the
    rotations must reproduce the single-rank records exactly."""

    def __init__(self):
        self._launches = 0

    def correlate_rotations(self, R, kind, out=None, stream=None):
        R = np.asarray(R.cpu() if hasattr(R, "cpu") else R, dtype=np.float64).reshape(-1, 9)
        rec = np.zeros(len(R), dtype=REC_DTYPE)
        rec["val"] = (R * np.arange(1, 10)).sum(axis=1)
        rec["idx"] = (np.abs(R[:, 0]) * 1e6).astype(np.int64)
        self._launches += 1
        buf = np.frombuffer(rec.tobytes(), dtype=np.uint8)
        out[: buf.size].copy_(__import__("torch").from_numpy(buf.copy()))
        return out

    def launch_count(self):
        return self._launches


def gather_records(out_local, n_local, cap, world, dev):
    """All-gather of the ranks' per-rotation records (16-byte bc_extremum each, padded to
    `cap` rotations per rank) into one [world * cap * 16] byte tensor on `dev` (NCCL over
    NVLink on the GPU box, gloo on CPU); rank r's block sits at [r * cap, r * cap + n_r)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return out_local
    send = out_local if n_local == cap else torch.cat(
        [out_local, torch.zeros((cap - n_local) * 16, dtype=torch.uint8, device=dev)])
    recv = torch.empty(world * cap * 16, dtype=torch.uint8, device=dev)
    dist.all_gather(list(recv.chunk(world)), send)
    return recv


def unpack_global(recv, n_rot, world):
    """Global rotation-order records from gather_records' buffer."""
    from paper_1711_05075_b200.sharding import rotation_block
    raw = np.frombuffer(recv.cpu().numpy().tobytes(), dtype=REC_DTYPE)
    if world == 1:
        return raw[:n_rot]
    cap = -(-n_rot // world)
    out = np.empty(n_rot, dtype=REC_DTYPE)
    for r in range(world):
        s0, e0 = rotation_block(n_rot, r, world)
        out[s0:e0] = raw[r * cap: r * cap + (e0 - s0)]
    return out


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1711_05075_b200.presets import correlator_kwargs
    from paper_1711_05075_b200.sharding import rotation_block, global_best

    dry = args.dry_run
    if not dry:
        from paper_1711_05075_b200 import ballcorr
    dev = torch.device("cpu") if dry else torch.device("cuda", local_rank)
    if not dry:
        torch.cuda.set_device(local_rank)
    w = make_config(args.workload, n_rot=args.rot_per_rank or None)
    n_all = w.n_rot
    if args.scaling == "strong":
        s0, e0 = rotation_block(n_all, rank, world)
        R = w.R[s0:e0]
        units_per_step = n_all            # the whole job: the config's rotations once
    else:
        R = w.R if rank == 0 else random_rotations(np.random.default_rng((0, rank)), n_all)
        s0, e0 = 0, n_all
        units_per_step = n_all * world
    n_rot = len(R)
    cap = -(-n_all // world) if args.scaling == "strong" else n_all
    kw = correlator_kwargs(w.name, w.N, w.h, w.t0, w.weights, max_batch=args.max_batch,
                           concurrency=args.concurrency)
    t = time.perf_counter()
    if dry:
        ctx = _DryCorrelator()
        stream = None
    else:
        ctx = ballcorr.Correlator(device=local_rank, **kw)
        stream = torch.cuda.current_stream(dev)
        ctx.shape_upload(0, w.A_xyzr, w.A_w)
        ctx.shape_upload(1, w.B_xyzr, w.B_w)
        p2p = args.collectives == "p2p" and args.scaling == "strong"
        if p2p:  # (a world of one needs no process group: the helpers skip the exchanges)
            from paper_1711_05075_b200.sharding import allreduce_spectrum_A_p2p
            allreduce_spectrum_A_p2p(ctx, len(w.A_xyzr))
        elif world > 1:  # rank 0 computes A's spectrum, NCCL broadcasts it (north_star)
            from paper_1711_05075_b200.sharding import broadcast_spectrum_A
            broadcast_spectrum_A(ctx, src=0)
        else:
            ctx.spectrum_A(stream=stream)
        torch.cuda.synchronize()
    setup_s = time.perf_counter() - t

    kind = w.output  # sweep: min_argmin; docking: max_real; the others: the full field
    reduced = kind != "full"
    if dry:
        out_bytes = n_rot * 16
    else:
        _, oshape, odt = ctx.out_shape(n_rot, kind)
        out_bytes = int(np.prod(oshape)) * np.dtype(odt).itemsize
    R_dev = torch.tensor(R, dtype=torch.float64, device=dev)
    out = torch.empty(max(out_bytes, 16), dtype=torch.uint8, device=dev)

    p2p = (not dry) and args.collectives == "p2p" and args.scaling == "strong" and reduced
    if p2p:  # the job's records, stored into every rank's buffer by the reduction epilogue
        from paper_1711_05075_b200.sharding import result_peers_p2p
        glob_ptr, glob_p2p = ctx.result_buffer(n_all * 16)  # an allocation base (IPC-exportable)
        _, mapped = result_peers_p2p(ctx, glob_ptr, n_all)

    def step():
        ctx.correlate_rotations(R_dev, kind, out=out, stream=stream)
        if p2p:  # nothing to launch: the epilogue stored the records in every rank's buffer
            return glob_p2p
        if reduced:  # the per-rotation results of every rank, in global order, on every rank
            return gather_records(out[:out_bytes], n_rot, cap, world if args.scaling == "strong" else 1, dev)
        return out

    def sync():
        if not dry:
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    sync()
    # small steps (one or a few rotations: Tiny, Single) are bound by the host-side cost of the
    # launches, not by the GPU: replay the call's kernels from a CUDA graph (captured from the
    # same library call on a side stream; the replay is bitwise the eager result)
    graph, graph_launches = None, 0
    if (not dry and world == 1 and not p2p and
            (args.graph == "on" or (args.graph == "auto" and n_rot <= 16))):
        gs = torch.cuda.Stream(dev)
        gs.wait_stream(stream)
        lc0 = ctx.launch_count()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            ctx.correlate_rotations(R_dev, kind, out=out, stream=gs)
        graph_launches = ctx.launch_count() - lc0
        stream.wait_stream(gs)
        graph.replay()
        sync()

        def step():  # noqa: F811
            graph.replay()
            if reduced:
                return gather_records(out[:out_bytes], n_rot, cap, 1, dev)
            return out

    sampler = None if dry else ClockSampler(local_rank)
    if sampler:
        sampler.start()
        time.sleep(0.3)
    l0 = ctx.launch_count()
    if world > 1:
        dist.barrier()
    sync()
    if dry:
        t0 = time.perf_counter()
    else:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
    for _ in range(args.steps):
        glob = step()
    if dry:
        ms = (time.perf_counter() - t0) * 1e3
    else:
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    if world > 1:
        dist.barrier()
    launches = ctx.launch_count() - l0 + graph_launches * args.steps
    clocks = sampler.stop() if sampler else None
    t_max = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms_max = float(t_max.item())
    value = units_per_step * w.N ** 3 * args.steps / (ms_max / 1e3)
    best = None
    if reduced and args.scaling == "strong":
        recs = (np.frombuffer(glob.cpu().numpy().tobytes(), dtype=REC_DTYPE) if p2p
                else unpack_global(glob, n_all, world))
        best = global_best(recs["val"], recs["idx"], "min" if kind == "min_argmin" else "max")
        best = {"rotation": best[0], "value": best[1], "translation_index": best[2],
                "records_sha1": __import__("hashlib").sha1(recs.tobytes()).hexdigest()}

    if dry:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": value, "unit": METRIC, "n_gpus": world, "steps": args.steps,
                              "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                              "scaling": args.scaling, "dry_run": True, "gpu_launches": 0,
                              "config": {"workload": w.name, "rotations_per_step": n_all,
                                         "rotations_per_rank": [rotation_block(n_all, r, world)
                                                                for r in range(world)]},
                              "result_sample": {"global_best": best}}), flush=True)
        return

    if p2p:
        ctx.set_result_peers([])  # the untimed legs below write no peer buffers
        for ptr in mapped:
            ctx.ipc_close(ptr)
    # per-stage device times: one more (untimed) step with the library's per-launch CUDA
    # events on (profiling serialises the batches), so shares refer to this profiled step
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

    # e2e through the public API with host buffers (pinned): the H2D copy of the rank's R block
    # and the D2H read of its results happen inside the call, inside the timed region
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
    e2e_value = units_per_step * w.N ** 3 * args.e2e_steps / (float(e2e_ms.item()) / 1e3)

    if rank != 0:
        return
    q = ctx.query
    spectral = kw["mode"] == "spectral"
    work = stage_work(q, w.N, kw["Np"], kw["K"], w.weights == "complex") if spectral else {}
    peak, peak_kind = measured_peaks()
    alu_peak = alu_peak_tflops()
    batch = int(q("batch")) if spectral else 1
    per_stage = {}
    for name, (tot_ms, nl) in stages.items():
        if name not in work:
            continue
        alg, impl, fl = work[name]
        avg_s = tot_ms / nl / 1e3
        per_stage[name] = {"ms_per_rot": tot_ms / n_rot, "share": tot_ms / prof_ms,
                           "alg_bytes_per_rot": alg,
                           "hbm_frac_alg": None if alg is None else alg * batch / avg_s / 1e9 / peak,
                           "impl_GBps": impl * batch / avg_s / 1e9, "hbm_frac_impl": impl * batch / avg_s / 1e9 / peak,
                           "fp32_TFLOPs": fl * batch / avg_s / 1e12, "alu_frac": fl * batch / avg_s / 1e12 / alu_peak}
    roof = None
    if per_stage:
        name = max(per_stage, key=lambda k: per_stage[k]["share"])
        st = per_stage[name]
        tot_ms, nl = stages[name]
        alg, impl, fl = work[name]
        by = alg if alg is not None else impl
        achieved = by * batch / (tot_ms / nl / 1e3) / 1e9
        traffic = ncu_traffic(name, batch, w.name)
        roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "bytes_basis": ("SURVEY.md §8(d) a5: A band read 8*M^3/2 + folded product write 8*Np^3/2 per "
                                "rotation x rotations per launch" if alg is not None else "kernel input + output"),
                "alg_bytes_per_launch": by * batch, "rotations_per_launch": batch,
                "avg_launch_ms": tot_ms / nl, "share_of_step": st["share"],
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (%s)" % peak_kind,
                "traffic_source": (_traffic_file()[0] or "none") + " (ncu --set full, dram__bytes_read.sum + "
                                  "dram__bytes_write.sum per rotation x rotations per launch)",
                "impl_view": {"bytes_per_launch": impl * batch, "GBps": st["impl_GBps"], "frac": st["hbm_frac_impl"],
                              "note": "compulsory read+write of the kernel's own input/output incl. FFT intermediates"},
                "alu_view": {"fp32_TFLOPs": st["fp32_TFLOPs"], "peak_TFLOPs": alu_peak, "frac": st["alu_frac"],
                             "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz"},
                "smem_view": smem_view(name, batch, tot_ms / nl / 1e3, (clocks or {}).get("sm_mhz"), w.name)}
    cpu = None
    rel_err = None
    if world == 1 and not args.no_cpu_baseline:
        cpu, (f_ref, x0, x1) = cpu_oracle_sample(w, w.R[0], args.cpu_slabs)
        # the metric's third part (BASELINE.json: "rel max error"): this GPU run's full f of the
        # same rotation (outside the timed region) against the oracle on the sampled slabs
        f_gpu = ctx.correlate_rotations(w.R[:1], "full")[0][x0:x1]
        if w.weights == "complex":
            f_gpu = f_gpu[..., 0] + 1j * f_gpu[..., 1]
        tol = 1e-9 if kw["precision"] == "f64" else 1e-4
        rel_err = {"value": float(np.abs(f_gpu - f_ref).max() / np.abs(f_ref).max()), "tolerance": tol,
                   "sample": "rotation 0, the cpu_baseline slabs (x %d..%d, %d translations), fp64 oracle"
                             % (x0, x1 - 1, f_ref.size)}
    line = {
        "metric": METRIC, "value": value, "unit": METRIC, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": kw["precision"], "data": "synthetic",
        "config": {"workload": w.name, "N": w.N, "n_A": len(w.A_xyzr), "n_B": len(w.B_xyzr),
                   "rotations_per_step": units_per_step, "rotations_per_rank": n_rot,
                   "mode": kw["mode"], "Np": kw["Np"], "K": kw["K"], "output": kind, "l2": l2_note(w, kw),
                   "timed": ("per step: every rank correlates its rotation block; its reduction epilogue stores "
                             "the records into every rank's job-wide buffer over peer memory (no gather launch)"
                             if p2p else
                             "per step: every rank correlates its rotation block, then the NCCL all-gather of "
                             "the per-rotation records (strong scaling, SURVEY.md §8(d)-(e))"
                             if args.scaling == "strong" else "per step: every rank its own full rotation set"),
                   "collectives": args.collectives,
                   "cuda_graph": graph is not None,
                   "setup_s": setup_s,
                   "spectrum_A": ("sharded by balls, partials reduced over peer memory in the A'' build" if p2p
                                  else "rank 0, NCCL broadcast" if world > 1 else "computed")},
        "clocks": clocks,
        "gpu_launches": launches,
        "e2e": {"value": e2e_value, "unit": METRIC, "h2d_bytes_per_step": int(R.size * 8),
                "d2h_bytes_per_step": out_bytes,
                "note": "bc_correlate_rotations with pinned host R and host out (copies inside the call); "
                        "per rank, max over ranks, without the all-gather"},
        "roofline": roof,
        "path_roofline": path_roofline(w.N, kw["Np"], kw["K"], w.weights == "complex",
                                       units_per_step * args.steps / (ms_max / 1e3) / world, peak) if spectral else None,
        "cpu_baseline": cpu,
        "rel_max_error": rel_err,
        "stages_ms_per_step": {k: v[0] for k, v in stages.items()},
        "profiled_step_ms": prof_ms,
        "stages": per_stage,
        "result_sample": {"global_best": best},
    }
    print(json.dumps(line), flush=True)


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` outside torchrun: one process per GPU under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        if not args.dry_run:
            torch.cuda.set_device(local_rank)
        dist.init_process_group("gloo" if args.dry_run else "nccl")
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
