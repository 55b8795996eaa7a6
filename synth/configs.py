"""The five BASELINE.json workloads as seeded synthetic arrays.

Readings of under-specified recipes (DESIGN.md §3 lists them with SURVEY
§8(c) numbering):

* C-11  seed 0 for every config, numpy PCG64 (`np.random.default_rng`);
        draw A, then B, then the rotations; within a shape centres, then radii.
        "uniform in a sphere of radius rho" = uniform in the solid ball (rejection).
* C-12  uniform SO(3) rotations by Shoemake's quaternion recipe, fp64.
* C-6   "unit cube" = [-0.5, 0.5)^3 (only a_i - b_j matters at R = I).
* C-7   torus: core circle radius 0.6 in z=0, theta ~ U[0, 2pi), jitter
        uniform in a ball of radius 0.05, r = 0.2 - 0.15 |j| / 0.05;
        B = same recipe (2,000 balls) with centres and radii scaled by 0.3.
* C-8   cube shell = [-0.4, 0.4]^3 minus (-0.3, 0.3)^3, by rejection.
* C-9   docking random walk: start at 0, step 1.5 u (u uniform on S^2),
        reflect at the walls of [-20, 20]^3, record every position,
        recentre on the centroid; radii from {1.2,1.5,1.6,1.7,1.8} A with
        p = {0.5,0.1,0.2,0.15,0.05}.
* C-4   docking weights: every atom gives a core ball B(c, r) with weight
        -15i and a skin ball B(c, r + 1.4) with weight +1.
* C-5   translation grids t_m = t0 + m h, m in [0, N)^3: [-1, 1)^3 for
        Tiny/Single/Torus/Sweep; [-64, 64)^3 A at h = 1 A for docking.
* C-2   rotations act about the origin of B's frame (x -> R x).

Arrays: `xyzr` is (n, 4) float64 rows (x, y, z, r); weights are float64
(real configs) or complex128 (docking).  Rotations are (n_rot, 3, 3) float64.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

CONFIG_NAMES = ("tiny", "single", "torus", "sweep", "docking")


@dataclass
class Workload:
    name: str
    A_xyzr: np.ndarray
    A_w: np.ndarray
    B_xyzr: np.ndarray
    B_w: np.ndarray
    R: np.ndarray
    N: int
    h: float
    t0: tuple
    precision: str  # "f64" | "f32"
    weights: str  # "real" | "complex"
    output: str  # "full" | "min_argmin" | "max_real"
    notes: dict = field(default_factory=dict)

    @property
    def n_rot(self) -> int:
        return int(self.R.shape[0])


# ----------------------------------------------------------------------------
# primitive samplers (input generation only)
# ----------------------------------------------------------------------------

def _uniform_in_ball(rng, n, radius):
    out = np.empty((0, 3))
    while out.shape[0] < n:
        p = rng.uniform(-radius, radius, size=(2 * n + 16, 3))
        p = p[np.einsum("ij,ij->i", p, p) <= radius * radius]
        out = np.concatenate([out, p], axis=0)
    return out[:n]


def _uniform_in_cube_shell(rng, n, outer_half, inner_half):
    out = np.empty((0, 3))
    while out.shape[0] < n:
        p = rng.uniform(-outer_half, outer_half, size=(2 * n + 16, 3))
        inside_inner = np.all(np.abs(p) < inner_half, axis=1)
        out = np.concatenate([out, p[~inside_inner]], axis=0)
    return out[:n]


def _unit_vectors(rng, n):
    v = rng.normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def random_rotations(rng, n):
    """Shoemake (1992) uniform quaternions -> rotation matrices (reading C-12)."""
    u1, u2, u3 = rng.uniform(size=(3, n))
    a = np.sqrt(1.0 - u1)
    b = np.sqrt(u1)
    qx = a * np.sin(2 * np.pi * u2)
    qy = a * np.cos(2 * np.pi * u2)
    qz = b * np.sin(2 * np.pi * u3)
    qw = b * np.cos(2 * np.pi * u3)
    R = np.empty((n, 3, 3))
    R[:, 0, 0] = 1 - 2 * (qy * qy + qz * qz)
    R[:, 0, 1] = 2 * (qx * qy - qz * qw)
    R[:, 0, 2] = 2 * (qx * qz + qy * qw)
    R[:, 1, 0] = 2 * (qx * qy + qz * qw)
    R[:, 1, 1] = 1 - 2 * (qx * qx + qz * qz)
    R[:, 1, 2] = 2 * (qy * qz - qx * qw)
    R[:, 2, 0] = 2 * (qx * qz - qy * qw)
    R[:, 2, 1] = 2 * (qy * qz + qx * qw)
    R[:, 2, 2] = 1 - 2 * (qx * qx + qy * qy)
    return R


def _torus_balls(rng, n, scale):
    theta = rng.uniform(0.0, 2 * np.pi, size=n)
    core = np.stack([0.6 * np.cos(theta), 0.6 * np.sin(theta), np.zeros(n)], axis=1)
    jit = _uniform_in_ball(rng, n, 0.05)
    centres = core + jit
    radii = 0.2 - 0.15 * np.linalg.norm(jit, axis=1) / 0.05
    return np.column_stack([centres * scale, radii * scale])


def _random_walk(rng, n, step=1.5, half_box=20.0):
    pos = np.zeros(3)
    out = np.empty((n, 3))
    dirs = _unit_vectors(rng, n)
    for k in range(n):
        pos = pos + step * dirs[k]
        for ax in range(3):  # reflect at the walls
            if pos[ax] > half_box:
                pos[ax] = 2 * half_box - pos[ax]
            elif pos[ax] < -half_box:
                pos[ax] = -2 * half_box - pos[ax]
        out[k] = pos
    return out - out.mean(axis=0)


_DOCK_RADII = np.array([1.2, 1.5, 1.6, 1.7, 1.8])
_DOCK_P = np.array([0.5, 0.1, 0.2, 0.15, 0.05])
DOCK_SKIN = 1.4
DOCK_CORE_WEIGHT = -15j
DOCK_SKIN_WEIGHT = 1.0 + 0j


def _docking_molecule(rng, n_atoms):
    centres = _random_walk(rng, n_atoms)
    radii = rng.choice(_DOCK_RADII, size=n_atoms, p=_DOCK_P)
    core = np.column_stack([centres, radii])
    skin = np.column_stack([centres, radii + DOCK_SKIN])
    xyzr = np.concatenate([core, skin], axis=0)
    w = np.concatenate([np.full(n_atoms, DOCK_CORE_WEIGHT), np.full(n_atoms, DOCK_SKIN_WEIGHT)])
    return xyzr, w.astype(np.complex128)


# ----------------------------------------------------------------------------
# the five configs
# ----------------------------------------------------------------------------

def make_config(name: str, seed: int = 0, n_rot: int | None = None) -> Workload:
    """Build one BASELINE.json config.  `n_rot` overrides the rotation count
    (rotations are drawn last, so the shapes do not depend on it)."""
    rng = np.random.default_rng(seed)
    if name == "tiny":
        ca = _uniform_in_ball(rng, 32, 0.5)
        ra = rng.uniform(0.05, 0.15, size=32)
        cb = _uniform_in_ball(rng, 32, 0.5)
        rb = rng.uniform(0.05, 0.15, size=32)
        R = np.eye(3)[None].repeat(n_rot or 1, axis=0)
        return Workload("tiny", np.column_stack([ca, ra]), np.ones(32),
                        np.column_stack([cb, rb]), np.ones(32), R,
                        N=32, h=2.0 / 32, t0=(-1.0, -1.0, -1.0),
                        precision="f64", weights="real", output="full")
    if name == "single":
        ca = rng.uniform(-0.5, 0.5, size=(1024, 3))
        ra = np.clip(rng.lognormal(np.log(0.03), 0.4, size=1024), 0.01, 0.1)
        cb = rng.uniform(-0.5, 0.5, size=(1024, 3))
        rb = np.clip(rng.lognormal(np.log(0.03), 0.4, size=1024), 0.01, 0.1)
        R = np.eye(3)[None].repeat(n_rot or 1, axis=0)
        return Workload("single", np.column_stack([ca, ra]), np.ones(1024),
                        np.column_stack([cb, rb]), np.ones(1024), R,
                        N=64, h=2.0 / 64, t0=(-1.0, -1.0, -1.0),
                        precision="f32", weights="real", output="full")
    if name == "torus":
        A = _torus_balls(rng, 10000, 1.0)
        B = _torus_balls(rng, 2000, 0.3)
        R = random_rotations(rng, n_rot or 64)
        return Workload("torus", A, np.ones(len(A)), B, np.ones(len(B)), R,
                        N=128, h=2.0 / 128, t0=(-1.0, -1.0, -1.0),
                        precision="f32", weights="real", output="full")
    if name == "sweep":
        ca = _uniform_in_cube_shell(rng, 50000, 0.4, 0.3)
        ra = rng.uniform(0.005, 0.03, size=50000)
        cb = _uniform_in_ball(rng, 5000, 0.2)
        rb = rng.uniform(0.005, 0.02, size=5000)
        R = random_rotations(rng, n_rot or 512)
        return Workload("sweep", np.column_stack([ca, ra]), np.ones(50000),
                        np.column_stack([cb, rb]), np.ones(5000), R,
                        N=256, h=2.0 / 256, t0=(-1.0, -1.0, -1.0),
                        precision="f32", weights="real", output="min_argmin")
    if name == "docking":
        A, wa = _docking_molecule(rng, 4000)
        B, wb = _docking_molecule(rng, 1500)
        R = random_rotations(rng, n_rot or 3600)
        return Workload("docking", A, wa, B, wb, R,
                        N=128, h=1.0, t0=(-64.0, -64.0, -64.0),
                        precision="f32", weights="complex", output="max_real")
    raise ValueError(f"unknown config {name!r}; expected one of {CONFIG_NAMES}")


def random_small_case(seed: int, n_a: int = 6, n_b: int = 5, n_rot: int = 2,
                      N: int = 12, complex_weights: bool = False,
                      r_lo: float = 0.08, r_hi: float = 0.25) -> Workload:
    """Small random case for brute-force / parity checks (fits the [-1,1)^3 grid)."""
    rng = np.random.default_rng(seed)
    ca = _uniform_in_ball(rng, n_a, 0.35)
    ra = rng.uniform(r_lo, r_hi, size=n_a)
    cb = _uniform_in_ball(rng, n_b, 0.3)
    rb = rng.uniform(r_lo, r_hi, size=n_b)
    if complex_weights:
        wa = rng.normal(size=n_a) + 1j * rng.normal(size=n_a)
        wb = rng.normal(size=n_b) + 1j * rng.normal(size=n_b)
    else:
        wa = rng.uniform(0.5, 2.0, size=n_a)
        wb = rng.uniform(0.5, 2.0, size=n_b)
    R = random_rotations(rng, n_rot)
    return Workload(f"small{seed}", np.column_stack([ca, ra]), wa,
                    np.column_stack([cb, rb]), wb, R,
                    N=N, h=2.0 / N, t0=(-1.0, -1.0, -1.0),
                    precision="f64", weights="complex" if complex_weights else "real",
                    output="full")
