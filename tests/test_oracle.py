"""Pins for oracle/ (CPU only): the oracle is checked against things other than itself.

* V(r, s, d) against an independent 1D quadrature of coaxial disc
  cross-sections, Monte Carlo, the spherical-cap tangency limit and the
  Fubini mass identity int V d^3x = vol_r vol_s.
* The pair sum against brute force without pruning, swap symmetry, rotation
  covariance, bilinearity in complex weights, the grid total-mass identity and
  the SPEC worked obstacle/collide examples (tests/golden/).
* The band-limited reference against the DC identity, the single-ball case,
  Hermitian symmetry, the radial inverse transform of beta_r beta_s (= V) and
  convergence to the lens oracle.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy import integrate

from synth import random_small_case, random_rotations

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def vol(r):
    return 4.0 / 3.0 * math.pi * r ** 3


def lens_by_discs(r, s, d):
    """Independent V: integrate the area of the intersection of the two coaxial
    cross-section discs, pi * min(r^2 - z^2, s^2 - (z - d)^2)_+, along the axis."""
    lo, hi = max(-r, d - s), min(r, d + s)
    if hi <= lo:
        return 0.0
    f = lambda z: math.pi * max(0.0, min(r * r - z * z, s * s - (z - d) ** 2))
    # the integrand has a kink where the two discs have equal radius
    zc = (r * r - s * s + d * d) / (2 * d) if d > 0 else None
    pts = [zc] if zc is not None and lo < zc < hi else None
    val, _ = integrate.quad(f, lo, hi, points=pts, epsabs=1e-15, epsrel=1e-12, limit=200)
    return val


# ------------------------------------------------------------------ V(r,s,d)

@pytest.mark.parametrize("r,s", [(1.0, 1.0), (0.05, 0.15), (0.3, 0.1), (1.2, 3.2), (0.02, 0.02)])
def test_lens_matches_disc_quadrature(oracle_mod, r, s):
    for frac in np.linspace(0.0, 1.05, 23):
        d = frac * (r + s)
        v = oracle_mod.lens_volume(r, s, d)
        ref = lens_by_discs(r, s, d) if d > 0 else vol(min(r, s))
        assert abs(v - ref) <= 1e-10 * vol(min(r, s)) + 1e-14, (r, s, d, v, ref)


def test_lens_special_cases(oracle_mod):
    r, s = 0.3, 0.1
    assert oracle_mod.lens_volume(r, s, r + s) == 0.0
    assert oracle_mod.lens_volume(r, s, 2.0) == 0.0
    plateau = vol(min(r, s))
    for d in (0.0, 0.05, 0.2 - 1e-12):
        assert oracle_mod.lens_volume(r, s, d) == pytest.approx(plateau, rel=1e-12)
    # continuity at both knots |r-s| and r+s
    eps = 1e-9
    assert oracle_mod.lens_volume(r, s, r - s + eps) == pytest.approx(plateau, rel=1e-7)
    assert oracle_mod.lens_volume(r, s, r + s - eps) < 1e-15
    # symmetric in r, s
    assert oracle_mod.lens_volume(r, s, 0.33) == pytest.approx(oracle_mod.lens_volume(s, r, 0.33), rel=1e-14)


@pytest.mark.parametrize("r,s", [(1.0, 1.0), (0.3, 0.1), (1.5, 3.1)])
def test_lens_tangency_limit(oracle_mod, r, s):
    """Two thin spherical caps of heights eps*s/(r+s), eps*r/(r+s): V ~ pi r s eps^2 / (r+s)."""
    for eps in (1e-3, 1e-4):
        v = oracle_mod.lens_volume(r, s, r + s - eps)
        assert v / eps ** 2 == pytest.approx(math.pi * r * s / (r + s), rel=5 * eps / min(r, s))


@pytest.mark.parametrize("r,s", [(1.0, 1.0), (0.05, 0.15), (0.7, 0.2)])
def test_lens_mass_identity(oracle_mod, r, s):
    """Fubini: int_{R^3} (1_{B_r} * 1_{B_s})(t) dt = vol(B_r) vol(B_s)."""
    f = lambda d: 4 * math.pi * d * d * oracle_mod.lens_volume(r, s, d)
    val, _ = integrate.quad(f, 0.0, r + s, points=[abs(r - s)], epsabs=0, epsrel=1e-13, limit=200)
    assert val == pytest.approx(vol(r) * vol(s), rel=1e-11)


def test_lens_monte_carlo(oracle_mod):
    rng = np.random.default_rng(7)
    r, s, d = 0.1, 0.15, 0.18
    n = 2_000_000
    p = rng.uniform(-r, r, size=(n, 3))
    inside_r = np.einsum("ij,ij->i", p, p) <= r * r
    q = p - np.array([d, 0, 0])
    inside_both = inside_r & (np.einsum("ij,ij->i", q, q) <= s * s)
    frac = inside_both.mean()
    est = frac * (2 * r) ** 3
    sigma = math.sqrt(frac * (1 - frac) / n) * (2 * r) ** 3
    assert abs(est - oracle_mod.lens_volume(r, s, d)) < 5 * sigma


# ------------------------------------------------------------------ pair sums

def _case(seed, **kw):
    return random_small_case(seed, **kw)


def test_grid_equals_bruteforce_points(oracle_mod):
    for seed, cplx in ((1, False), (2, True)):
        w = _case(seed, complex_weights=cplx)
        for r in range(w.n_rot):
            f = oracle_mod.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[r], w.N, w.h, w.t0)
            idx = np.arange(w.N ** 3)
            fp = oracle_mod.correlate_points(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[r], w.N, w.h, w.t0, idx)
            assert np.abs(f.reshape(-1) - fp).max() <= 1e-14 * max(1.0, np.abs(fp).max())
            assert np.abs(fp).max() > 0


def test_grid_subbox(oracle_mod):
    w = _case(3)
    full = oracle_mod.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[0], w.N, w.h, w.t0)
    lo, hi = (2, 3, 1), (9, 7, 11)
    sub = oracle_mod.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[0], w.N, w.h, w.t0, lo, hi)
    s = tuple(slice(a, b) for a, b in zip(lo, hi))
    assert np.array_equal(sub[s], full[s])
    mask = np.ones_like(full, dtype=bool)
    mask[s] = False
    assert np.all(sub[mask] == 0)


def test_single_pair_is_lens_volume(oracle_mod):
    A = np.array([[0.1, -0.05, 0.02, 0.3]])
    B = np.array([[-0.2, 0.1, 0.05, 0.2]])
    R = random_rotations(np.random.default_rng(5), 1)[0]
    N, h, t0 = 10, 0.2, (-1.0, -1.0, -1.0)
    f = oracle_mod.correlate_grid(A, None, B, None, R, N, h, t0)
    c = A[0, :3] - R @ B[0, :3]
    for m in [(5, 5, 5), (6, 4, 5), (5, 6, 6), (3, 5, 5), (7, 7, 7)]:
        t = np.array(t0) + h * np.array(m)
        d = np.linalg.norm(c - t)
        assert f[m] == pytest.approx(lens_by_discs(0.3, 0.2, d) if d > 0 else vol(0.2), abs=1e-12)


def test_swap_symmetry(oracle_mod):
    """f_{A,RB}(t) = f_{RB,A}(-t); on t0=-1, h=2/N grids -t_m = t_{N-m}."""
    w = _case(4, complex_weights=True)
    R = w.R[0]
    RB = np.column_stack([w.B_xyzr[:, :3] @ R.T, w.B_xyzr[:, 3]])
    f1 = oracle_mod.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, R, w.N, w.h, w.t0)
    f2 = oracle_mod.correlate_grid(RB, w.B_w, w.A_xyzr, w.A_w, np.eye(3), w.N, w.h, w.t0)
    f2m = f2[::-1, ::-1, ::-1]
    f2m = np.roll(f2m, 1, axis=(0, 1, 2))  # index m -> N - m
    assert np.abs(f1[1:, 1:, 1:] - f2m[1:, 1:, 1:]).max() <= 1e-13 * np.abs(f1).max()
    assert np.abs(f1).max() > 0


def test_rotation_covariance(oracle_mod):
    """f_{A,RB}(t) = f_{Q A, Q R B}(Q t) for any rotation Q (isometry)."""
    w = _case(5)
    rng = np.random.default_rng(11)
    Q = random_rotations(rng, 1)[0]
    QA = np.column_stack([w.A_xyzr[:, :3] @ Q.T, w.A_xyzr[:, 3]])
    for _ in range(20):
        t = rng.uniform(-0.5, 0.5, size=3)
        f1 = oracle_mod.correlate_points(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[0], 1, 1.0, t, [0])
        f2 = oracle_mod.correlate_points(QA, w.A_w, w.B_xyzr, w.B_w, Q @ w.R[0], 1, 1.0, Q @ t, [0])
        assert f1[0] == pytest.approx(f2[0], rel=1e-12, abs=1e-16)


def test_complex_bilinearity(oracle_mod):
    w = _case(6, complex_weights=True)
    args = (w.R[1], w.N, w.h, w.t0)
    fc = oracle_mod.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, *args)
    a, b = w.A_w.real, w.A_w.imag
    c, d = w.B_w.real, w.B_w.imag
    g = lambda x, y: oracle_mod.correlate_grid(w.A_xyzr, x, w.B_xyzr, y, *args)
    ref = (g(a, c) - g(b, d)) + 1j * (g(a, d) + g(b, c))  # (a+ib)(c+id), no conjugation (reading C-3)
    assert np.abs(fc - ref).max() <= 1e-13 * np.abs(ref).max()


def test_grid_total_mass(oracle_mod):
    """sum_t f(t) h^3 -> (sum w vol_A)(sum v vol_B) on a grid covering the support."""
    w = random_small_case(8, n_a=4, n_b=3, N=48, r_lo=0.1, r_hi=0.2)
    f = oracle_mod.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[0], w.N, w.h, w.t0)
    mass = f.sum() * w.h ** 3
    ref = (w.A_w * vol(w.A_xyzr[:, 3])).sum() * (w.B_w * vol(w.B_xyzr[:, 3])).sum()
    assert mass == pytest.approx(ref, rel=2e-3)


def test_golden_obstacle_examples(oracle_mod):
    g = json.load(open(os.path.join(GOLDEN, "obstacle_examples.json")))
    Rz90 = np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]])
    for ex in g["obstacle_knots"]:
        R = np.eye(3) if ex["R"] == "I" else Rz90
        A, B = np.array([ex["a"]]), np.array([ex["b"]])
        c, rad = np.array(ex["obstacle_centre"], float), ex["obstacle_radius"]
        rng = np.random.default_rng(0)
        for _ in range(50):  # f(t) > 0 exactly inside the obstacle ball B(c, r1 + r2)
            t = c + rng.uniform(-1.2, 1.2, size=3) * rad
            dist = np.linalg.norm(t - c)
            if abs(dist - rad) < 1e-3:
                continue
            f = oracle_mod.correlate_points(A, None, B, None, R, 1, 1.0, t, [0])[0]
            assert (f > 0) == (dist < rad), (ex["cite"], t, f)
    for ex in g["collide"]:
        A = np.array([[0.0, 0.0, 0.0, ex["r"]]])
        B = np.array([[0.0, 0.0, 0.0, ex["s"]]])
        # B translated by t = (d, 0, 0): the relative configuration (I, t)
        f = oracle_mod.correlate_points(A, None, B, None, np.eye(3), 1, 1.0, (ex["d"], 0.0, 0.0), [0])[0]
        assert (f > 0) == ex["collides"], ex["cite"]


# ------------------------------------------------------------------ band-limited reference

def test_ball_transform_quadrature(oracle_mod):
    """beta_hat(r, rho) = int_0^r 4 pi x^2 sinc(2 pi rho x) dx (radial CFT of the indicator)."""
    for r in (0.005, 0.1, 1.7):
        for rho in (0.0, 1e-4 / r, 0.01 / r, 0.3 / r, 2.0 / r, 7.3 / r):
            k = 2 * math.pi * rho
            f = (lambda x: 4 * math.pi * x * x * (math.sin(k * x) / (k * x) if k * x > 0 else 1.0))
            ref, _ = integrate.quad(f, 0, r, epsabs=0, epsrel=1e-12, limit=400)
            got = float(oracle_mod.ball_transform(r, rho))
            assert got == pytest.approx(ref, rel=1e-10, abs=1e-14 * vol(r)), (r, rho)


def test_radial_inverse_of_kernel_product_is_lens(oracle_mod):
    """V(r,s,d) = int_0^inf 4 pi rho^2 beta_r(rho) beta_s(rho) sinc(2 pi rho d) d rho (convolution theorem, L816-L826)."""
    r, s = 0.1, 0.07
    for d in (0.0, 0.02, 0.05, 0.1, 0.16):
        def f(rho):
            k = 2 * math.pi * rho
            sinc = math.sin(k * d) / (k * d) if k * d > 0 else 1.0
            return 4 * math.pi * rho * rho * float(oracle_mod.ball_transform(r, rho)) * \
                float(oracle_mod.ball_transform(s, rho)) * sinc
        val, _ = integrate.quad(f, 0, 4000.0, limit=20000, epsabs=1e-16, epsrel=1e-10)
        assert val == pytest.approx(oracle_mod.lens_volume(r, s, d), abs=3e-5 * vol(s))


def test_ndft_single_ball_and_hermitian(oracle_mod):
    P, K = 2.0, 6
    one = oracle_mod.ndft_density(np.array([[0, 0, 0, 0.3]]), None, P, K)
    k = np.arange(-K, K + 1)
    rho = np.sqrt(k[:, None, None] ** 2 + k[None, :, None] ** 2 + k[None, None, :] ** 2) / P
    assert np.abs(one - oracle_mod.ball_transform(0.3, rho)).max() < 1e-14
    w = random_small_case(9)
    F = oracle_mod.ndft_density(w.A_xyzr, w.A_w, P, K)
    assert np.abs(F - np.conj(F[::-1, ::-1, ::-1])).max() < 1e-13 * np.abs(F).max()
    # shift theorem: moving every knot by x0 multiplies by exp(-2 pi i k.x0/P)
    x0 = np.array([0.13, -0.07, 0.21])
    Fs = oracle_mod.ndft_density(w.A_xyzr + np.r_[x0, 0.0], w.A_w, P, K)
    ph = np.exp(-2j * np.pi * (k[:, None, None] * x0[0] + k[None, :, None] * x0[1] + k[None, None, :] * x0[2]) / P)
    assert np.abs(Fs - F * ph).max() < 1e-12 * np.abs(F).max()


def test_bandlimited_dc_identity(oracle_mod):
    """K = 0 keeps only g_hat(0) = (sum w vol_A)(sum v vol_B): f~ is the constant g_hat(0)/P^3."""
    w = random_small_case(10)
    P = 2.5
    f0 = oracle_mod.bandlimited_correlation(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[0], 6, w.h, w.t0, P, 0)
    ref = (w.A_w * vol(w.A_xyzr[:, 3])).sum() * (w.B_w * vol(w.B_xyzr[:, 3])).sum() / P ** 3
    assert np.allclose(f0, ref, rtol=1e-13)


def test_bandlimited_converges_to_lens(oracle_mod):
    w = random_small_case(12, n_a=3, n_b=3, N=16, r_lo=0.15, r_hi=0.3)
    f = oracle_mod.correlate_grid(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[0], w.N, w.h, w.t0)
    errs = []
    for K in (8, 16, 32):
        fb = oracle_mod.bandlimited_correlation(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[0],
                                                w.N, w.h, w.t0, 2.5, K)
        errs.append(np.abs(fb - f).max() / np.abs(f).max())
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 3e-3


# ------------------------------------------------------------------ spherical band (K_sphere)
# bandlimited_correlation(K_sphere=rho) keeps the modes |k_i| <= K with |k| <= rho (the
# truncated Fourier sum of the single-configuration query orders its modes by |k|,
# PAPER.md L432-L439 "spiral traversal ... starting from the dominant modes").

def test_sphere_band_covering_the_cube_is_the_cube(oracle_mod):
    """rho >= sqrt(3) K keeps every cube mode: the result is bitwise the cube band's."""
    w = random_small_case(21, n_a=4, n_b=3, N=8)
    args = (w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[0], w.N, w.h, w.t0, 2.5, 5)
    cube = oracle_mod.bandlimited_correlation(*args)
    sph = oracle_mod.bandlimited_correlation(*args, K_sphere=math.sqrt(3) * 5 + 1e-9)
    assert np.array_equal(cube, sph)
    # and one just inside the corner drops the 8 corner modes: a different result
    sph2 = oracle_mod.bandlimited_correlation(*args, K_sphere=math.sqrt(3) * 5 - 1e-6)
    assert np.abs(sph2 - cube).max() > 1e-6 * np.abs(cube).max()


def test_sphere_band_dc_and_seven_mode_closed_form(oracle_mod):
    """rho < 1 keeps only k = 0: f~ = g_hat(0) / P^3 = (sum w vol_A)(sum v vol_B) / P^3.
    rho = 1 keeps k = 0 and the six unit vectors +-e_i: for real weights
    f~(t) = (1/P^3) [g_0 + 2 sum_i Re(g(e_i) exp(2 pi i t_i / P))] with
    g(e_i) = fA(e_i) conj(fB(e_i)) of the NDFT (pinned above)."""
    w = random_small_case(22, n_a=5, n_b=4, N=6)
    P = 2.5
    args = (w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[1], w.N, w.h, w.t0, P, 3)
    f0 = oracle_mod.bandlimited_correlation(*args, K_sphere=0.5)
    ref0 = (w.A_w * vol(w.A_xyzr[:, 3])).sum() * (w.B_w * vol(w.B_xyzr[:, 3])).sum() / P ** 3
    assert np.allclose(f0, ref0, rtol=1e-13, atol=0)
    f1 = oracle_mod.bandlimited_correlation(*args, K_sphere=1.0)
    RB = np.column_stack([w.B_xyzr[:, :3] @ w.R[1].T, w.B_xyzr[:, 3]])
    fA = oracle_mod.ndft_density(w.A_xyzr, w.A_w, P, 1)
    fB = oracle_mod.ndft_density(RB, w.B_w, P, 1)
    e = [(2, 1, 1), (1, 2, 1), (1, 1, 2)]  # index k + K of +e_x, +e_y, +e_z
    for m in [(0, 0, 0), (1, 4, 2), (5, 5, 5), (3, 0, 1)]:
        t = np.asarray(w.t0) + w.h * np.asarray(m)
        val = fA[1, 1, 1] * np.conj(fB[1, 1, 1])
        for i, ix in enumerate(e):
            val += 2 * (fA[ix] * np.conj(fB[ix]) * np.exp(2j * np.pi * t[i] / P)).real
        assert f1[m] == pytest.approx(val.real / P ** 3, rel=1e-12)


def test_sphere_band_parseval(oracle_mod):
    """Parseval on the full period lattice (N = Np points spanning P, Np > 2K so the band
    modes are orthogonal): sum_m |f~(t_m)|^2 h^3 = (1/P^3) sum_{|k_i|<=K, |k|<=rho} |g(k)|^2,
    with g(k) = fA(k) fB(-k) of the NDFT.  A wrong mask (|k| < rho, rho^2 vs rho, a missing
    octant) changes the right-hand side."""
    w = random_small_case(23, n_a=4, n_b=4, N=8, complex_weights=True)
    P, K, Np = 2.0, 6, 16
    h = P / Np
    RB = np.column_stack([w.B_xyzr[:, :3] @ w.R[0].T, w.B_xyzr[:, 3]])
    fA = oracle_mod.ndft_density(w.A_xyzr, w.A_w, P, K)
    fBn = oracle_mod.ndft_density(RB, w.B_w, P, K, sign=+1.0)   # fB(-k)
    g2 = np.abs(fA * fBn) ** 2
    k = np.arange(-K, K + 1)
    kk = k[:, None, None] ** 2 + k[None, :, None] ** 2 + k[None, None, :] ** 2
    for rho in (2.0, 3.5, 5.0, 7.9):
        f = oracle_mod.bandlimited_correlation(w.A_xyzr, w.A_w, w.B_xyzr, w.B_w, w.R[0], Np, h,
                                               (-1.0, -1.0, -1.0), P, K, K_sphere=rho)
        lhs = (np.abs(f) ** 2).sum() * h ** 3
        rhs = g2[kk <= rho * rho].sum() / P ** 3
        assert lhs == pytest.approx(rhs, rel=1e-11), rho
        # the retained mode count is the lattice-point count of the ball
        n_brute = sum(1 for a in k for b in k for c in k if a * a + b * b + c * c <= rho * rho)
        assert (kk <= rho * rho).sum() == n_brute
