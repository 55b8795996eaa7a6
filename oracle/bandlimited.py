"""Band-limited reference of the spectral method, step by step (TEST INFRASTRUCTURE ONLY).

This is the paper's Fourier route written out with direct sums, no FFT, no
NUFFT, no blocking, fp64 (numpy):

1. Knot density transform (eq_rhoPhat):
       rho_hat_P(w) = sum_i c_i exp(-2 pi i w . x_i)
   with each ball's own kernel transform multiplied in (L276-L278, eq_fballhat:
   f_hat = rho_hat * f_hat_B0; with one radius per knot, eq_un L96 sums the
   per-ball products):
       f_hat_A(w) = sum_i w_i beta_hat(r_i, |w|) exp(-2 pi i w . a_i)
   beta_hat(r, rho) = 4 pi (sin kr - kr cos kr) / k^3, k = 2 pi rho: the CFT
   (L796-L799, eq_CFT_int, frequency in cycles per length) of the indicator of
   B(0, r).  The paper leaves the kernel transform implicit ("precomputed to
   full precision", L531); this is the textbook closed form, pinned in tests.
2. Rotation by relocating the knots (L235-L257, eq_Mink0/eq_rhoAtrans):
   b_j -> R b_j, radii unchanged.
3. Fourier correlation (L398-L404, eq_ccghat):
       g_hat(w) = f_hat_A(w) * f_hat_RB(-w)
   (= f_hat_A conj(f_hat_RB) for real weights; reading C-3 for complex ones).
4. Inverse transform restricted to a band of modes k (w = k / P) on the
   P-periodic lattice (DFT as a Riemann sum of the CFT, L829-L833):
       f~(t_m) = (1/P^3) sum_{k in band} g_hat(k/P) exp(+2 pi i k . t_m / P)

The band is a symmetric cube |k_i| <= K (reading C-13: Nyquist planes
excluded, so the result is exactly real for real weights), optionally
intersected with the ball |k| <= K_sphere.
"""
from __future__ import annotations

import numpy as np


def ball_transform(r, rho):
    """beta_hat(r, rho): CFT of 1{|x| <= r} at spatial frequency |w| = rho (cycles/length).

    Closed form 4 pi (sin x - x cos x) / k^3 with k = 2 pi rho, x = k r; below
    x = 0.1 the Taylor series (4 pi r^3) sum_n (-1)^n 3 x^{2n} / ((2n+3) (2n+1)!)
    ... written as r^3 * 4 pi * (1/3 - x^2/30 + x^4/840 - x^6/45360 + x^8/3991680)
    avoids the fp64 cancellation of the closed form.
    """
    r = np.asarray(r, dtype=np.float64)
    rho = np.asarray(rho, dtype=np.float64)
    k = 2.0 * np.pi * rho
    x = k * r
    small = np.abs(x) < 0.1
    xs = np.where(small, x, 0.0)
    x2 = xs * xs
    series = 4.0 * np.pi * r ** 3 * (1.0 / 3.0 - x2 / 30.0 + x2 ** 2 / 840.0
                                     - x2 ** 3 / 45360.0 + x2 ** 4 / 3991680.0)
    kk = np.where(small, 1.0, k)
    xx = np.where(small, 1.0, x)
    closed = 4.0 * np.pi * (np.sin(xx) - xx * np.cos(xx)) / kk ** 3
    return np.where(small, series, closed)


def band_modes(K: int, K_sphere: float | None = None):
    """Integer mode vectors of the band as three broadcastable 1D axes + mask."""
    k = np.arange(-K, K + 1)
    kx, ky, kz = np.meshgrid(k, k, k, indexing="ij")
    mask = np.ones(kx.shape, dtype=bool)
    if K_sphere is not None:
        mask = kx * kx + ky * ky + kz * kz <= K_sphere * K_sphere
    return k, mask


def ndft_density(xyzr, w, P: float, K: int, sign: float = -1.0):
    """f_hat(k/P) = sum_j w_j beta_hat(r_j, |k|/P) exp(sign 2 pi i k . x_j / P) on the
    cube band |k_i| <= K (returned as a (2K+1)^3 complex array, index k + K)."""
    xyzr = np.asarray(xyzr, dtype=np.float64)
    w = np.ones(len(xyzr)) if w is None else np.asarray(w)
    k = np.arange(-K, K + 1, dtype=np.float64)
    rho = np.sqrt(k[:, None, None] ** 2 + k[None, :, None] ** 2 + k[None, None, :] ** 2) / P
    out = np.zeros((2 * K + 1,) * 3, dtype=np.complex128)
    for j in range(len(xyzr)):
        x, y, z, r = xyzr[j]
        ex = np.exp(sign * 2j * np.pi * k * x / P)
        ey = np.exp(sign * 2j * np.pi * k * y / P)
        ez = np.exp(sign * 2j * np.pi * k * z / P)
        out += w[j] * ball_transform(r, rho) * (ex[:, None, None] * ey[None, :, None] * ez[None, None, :])
    return out


def bandlimited_correlation(A, wA, B, wB, R, N: int, h: float, t0, P: float, K: int,
                            K_sphere: float | None = None):
    """f~_R(t_m) on the N^3 grid t_m = t0 + m h for the band |k_i| <= K (and |k| <= K_sphere).

    Returns float64 (real weights) or complex128 (complex weights), shape (N, N, N).
    """
    R = np.asarray(R, dtype=np.float64).reshape(3, 3)
    B = np.asarray(B, dtype=np.float64)
    RB = np.column_stack([B[:, :3] @ R.T, B[:, 3]])          # step 2: b_j -> R b_j
    fA = ndft_density(A, wA, P, K, sign=-1.0)                   # f_hat_A(+k/P)
    fB_neg = ndft_density(RB, wB, P, K, sign=+1.0)              # f_hat_RB(-k/P)
    g = fA * fB_neg                                             # step 3
    _, mask = band_modes(K, K_sphere)
    g = np.where(mask, g, 0.0)
    k = np.arange(-K, K + 1, dtype=np.float64)
    out = None
    for ax in range(3):                                         # step 4, axis by axis
        t = t0[ax] + h * np.arange(N)
        E = np.exp(2j * np.pi * np.outer(k, t) / P)             # (2K+1, N)
        g = np.tensordot(g, E, axes=([0], [0]))                 # contracts the leading k axis
    out = g / P ** 3
    complex_w = np.iscomplexobj(wA) or np.iscomplexobj(wB)
    return out if complex_w else out.real
