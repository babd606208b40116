"""Exact references and the DoS reconstruction, numpy/scipy (O4-O7).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Each function cites the
passage it writes out.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np


def exact_moments_from_eigs(lam, a: float, b: float, N: int, chunk: int = 1 << 16) -> np.ndarray:
    """Eq (13): mu_n = (1/D) sum_k T_n(E~_k), E~_k = (E_k - b)/a (Eq 8),
    with T_n(x) = cos(n arccos x) (Eq 3).  x is clipped to [-1, 1] against rounding."""
    lam = np.asarray(lam, dtype=np.float64).ravel()
    x = np.clip((lam - b) / a, -1.0, 1.0)
    th = np.arccos(x)
    n = np.arange(N, dtype=np.float64)
    acc = np.zeros(N, dtype=np.float64)
    for s in range(0, len(th), chunk):
        acc += np.cos(np.outer(n, th[s:s + chunk])).sum(axis=1)
    return acc / len(lam)


def exact_moments_dense(H, a: float, b: float, N: int) -> np.ndarray:
    """O4: exact trace of T_n(H~) from dense diagonalisation of a tiny H (CSR or array)."""
    Hd = H.dense() if hasattr(H, "dense") else np.asarray(H)
    return exact_moments_from_eigs(np.linalg.eigvalsh(Hd), a, b, N)


def lattice_spectrum(ndim: int, L, t: float) -> np.ndarray:
    """O5: spectrum of the clean periodic nearest-neighbour lattice:
    plane waves give E(k) = 2 t sum_d cos(2 pi k_d / L_d), k_d = 0..L_d-1."""
    E = np.zeros(1)
    for d in range(ndim):
        e = 2.0 * t * np.cos(2.0 * np.pi * np.arange(L[d]) / L[d])
        E = (E[:, None] + e[None, :]).ravel()
    return E


def harper_spectrum(L0: int, L1: int, t: float, flux: float) -> np.ndarray:
    """O5 (Peierls): exact spectrum of the 2D lattice whose y-bond (x,y)->(x,y+1)
    carries t e^{i 2 pi flux x} (reading X15).  With flux = p/q and plane waves
    e^{i k_y y} e^{i k_x q X} (x = q X + s) H splits into L1 * L0/q Hermitian q x q
    blocks: M_ss = 2t cos(2 pi flux s - k_y), M_{s,s+-1} = t, corner terms
    t e^{+-i k_x q}.  k_y = 2 pi m / L1, k_x = 2 pi j / L0, j < L0/q."""
    fr = Fraction(flux).limit_denominator(1 << 20)
    q = fr.denominator
    assert L0 % q == 0, "flux * L0 must be an integer"
    out = []
    s = np.arange(q)
    for m in range(L1):
        ky = 2.0 * np.pi * m / L1
        for j in range(L0 // q):
            kx = 2.0 * np.pi * j / L0
            M = np.zeros((q, q), dtype=np.complex128)
            M[s, s] += 2.0 * t * np.cos(2.0 * np.pi * float(fr) * s - ky)
            for u in range(q):
                v = u + 1
                if v < q:
                    M[u, v] += t
                    M[v, u] += t
                else:  # bond from cell X to X+1: psi(x + q) = e^{i kx q} psi(x)
                    M[u, 0] += t * np.exp(1j * kx * q)
                    M[0, u] += t * np.exp(-1j * kx * q)
            out.append(np.linalg.eigvalsh(M))
    return np.concatenate(out)


def jackson(N: int) -> np.ndarray:
    """Jackson kernel g_n, n = 0..N-1 (named at PAPER.md:25, formula from the paper's
    ref [10], Weisse et al. RMP 78, 275; reading X8):
    g_n = [(N-n+1) cos(pi n/(N+1)) + sin(pi n/(N+1)) cot(pi/(N+1))] / (N+1)."""
    n = np.arange(N, dtype=np.float64)
    q = np.pi / (N + 1)
    return ((N - n + 1) * np.cos(q * n) + np.sin(q * n) / np.tan(q)) / (N + 1)


def kernel_coeffs(N: int, kind: str = "jackson", lam: float = 4.0) -> np.ndarray:
    """Damping factors g_n, n = 0..N-1, of Eq (6) ("a kernel which satisfies the
    limit" Eq 7).  The paper names the Jackson kernel; the others
    are the standard ones of its ref [10] (Weisse et al., RMP 78, 275):
      jackson  reading X8 (jackson() above)
      lorentz  g_n = sinh(lam (1 - n/N)) / sinh(lam)      (for Green's functions; lam ~ 3-5)
      fejer    g_n = 1 - n/N                               (Cesaro mean of the partial sums)
      none     g_n = 1                                     (Dirichlet: truncated series, Eq 1)"""
    n = np.arange(N, dtype=np.float64)
    if kind == "jackson":
        return jackson(N)
    if kind == "lorentz":
        return np.sinh(lam * (1.0 - n / N)) / np.sinh(lam)
    if kind == "fejer":
        return 1.0 - n / N
    if kind == "none":
        return np.ones(N)
    raise ValueError(kind)


def green(mu, a: float, b: float, omega, kernel: str = "jackson", lam: float = 4.0) -> np.ndarray:
    """Retarded Green's function G(omega) = (1/D) Tr 1/(omega + i0 - H) from the damped
    moments (the paper's "Green's functions"; expansion of ref [10]), reading
    X24: with x = (omega - b)/a, c_0 = g_0 mu_0, c_n = 2 g_n mu_n and
      |x| < 1:  G~(x) = -i sum_n c_n e^{-i n theta} / sin(theta),  theta = arccos x
      |x| > 1:  G~(x) = sum_n c_n t^n / (sgn(x) sqrt(x^2 - 1)),     t = x - sgn(x) sqrt(x^2 - 1)
    (both from 1/(z - y) = sum_n (2 - delta_n0) T_n(y) t^n / sqrt(z^2 - 1), t = z - sqrt(z^2-1));
    G(omega) = G~(x) / a.  |x| = 1 is singular: NaN."""
    mu = np.asarray(mu, dtype=np.float64)
    N = len(mu)
    c = kernel_coeffs(N, kernel, lam) * mu
    c[1:] *= 2.0
    x = (np.asarray(omega, dtype=np.float64) - b) / a
    out = np.full(x.shape, np.nan + 1j * np.nan, dtype=np.complex128)
    n = np.arange(N, dtype=np.float64)
    ins = np.abs(x) < 1.0
    th = np.arccos(x[ins])
    out[ins] = -1j * (np.exp(-1j * np.outer(th, n)) @ c) / np.sin(th)
    outs = np.abs(x) > 1.0
    xo = x[outs]
    sg = np.sign(xo)
    sq = np.sqrt(xo * xo - 1.0)
    t = xo - sg * sq
    out[outs] = (np.power.outer(t, n) @ c) / (sg * sq)
    return out / a


def green_closed_1d(E, t: float = -1.0) -> np.ndarray:
    """O7: Green's function of the infinite 1D chain, G(E + i0) = 1/sqrt((E+i0)^2 - 4t^2):
    -i/sqrt(4t^2 - E^2) inside the band, 1/(sgn(E) sqrt(E^2 - 4t^2)) outside."""
    E = np.asarray(E, dtype=np.float64)
    w = 2 * abs(t)
    out = np.empty(E.shape, dtype=np.complex128)
    ins = np.abs(E) < w
    out[ins] = -1j / np.sqrt(w * w - E[ins] ** 2)
    out[~ins] = 1.0 / (np.sign(E[~ins]) * np.sqrt(E[~ins] ** 2 - w * w))
    return out


def moment_stats(mu_pv):
    """Error bars of the stochastic trace (Eq 16: mu_n is the average over
    R random vectors; reading X28).  mu_pv[r][n] = the moment from vector r alone.
    Returns (mean_n, sem_n): the sample mean over r and its standard error
    sqrt(sum_r (mu_n^(r) - mean_n)^2 / ((R - 1) R)); sem = NaN for R = 1."""
    pv = np.asarray(mu_pv, dtype=np.float64)
    R = pv.shape[0]
    mean = pv.sum(axis=0) / R
    if R < 2:
        return mean, np.full(pv.shape[1], np.nan)
    dev = pv - mean[None, :]
    return mean, np.sqrt((dev * dev).sum(axis=0) / ((R - 1) * R))


def chebyshev_nodes(K: int) -> np.ndarray:
    """x_k = cos(pi (k + 1/2) / K), k = 0..K-1 (reading X7)."""
    return np.cos(np.pi * (np.arange(K) + 0.5) / K)


def dos(mu, a: float, b: float, omega, kernel: str = "jackson", lam: float = 4.0) -> np.ndarray:
    """Eq (6), mapped back to omega (Eq 11-12; reading X9):
    rho(omega) = [g_0 mu_0 + 2 sum_{n=1}^{N-1} g_n mu_n T_n(x)] / (pi sqrt(1-x^2)) / a,
    x = (omega - b)/a; rho = 0 for |x| >= 1 (reading X7)."""
    mu = np.asarray(mu, dtype=np.float64)
    N = len(mu)
    g = kernel_coeffs(N, kernel, lam)
    x = (np.asarray(omega, dtype=np.float64) - b) / a
    out = np.zeros_like(x)
    inside = np.abs(x) < 1.0
    xi = x[inside]
    c = g * mu
    c[1:] *= 2.0
    T = np.cos(np.outer(np.arccos(xi), np.arange(N)))  # T_n(x) = cos(n arccos x), Eq (3)
    out[inside] = (T @ c) / (np.pi * np.sqrt(1.0 - xi * xi)) / a
    return out


def dos_closed_1d(E, t: float = -1.0) -> np.ndarray:
    """O7: DoS of the infinite 1D chain, rho(E) = 1/(pi sqrt(4t^2 - E^2)), |E| < 2|t|."""
    E = np.asarray(E, dtype=np.float64)
    out = np.zeros_like(E)
    m = np.abs(E) < 2 * abs(t)
    out[m] = 1.0 / (np.pi * np.sqrt(4 * t * t - E[m] ** 2))
    return out


def dos_closed_2d(E, t: float = -1.0) -> np.ndarray:
    """O7: DoS of the infinite square lattice, rho(E) = K(1 - E^2/16t^2) / (2 pi^2 |t|),
    |E| < 4|t| (K the complete elliptic integral of the first kind, parameter m = k^2)."""
    from scipy.special import ellipk
    E = np.asarray(E, dtype=np.float64)
    out = np.zeros_like(E)
    m = (np.abs(E) < 4 * abs(t)) & (E != 0)
    out[m] = ellipk(1.0 - E[m] ** 2 / (16 * t * t)) / (2 * np.pi ** 2 * abs(t))
    out[E == 0] = np.inf
    return out
