"""Pins of the CPU oracle to what the paper and the mathematics fix (-m "not gpu").

Each test names the oracle function(s) it pins and the independent fact used:
closed forms, combinatorial moments (tests/golden/), library diagonalisation,
invariants, brute force.  A plausible mistake in the oracle (dropped term, wrong
sign of b, transposed phase, wrong neighbour index, off-by-one in the doubling
loop) fails at least one of them.
"""
import math
import os

import numpy as np
import pytest

import kpm_inputs as ki
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "lattice_moments.txt")


def golden_moments(ndim):
    rows = [l.split() for l in open(GOLDEN) if not l.startswith("#")]
    return np.array([float(m) for d, n, m in rows if int(d) == ndim])


def unit_vectors(D):
    """R = D vectors sqrt(D) e_i: the estimator then equals the exact trace (reading X2)."""
    return np.sqrt(D) * np.eye(D)


def lat(ndim, L, t=-1.0, onsite=None, flux=0.0):
    L = tuple(L) + (1,) * (3 - len(L))
    return dict(ndim=ndim, L=L, D=L[0] * L[1] * L[2], t=t, onsite=onsite, flux=flux)


# ---------------------------------------------------------------- O1: the lattice H
def test_paper_10cube_lattice_structure():
    """10x10x10 cubic lattice, H is 1000x1000, sparse, symmetric, every row has
    seven non-zero positions, the diagonal ones zero and the others -1 (periodic BCs, X12)."""
    H = oracle.lattice_csr(lat(3, (10, 10, 10), onsite=np.zeros(1000)))
    assert H.D == 1000
    assert np.all(np.diff(H.rowptr) == 7)
    Hd = H.dense()
    assert np.array_equal(Hd, Hd.T)
    assert np.all(np.diag(Hd) == 0.0)
    off = Hd[~np.eye(1000, dtype=bool)]
    assert set(np.unique(off)) == {0.0, -1.0}
    assert np.all((Hd == -1.0).sum(axis=1) == 6)


@pytest.mark.parametrize("ndim,L", [(1, (9,)), (1, (2,)), (2, (6, 5)), (2, (2, 7)), (3, (4, 3, 5))])
def test_csr_spectrum_equals_plane_wave_spectrum(ndim, L):
    """O1 vs O5: eigenvalues of the built H equal 2t sum_d cos(2 pi k_d/L_d) (plane waves)."""
    H = oracle.lattice_csr(lat(ndim, L, t=-1.3))
    ev = np.sort(np.linalg.eigvalsh(H.dense()))
    an = np.sort(oracle.lattice_spectrum(ndim, L, -1.3))
    assert ev.shape == an.shape
    assert np.abs(ev - an).max() < 1e-12


def test_lattice_spectrum_invariants():
    """O5 pinned by Tr H = 0 and Tr H^2 = D * 2 ndim t^2 (each site has 2 ndim bonds)."""
    for ndim, L in [(1, (7, 1, 1)), (2, (8, 6, 1)), (3, (5, 4, 3))]:
        E = oracle.lattice_spectrum(ndim, L, 0.7)
        D = int(np.prod(L))
        assert len(E) == D
        assert abs(E.sum()) < 1e-12 * D
        assert abs((E ** 2).sum() - D * 2 * ndim * 0.49) < 1e-10 * D


def test_peierls_uniform_flux_per_plaquette():
    """O1 Peierls phase (reading X15) pinned gauge-invariantly: the product of hoppings
    around every plaquette (x,y)->(x+1,y)->(x+1,y+1)->(x,y+1)->(x,y) is t^4 e^{i 2 pi phi}."""
    L0, L1, phi, t = 16, 8, 3 / 16, -1.0
    Hd = oracle.lattice_csr(lat(2, (L0, L1), t=t, flux=phi)).dense()
    assert np.abs(Hd - Hd.conj().T).max() == 0.0
    s = lambda x, y: (x % L0) + L0 * (y % L1)
    for x in range(L0):
        for y in range(L1):
            path = [s(x, y), s(x + 1, y), s(x + 1, y + 1), s(x, y + 1), s(x, y)]
            prod = np.prod([Hd[path[k + 1], path[k]] for k in range(4)])
            assert abs(prod - t ** 4 * np.exp(2j * np.pi * phi)) < 1e-13


@pytest.mark.parametrize("L,phi", [((16, 16), 1 / 8), ((24, 8), 1 / 8), ((16, 12), 1 / 4),
                                   ((16, 6), 1 / 2), ((12, 10), 0.0)])
def test_peierls_spectrum_equals_harper_blocks(L, phi):
    """O1 (complex H) vs O5 Harper q x q decomposition (independent derivation)."""
    Hd = oracle.lattice_csr(lat(2, L, flux=phi)).dense()
    ev = np.sort(np.linalg.eigvalsh(Hd))
    hp = np.sort(oracle.harper_spectrum(L[0], L[1], -1.0, phi))
    assert np.abs(ev - hp).max() < 1e-12


def test_harper_reduces_to_plane_waves_at_zero_flux_and_trace_h2():
    hp = np.sort(oracle.harper_spectrum(12, 10, -1.0, 0.0))
    assert np.abs(hp - np.sort(oracle.lattice_spectrum(2, (12, 10, 1), -1.0))).max() < 1e-12
    hp = oracle.harper_spectrum(32, 16, -1.0, 1 / 8)
    assert abs((hp ** 2).sum() - 4 * 32 * 16) < 1e-9  # Tr H^2 = 4 D t^2 for any flux


def test_anderson_diagonal():
    eps = ki.anderson_onsite(3, 64, 2.0)
    Hd = oracle.lattice_csr(lat(3, (4, 4, 4), onsite=eps)).dense()
    assert np.array_equal(np.diag(Hd), eps)


# ---------------------------------------------------------------- Gerschgorin (Eq 8-9)
def test_gershgorin_closed_forms_and_enclosure():
    for ndim, L in [(1, (16,)), (2, (8, 8)), (3, (4, 4, 4))]:
        a, b = oracle.gershgorin(oracle.lattice_csr(lat(ndim, L)))
        assert (a, b) == (2.0 * ndim, 0.0)
    eps = ki.anderson_onsite(5, 216, 2.0)
    a, b = oracle.gershgorin(oracle.lattice_csr(lat(3, (6, 6, 6), onsite=eps)))
    Eu, El = eps.max() + 6, eps.min() - 6
    assert abs(a - (Eu - El) / 2) < 1e-15 and abs(b - (Eu + El) / 2) < 1e-15
    rng = np.random.default_rng(0)
    for _ in range(5):
        A = rng.normal(size=(30, 30)) + 1j * rng.normal(size=(30, 30))
        A = A + A.conj().T + np.diag(rng.normal(size=30) * 5)
        a, b = oracle.gershgorin(oracle.csr_from_dense(A))
        ev = np.linalg.eigvalsh(A)
        assert ev.max() <= b + a + 1e-12 and ev.min() >= b - a - 1e-12


# ---------------------------------------------------------------- exact traces (Eq 13)
@pytest.mark.parametrize("ndim,L", [(1, (200,)), (2, (64, 64)), (3, (20, 20, 20))])
def test_exact_moments_match_closed_walk_golden(ndim, L):
    """O4/O5 pinned to tests/golden/lattice_moments.txt (pure combinatorics) for n < L."""
    g = golden_moments(ndim)
    n = min(len(g), min(L[:ndim]))
    mu = oracle.exact_moments_from_eigs(oracle.lattice_spectrum(ndim, L + (1,) * (3 - len(L)), -1.0),
                                        2.0 * ndim, 0.0, n)
    assert np.abs(mu - g[:n]).max() < 1e-13


def test_1d_chain_exact_moments_are_kronecker_delta():
    """Q3: periodic chain, a = 2, b = 0: mu_n = (1/D) sum_k cos(n 2 pi k / D) = delta_{n0} (n < D)."""
    mu = oracle.exact_moments_from_eigs(oracle.lattice_spectrum(1, (1024, 1, 1), -1.0), 2.0, 0.0, 128)
    assert mu[0] == 1.0
    assert np.abs(mu[1:]).max() < 1e-13


# ---------------------------------------------------------------- O2 / O3: the recursion
def _random_hermitian(D, seed, cplx):
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(D, D)) * (rng.random((D, D)) < 0.2)
    if cplx:
        A = A + 1j * rng.normal(size=(D, D)) * (rng.random((D, D)) < 0.2)
    A = A + A.conj().T + np.diag(rng.normal(size=D))
    return A


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("fn", [oracle.moments_direct, oracle.moments_doubling])
def test_unit_vectors_reproduce_exact_trace_random_H(fn, cplx):
    """Q2 on an arbitrary Hermitian H with a loose (a, b) and b != 0 (catches a wrong sign or
    a dropped shift in H~ = (H - b)/a): the estimator with R = D unit vectors is the trace."""
    A = _random_hermitian(40, 11 + cplx, cplx)
    ev = np.linalg.eigvalsh(A)
    a = 1.3 * (ev.max() - ev.min()) / 2
    b = (ev.max() + ev.min()) / 2 + 0.1 * a
    N = 37
    mu = fn(oracle.csr_from_dense(A), a, b, unit_vectors(40), N)
    assert np.abs(mu - oracle.exact_moments_from_eigs(ev, a, b, N)).max() < 1e-12


@pytest.mark.parametrize("case", ["1d", "2d", "3d_paper", "anderson", "peierls"])
def test_unit_vectors_reproduce_exact_trace_lattices(case):
    """Q2 on the lattices of the configs (small): estimator with R = D unit vectors equals the
    dense-diagonalisation trace; includes the paper's own 10x10x10 lattice."""
    if case == "1d":
        l, N = lat(1, (64,)), 64
    elif case == "2d":
        l, N = lat(2, (12, 10)), 80
    elif case == "3d_paper":
        l, N = lat(3, (10, 10, 10)), 256
    elif case == "anderson":
        l, N = lat(3, (5, 6, 4), onsite=ki.anderson_onsite(9, 120, 2.0)), 100
    else:
        l, N = lat(2, (16, 16), flux=1 / 8), 128
    H = oracle.lattice_csr(l)
    a, b = oracle.gershgorin(H)
    ex = oracle.exact_moments_dense(H, a, b, N)
    mu = oracle.moments_doubling(H, a, b, unit_vectors(H.D), N)
    assert np.abs(mu - ex).max() < 1e-12
    if case != "3d_paper":
        mud = oracle.moments_direct(H, a, b, unit_vectors(H.D), N)
        assert np.abs(mud - ex).max() < 1e-12


def test_unit_vectors_match_closed_walk_golden_2d_3d():
    """The whole chain (O1 CSR, H~, recursion, doubling, normalisation) against pure
    combinatorics: 2D 24x24 and 3D 10^3 (the paper's lattice) for n < L."""
    for ndim, L in [(2, (24, 24)), (3, (10, 10, 10))]:
        H = oracle.lattice_csr(lat(ndim, L))
        n = L[0]
        mu = oracle.moments_doubling(H, 2.0 * ndim, 0.0, unit_vectors(H.D), n)
        assert np.abs(mu - golden_moments(ndim)[:n]).max() < 1e-13


def test_c1_direct_equals_doubling_bitwise_and_mu0_exact():
    """Q1 + Q4: config c1 (t = -1, a = 2, +-1 vectors): every a_n has entries in {-1, 0, 1}, so
    any correct evaluation order gives identical bits; mu_0 = 1 exactly."""
    c = ki.CONFIGS["c1"]
    H = oracle.lattice_csr(ki.lattice(c))
    r = ki.rademacher(c["seed"], c["R"], 1024)
    m1 = oracle.moments_direct(H, 2.0, 0.0, r, c["N"])
    m2 = oracle.moments_doubling(H, 2.0, 0.0, r, c["N"])
    assert np.array_equal(m1, m2)
    assert m1[0] == 1.0
    # every moment is an integer multiple of 1/(D R) (sums of integer products)
    assert np.array_equal(np.round(m1 * 1024 * 8), m1 * 1024 * 8)


@pytest.mark.parametrize("N", list(range(1, 11)) + [31, 64])
def test_doubling_equals_direct_every_N(N):
    """Q10 and the odd-N tail (reading X11): doubling == direct for every N."""
    l = lat(2, (8, 8), onsite=ki.anderson_onsite(4, 64, 1.0))
    H = oracle.lattice_csr(l)
    a, b = oracle.gershgorin(H)
    r = ki.rademacher(3, 3, 64)
    m1, p1 = oracle.moments_direct(H, a, b, r, N, per_vector=True)
    m2, p2 = oracle.moments_doubling(H, a, b, r, N, per_vector=True)
    assert np.abs(m1 - m2).max() < 1e-14
    assert np.abs(p1 - p2).max() < 1e-14
    assert np.allclose(p1.mean(axis=0), m1, atol=1e-15)


def test_complex_direct_equals_doubling_and_odd_moments_vanish():
    """Peierls (complex H, real vectors, reading X16): direct == doubling; b = 0 bipartite
    lattice => exact odd moments 0 (Q8); |mu_n| <= mu_0 = 1 (Q11)."""
    H = oracle.lattice_csr(lat(2, (32, 32), flux=1 / 8))
    r = ki.rademacher(4, 4, 1024)
    m1 = oracle.moments_direct(H, 4.0, 0.0, r, 200)
    m2 = oracle.moments_doubling(H, 4.0, 0.0, r, 200)
    assert np.abs(m1 - m2).max() < 1e-14
    assert m1[0] == 1.0 and np.abs(m1).max() <= 1.0
    ex = oracle.exact_moments_from_eigs(oracle.harper_spectrum(32, 32, -1.0, 1 / 8), 4.0, 0.0, 200)
    assert np.abs(ex[1::2]).max() < 1e-14


def test_stochastic_estimator_unbiased_with_exact_variance():
    """Q9 (Eq 16): for Rademacher vectors Var(mu^_n) = 2 sum_{i!=j} [T_n(H~)]_ij^2 / (D^2 R).
    z-scores over many seeds must look standard normal; checks normalisation 1/(DR) and the
    recursion statistically, independently of the unit-vector path."""
    L, R, N, trials = 12, 4, 24, 60
    H = oracle.lattice_csr(lat(2, (L, L), onsite=ki.anderson_onsite(1, L * L, 1.5)))
    a, b = oracle.gershgorin(H)
    w, V = np.linalg.eigh(H.dense())
    x = np.clip((w - b) / a, -1, 1)
    D = L * L
    ex, var = np.zeros(N), np.zeros(N)
    for n in range(N):
        Tn = (V * np.cos(n * np.arccos(x))) @ V.T
        ex[n] = np.trace(Tn) / D
        var[n] = 2 * ((Tn ** 2).sum() - (np.diag(Tn) ** 2).sum()) / (D * D * R)
    z = []
    for s in range(trials):
        mu = oracle.moments_doubling(H, a, b, ki.rademacher(100 + s, R, D), N)
        z.append((mu[1:] - ex[1:]) / np.sqrt(var[1:]))
    z = np.array(z)
    assert np.abs(z).max() < 5.5
    assert 0.85 < z.std() < 1.15
    assert abs(z.mean()) < 4 / math.sqrt(z.size)


# ---------------------------------------------------------------- Jackson + DoS (Eq 6)
def test_jackson_equals_autocorrelation_definition():
    """Reading X8 closed form vs the kernel's defining construction (ref [10]): g_n is the
    normalised autocorrelation of a_v = sin(pi (v+1)/(N+1)), v = 0..N-1."""
    for N in (1, 2, 3, 17, 256, 1000):
        av = np.sin(np.pi * (np.arange(N) + 1) / (N + 1))
        g = np.array([av[:N - n] @ av[n:] for n in range(N)]) / (av @ av)
        assert np.abs(oracle.jackson(N) - g).max() < 1e-14
    g = oracle.jackson(64)
    assert g[0] == pytest.approx(1.0, abs=1e-15) and np.all(np.diff(g) < 0) and g[-1] > 0


def test_dos_gauss_chebyshev_normalisation_and_dct3():
    """Q12/Q13: on K >= N Chebyshev nodes sum_k (pi/K) sqrt(1-x_k^2) f(x_k) = mu_0; the direct
    sum of Eq (6) equals scipy's DCT-III."""
    from scipy.fft import dct
    H = oracle.lattice_csr(lat(2, (16, 16), flux=1 / 8))
    mu = oracle.moments_doubling(H, 4.0, 0.0, ki.rademacher(2, 4, 256), 64)
    K = 256
    x = oracle.chebyshev_nodes(K)
    a, b = 4.0, 0.0
    rho = oracle.dos(mu, a, b, a * x + b)
    f = rho * a  # f_KPM(x) = a rho(omega)
    assert abs((np.pi / K) * (np.sqrt(1 - x * x) * f).sum() - mu[0]) < 1e-14
    c = oracle.jackson(64) * mu
    ref = dct(np.concatenate([c, np.zeros(K - 64)]), type=3) / (np.pi * np.sqrt(1 - x * x))
    # scipy DCT-III: y_k = x_0 + 2 sum_{n>=1} x_n cos(pi n (2k+1)/(2K))
    assert np.abs(f - ref).max() < 1e-12


def test_dos_1d_exact_moments_reproduce_closed_form():
    """Q7: exact 1D moments (delta_{n0}) through Eq (6) give f = 1/(pi sqrt(1-x^2)), i.e. the
    closed-form chain DoS rho(E) = 1/(pi sqrt(4t^2 - E^2)) with a = 2 (checks the 1/a Jacobian)."""
    mu = oracle.exact_moments_from_eigs(oracle.lattice_spectrum(1, (1024, 1, 1), -1.0), 2.0, 0.0, 128)
    E = np.linspace(-1.95, 1.95, 101)
    rho = oracle.dos(mu, 2.0, 0.0, E)
    assert np.abs(rho / oracle.dos_closed_1d(E) - 1).max() < 1e-11
    assert np.all(oracle.dos(mu, 2.0, 0.0, np.array([-2.5, 2.0, 3.0])) == 0.0)


def test_closed_form_dos_moments():
    """O7 pinned by its power moments: int rho = 1, int E^2 rho = 2 ndim t^2,
    int E^4 rho = closed walks of length 4 (1D: 6, 2D: 36)."""
    from scipy.integrate import quad
    for f, ndim, W4 in [(oracle.dos_closed_1d, 1, 6), (oracle.dos_closed_2d, 2, 36)]:
        w = 2.0 * ndim
        for k, expect in [(0, 1.0), (2, 2.0 * ndim), (4, W4)]:
            val = sum(quad(lambda e: e ** k * f(np.array([e]))[0], lo, hi, limit=400)[0]
                      for lo, hi in [(-w, 0), (0, w)])
            assert abs(val - expect) < 1e-6 * max(1, expect)


def test_2d_kpm_dos_converges_to_elliptic_closed_form():
    """Paper Fig 6 claim: larger N resolves the DoS better.  With exact moments of
    a 256^2 lattice (equal to the infinite-lattice moments for n < 256) the Jackson-KPM DoS
    approaches the elliptic-K closed form away from the van Hove point: the error falls ~4x
    per doubling of N (Jackson resolution ~ pi/N)."""
    E = np.linspace(-3.5, 3.5, 57)
    E = E[np.abs(E) > 0.5]
    lam = oracle.lattice_spectrum(2, (256, 256, 1), -1.0)
    err = {}
    for N in (64, 128, 256):
        mu = oracle.exact_moments_from_eigs(lam, 4.0, 0.0, N)
        err[N] = np.abs(oracle.dos(mu, 4.0, 0.0, E) - oracle.dos_closed_2d(E)).max()
    assert err[256] < err[128] / 3 < err[64] / 9 < 0.001


# ---------------------------------------------------------------- NEXT-1: kernels, G, LDoS
def test_fejer_kernel_is_cesaro_mean_of_partial_sums():
    """kernel_coeffs('fejer') pinned by its construction: the Fejer-damped series equals the
    arithmetic mean of the truncated (Dirichlet, g = 1) series with 1..N terms."""
    H = oracle.lattice_csr(lat(2, (12, 10)))
    mu = oracle.moments_doubling(H, 4.0, 0.0, ki.rademacher(4, 3, 120), 24)
    E = np.linspace(-3.9, 3.9, 41)
    mean = np.mean([oracle.dos(mu[:m], 4.0, 0.0, E, kernel="none") for m in range(1, 25)], axis=0)
    assert np.abs(oracle.dos(mu, 4.0, 0.0, E, kernel="fejer") - mean).max() < 1e-13


def test_lorentz_kernel_limits():
    """kernel_coeffs('lorentz'): g_0 = 1, decreasing to g_N = 0 (beyond the last moment), and
    the lam -> 0 limit is the Fejer kernel (sinh(lam u)/sinh(lam) -> u)."""
    N = 50
    g = oracle.kernel_coeffs(N, "lorentz", 4.0)
    assert g[0] == 1.0 and np.all(np.diff(g) < 0) and 0 < g[-1] < 0.1
    assert np.abs(oracle.kernel_coeffs(N, "lorentz", 1e-5) - oracle.kernel_coeffs(N, "fejer")).max() < 1e-9
    assert np.array_equal(oracle.kernel_coeffs(N, "none"), np.ones(N))
    assert np.array_equal(oracle.kernel_coeffs(N, "jackson"), oracle.jackson(N))


def test_green_1d_exact_moments_equal_closed_form():
    """green() with the exact infinite-chain moments (mu_n = delta_n0, a = 2) is the textbook
    chain Green's function 1/sqrt((E + i0)^2 - 4t^2) inside and outside the band, for every
    kernel (g_0 = 1)."""
    mu = oracle.exact_moments_from_eigs(oracle.lattice_spectrum(1, (1024, 1, 1), -1.0), 2.0, 0.0, 64)
    E = np.concatenate([np.linspace(-1.9, 1.9, 39), [-3.0, -2.2, 2.1, 2.7, 5.0]])
    ref = oracle.green_closed_1d(E)
    for k in ("jackson", "lorentz", "none"):
        G = oracle.green(mu, 2.0, 0.0, E, kernel=k)
        assert np.abs(G / ref - 1).max() < 1e-10, k


def test_green_outside_spectrum_equals_resolvent_trace():
    """Outside [b-a, b+a] the undamped expansion converges geometrically (|t| < 1) to the exact
    resolvent (1/D) sum_k 1/(omega - E_k) of a random Hermitian H (dense eigvalsh)."""
    rng = np.random.default_rng(3)
    D = 40
    A = rng.standard_normal((D, D)) + 1j * rng.standard_normal((D, D))
    Hd = (A + A.conj().T) / 2
    ev = np.linalg.eigvalsh(Hd)
    b = 0.3
    a = 1.02 * max(ev.max() - b, b - ev.min())
    mu = oracle.exact_moments_from_eigs(ev, a, b, 400)
    w = np.array([b - 1.6 * a, b - 1.1 * a, b + 1.05 * a, b + 2.0 * a])
    ref = (1.0 / (w[:, None] - ev[None, :])).mean(axis=1)
    G = oracle.green(mu, a, b, w, kernel="none")
    assert np.abs(G.imag).max() == 0.0
    assert np.abs(G.real - ref).max() < 1e-12 * np.abs(ref).max()


def test_green_imaginary_part_is_minus_pi_dos():
    """Inside the band -Im G / pi is the KPM DoS of Eq (6) (same kernel), and Re G is an odd
    function of omega for a symmetric spectrum (b = 0, bipartite 2D lattice)."""
    H = oracle.lattice_csr(lat(2, (16, 16)))
    mu = oracle.moments_doubling(H, 4.0, 0.0, ki.rademacher(8, 5, 256), 64)
    mu[1::2] = 0.0  # exact odd moments of the bipartite lattice (Q8)
    E = np.linspace(-3.9, 3.9, 53)
    for k in ("jackson", "lorentz"):
        G = oracle.green(mu, 4.0, 0.0, E, kernel=k)
        assert np.abs(-G.imag / np.pi - oracle.dos(mu, 4.0, 0.0, E, kernel=k)).max() < 1e-13
        assert np.abs(G.real + G.real[::-1]).max() < 1e-12


def test_local_moments_average_to_trace_and_are_uniform_on_clean_lattices():
    """local_moments: (i) the average over all sites is the exact trace (dense eigvalsh, with
    Anderson disorder so sites differ); (ii) on a clean periodic lattice every site has the
    same local moments, equal to the exact DoS moments (translation invariance)."""
    onsite = ki.anderson_onsite(9, 60, 2.0)
    H = oracle.lattice_csr(lat(2, (10, 6), onsite=onsite))
    a, b = oracle.gershgorin(H)
    lm = oracle.local_moments(H, a, b, np.arange(60), 40)
    ex = oracle.exact_moments_dense(H, a, b, 40)
    assert np.abs(lm.mean(axis=0) - ex).max() < 1e-13
    assert np.abs(lm - lm[0]).max() > 1e-3  # disorder: sites differ
    H2 = oracle.lattice_csr(lat(3, (6, 5, 4)))
    lm2 = oracle.local_moments(H2, 6.0, 0.0, [0, 7, 33, 119], 30)
    ex2 = oracle.exact_moments_from_eigs(oracle.lattice_spectrum(3, (6, 5, 4), -1.0), 6.0, 0.0, 30)
    assert np.abs(lm2 - ex2[None, :]).max() < 1e-13


# ---------------------------------------------------------------- error bars (X28)
def test_moment_stats_textbook_mean_and_standard_error():
    """oracle.moment_stats against the textbook sample mean / stdev (statistics module) on a
    fixed table, column by column; R = 1 gives NaN standard errors."""
    import statistics
    pv = np.array([[1.0, 0.5, -2.0], [3.0, 0.25, 4.0], [2.0, -1.0, 1.5], [0.5, 0.0, 2.5]])
    mean, sem = oracle.moment_stats(pv)
    for n in range(3):
        col = list(pv[:, n])
        assert mean[n] == pytest.approx(statistics.fmean(col), rel=1e-15)
        assert sem[n] == pytest.approx(statistics.stdev(col) / math.sqrt(len(col)), rel=1e-14)
    m1, s1 = oracle.moment_stats(pv[:1])
    assert np.array_equal(m1, pv[0]) and np.isnan(s1).all()


def test_moment_stats_mean_is_the_estimate_and_diagonal_H_has_zero_error():
    """Mean over per-vector moments = the R-vector estimate (Eq 16 is their average); for a
    diagonal H (t = 0, Anderson only) xi^2 = 1 makes every vector's moment equal exactly, so
    the standard error is 0 up to the rounding of the mean; mu_0^(r) = 1 exactly for every vector on any H."""
    D, R, N = 64, 9, 20
    lat0 = lat(2, (8, 8), t=0.0, onsite=ki.anderson_onsite(4, D, 2.0))
    H0 = oracle.lattice_csr(lat0)
    a, b = oracle.gershgorin(H0, eps=0.01)
    mu, pv = oracle.moments_doubling(H0, a, b, ki.rademacher(8, R, D), N, per_vector=True)
    mean, sem = oracle.moment_stats(pv)
    assert np.abs(mean - mu).max() < 1e-14
    assert (pv == pv[0]).all() and sem.max() < 1e-15  # only the rounding of sum/R
    H = oracle.lattice_csr(lat(2, (8, 8), onsite=ki.anderson_onsite(4, D, 2.0)))
    a, b = oracle.gershgorin(H)
    mu, pv = oracle.moments_doubling(H, a, b, ki.rademacher(8, R, D), N, per_vector=True)
    mean, sem = oracle.moment_stats(pv)
    assert np.abs(mean - mu).max() < 1e-14
    assert sem[0] == 0.0 and (sem[1:] > 0).all()


def test_moment_stats_standard_error_matches_rademacher_variance_closed_form():
    """For Rademacher vectors Var(mu_n^(r)) = 2 sum_{i!=j} [T_n(H~)]_ij^2 / D^2 (Hutchinson);
    the sample standard error times sqrt(R) must approach it (R = 4000: the relative error
    of a sample variance is ~ sqrt(2/R) times the kurtosis factor, well inside 20%)."""
    L, R, N = 6, 4000, 12
    D = L * L
    H = oracle.lattice_csr(lat(2, (L, L), onsite=ki.anderson_onsite(2, D, 1.5)))
    a, b = oracle.gershgorin(H)
    w, V = np.linalg.eigh(H.dense())
    x = np.clip((w - b) / a, -1, 1)
    sig = np.zeros(N)
    for n in range(N):
        Tn = (V * np.cos(n * np.arccos(x))) @ V.T
        sig[n] = np.sqrt(2 * ((Tn ** 2).sum() - (np.diag(Tn) ** 2).sum())) / D
    _, pv = oracle.moments_doubling(H, a, b, ki.rademacher(77, R, D), N, per_vector=True)
    _, sem = oracle.moment_stats(pv)
    assert sem[0] == 0.0 and sig[0] < 1e-12
    ratio = sem[1:] * math.sqrt(R) / sig[1:]
    assert np.abs(ratio - 1).max() < 0.2, ratio
