"""GPU parity of SURVEY.md 8(f) NEXT-1 (through the C ABI) against the CPU oracle:
damping kernels (Eq 6-7 with the kernels of ref [10]), the DoS with every kernel, the
retarded Green's function (reading X24), and local moments <i|T_n(H~)|i> from unit start
vectors (KPM_LOCAL).  Tolerances: reading X17 (normwise 1e-10) for moments.  The expansions
evaluate T_n = cos(n theta) (and sin(n theta)) term by term on both sides (theta = arccos x).
Near x = +-1 the expansion is ill-conditioned for ANY evaluation: the terms cancel and the sum is
divided by sin theta, so the bar is pointwise (X27):
|drho(x)| <= eps sum_n |c_n| (2 + 4 n theta) / (pi a sin theta), plus 1e-10 relative to max|value|
on |x| <= 1 - 1e-6 (where 1/sin theta <= 708), at the configs' N = 1024-4096 too."""
import numpy as np
import pytest

import kpm_inputs as ki
import oracle

pytestmark = pytest.mark.gpu
KERNELS = {"jackson": 0, "none": 1, "lorentz": 2, "fejer": 3}


@pytest.fixture(scope="module")
def kpm():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1105_5481_b200 import kpm as k
    return k


def lat_of(ndim, L, W=0.0, flux=0.0, dseed=5):
    L = tuple(L) + (1,) * (3 - len(L))
    D = L[0] * L[1] * L[2]
    return dict(ndim=ndim, L=L, D=D, t=-1.0, onsite=ki.anderson_onsite(dseed, D, W) if W else None, flux=flux)


def rel(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300)


def check_expansion(got, ref, mu, a, b, om, name, lam=4.0, what="dos"):
    """DESIGN.md X27: normwise 1e-10 on |x| <= 1 - 1e-6, and everywhere inside the band the
    pointwise rounding bound eps sum|c_n| (2 + 4 n theta) / (pi a sin theta) (x 2 for G's two sums)."""
    N = len(mu)
    x = (np.asarray(om) - b) / a
    inner = np.abs(x) <= 1 - 1e-6
    assert rel(got[inner], ref[inner]) < 1e-10
    c = oracle.kernel_coeffs(N, name, lam) * mu
    c[1:] *= 2
    ins = np.abs(x) < 1
    th = np.arccos(x[ins])
    n = np.arange(N)
    bound = np.finfo(float).eps * (np.abs(c)[None, :] * (2 + 4 * np.outer(th, n))).sum(axis=1) / (a * np.sin(th))
    if what == "dos":
        bound /= np.pi
    err = np.abs(got[ins] - ref[ins])
    assert np.all(err <= bound), (err / bound).max()


@pytest.mark.parametrize("name", sorted(KERNELS))
@pytest.mark.parametrize("N", [1, 2, 7, 64, 1000])
def test_damping_matches_oracle(kpm, name, N):
    for lam in (0.5, 4.0):
        g = kpm.kpm_damping(N, KERNELS[name], lam)
        assert rel(g, oracle.kernel_coeffs(N, name, lam)) < 1e-13


@pytest.mark.parametrize("name", sorted(KERNELS))
def test_dos_every_kernel_matches_oracle(kpm, name):
    lat = lat_of(2, (24, 20), flux=1 / 4, W=1.0)
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    mu = oracle.moments_doubling(H, a, b, ki.rademacher(3, 6, lat["D"]), 200)
    om = np.concatenate([np.linspace(b - 1.2 * a, b + 1.2 * a, 301), [b - a, b + a]])
    rho = kpm.kpm_dos_ex(mu, a, b, om, kernel=KERNELS[name], lam=3.0)
    check_expansion(rho, oracle.dos(mu, a, b, om, kernel=name, lam=3.0), mu, a, b, om, name, lam=3.0)
    if name == "jackson":
        assert np.array_equal(rho, kpm.kpm_dos(mu, a, b, om))


@pytest.mark.parametrize("name", ["jackson", "lorentz", "none"])
def test_green_matches_oracle_inside_and_outside(kpm, name):
    lat = lat_of(3, (8, 7, 6), W=2.0)
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    mu = oracle.moments_doubling(H, a, b, ki.rademacher(4, 5, lat["D"]), 128)
    om = np.concatenate([np.linspace(b - 0.999 * a, b + 0.999 * a, 257),
                         b + a * np.array([-3.0, -1.5, -1.001, 1.001, 1.2, 4.0])])
    G = kpm.kpm_green(mu, a, b, om, kernel=KERNELS[name], lam=4.0)
    ref = oracle.green(mu, a, b, om, kernel=name, lam=4.0)
    assert rel(G.real, ref.real) < 1e-10 and rel(G.imag, ref.imag) < 1e-10
    assert np.all(np.isnan(kpm.kpm_green(mu, a, b, [b - a, b + a], kernel=KERNELS[name])))
    # Im G = -pi rho (same kernel)
    ins = np.abs(om - b) < a
    rho = kpm.kpm_dos_ex(mu, a, b, om[ins], kernel=KERNELS[name], lam=4.0)
    assert rel(-G.imag[ins] / np.pi, rho) < 1e-12  # same terms on both


# the configs' moment counts (BASELINE.json c2 N=1024, c3 N=2048, c4 N=4096), on lattices of the
# same kinds (moments from the oracle; only the expansion is under test here)
BIG_N = {
    "c2_like_N1024": (lat_of(2, (40, 36)), 1024),
    "c3_like_N2048": (lat_of(3, (12, 11, 10), W=2.0), 2048),
    "c4_like_N4096": (lat_of(2, (32, 24), flux=1 / 8), 4096),
}


@pytest.mark.parametrize("name", ["jackson", "lorentz", "none"])
@pytest.mark.parametrize("case", sorted(BIG_N))
def test_dos_green_at_config_N(kpm, case, name):
    """DoS and Green's function at N = 1024, 2048, 4096: normwise 1e-10 against the oracle and
    the pointwise bound of reading X27, on a grid that reaches x = +-(1 - 1e-9) and on the N
    Chebyshev nodes."""
    lat, N = BIG_N[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    mu = oracle.moments_doubling(H, a, b, ki.rademacher(7, 3, lat["D"]), N)
    x = np.concatenate([np.linspace(-1 + 1e-9, 1 - 1e-9, 2001), oracle.chebyshev_nodes(N),
                        [-1 + 1e-12, 1 - 1e-12]])
    om = b + a * x
    rho = kpm.kpm_dos_ex(mu, a, b, om, kernel=KERNELS[name], lam=4.0)
    check_expansion(rho, oracle.dos(mu, a, b, om, kernel=name, lam=4.0), mu, a, b, om, name)
    G = kpm.kpm_green(mu, a, b, om, kernel=KERNELS[name], lam=4.0)
    Gr = oracle.green(mu, a, b, om, kernel=name, lam=4.0)
    check_expansion(G.real, Gr.real, mu, a, b, om, name, what="green")
    check_expansion(G.imag, Gr.imag, mu, a, b, om, name, what="green")
    out = b + a * np.array([-2.0, -1.01, 1.01, 3.0])  # outside the band
    Go = kpm.kpm_green(mu, a, b, out, kernel=KERNELS[name], lam=4.0)
    assert rel(Go.real, oracle.green(mu, a, b, out, kernel=name, lam=4.0).real) < 1e-10


LOCAL_CASES = {
    "2d_anderson": (lat_of(2, (37, 29), W=2.0), 41, [0, 1, 36, 500, 1072]),
    "3d_tma_march": (lat_of(3, (32, 32, 20), W=1.0), 24, list(range(0, 20480, 1301))),  # 16 sites: 8 lanes
    "2d_two_step": (lat_of(2, (128, 24)), 40, list(range(3, 3072, 97))),               # 32 sites
    "peierls": (lat_of(2, (32, 20), flux=1 / 8), 30, [5, 17, 639]),
    "1d": (lat_of(1, (1000,)), 33, [0, 999, 500]),
}


@pytest.mark.parametrize("path", ["default", "no_small"])
@pytest.mark.parametrize("case", sorted(LOCAL_CASES))
def test_local_moments_match_oracle(kpm, case, path):
    """KPM_LOCAL: unit start vectors e_i generated on the GPU; every launch path (single-launch
    smem, first step + TMA march / two-step / generic step kernels)."""
    lat, N, sites = LOCAL_CASES[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    ref = oracle.local_moments(H, a, b, sites, N)
    h = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"], flux=lat["flux"])
    h.set_plan_opts(no_small=int(path == "no_small"))
    lm = h.moments_local(N, sites)
    assert lm.shape == (len(sites), N)
    assert rel(lm, ref) < 1e-10
    assert np.all(lm[:, 0] == 1.0)
    # the same through the generic call, and the direct scheme (Eq 19)
    lm2 = h.moments_ex(N, len(sites), 0, r0=np.asarray(sites, dtype=np.int64), flags=kpm.KPM_LOCAL)
    assert np.array_equal(lm, lm2)


def test_local_moments_csr_and_vector_partition(kpm):
    """KPM_LOCAL through CSR input (ELL kernel), and split over 3 ranks of the vector partition:
    each rank returns its share of the sites."""
    lat = lat_of(2, (20, 18), W=1.5)
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    sites = [0, 3, 77, 100, 255, 359, 12]
    ref = oracle.local_moments(H, a, b, sites, 36)
    h = kpm.kpm_create_csr(H.D, H.rowptr, H.col, H.val_re, a, b)
    assert rel(h.moments_local(36, sites), ref) < 1e-10
    parts = []
    for r in range(3):
        hr = kpm.kpm_create_stencil(2, lat["L"], -1.0, a, b, onsite=lat["onsite"],
                                    dist=(kpm.KPM_PART_VECTORS, r, 3))
        parts.append(hr.moments_local(36, sites))
    assert rel(np.concatenate(parts), ref) < 1e-10


def test_local_moments_bad_sites_rejected(kpm):
    lat = lat_of(2, (16, 8))
    h = kpm.kpm_create_stencil(2, lat["L"], -1.0, 4.0, 0.0)
    for bad in ([-1], [128], [0, 5, 1 << 40]):
        with pytest.raises(kpm.KPMError):
            h.moments_local(10, bad)


def test_ldos_green_of_gpu_local_moments_matches_dense_resolvent(kpm):
    """End to end: G_ii(omega) from the GPU local moments (no damping, many moments) equals the
    diagonal of the dense resolvent (omega - H)^-1 outside the spectrum (geometric convergence)."""
    lat = lat_of(2, (10, 8), W=2.0)
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    a *= 1.05
    sites = [0, 9, 41, 79]
    h = kpm.kpm_create_stencil(2, lat["L"], -1.0, a, b, onsite=lat["onsite"])
    lm = h.moments_local(400, sites)
    om = b + a * np.array([-1.8, -1.1, 1.15, 2.5])
    Hd = H.dense()
    for k, i in enumerate(sites):
        G = kpm.kpm_green(lm[k], a, b, om, kernel=kpm.KPM_KERNEL_NONE)
        ref = np.array([np.linalg.inv(w * np.eye(H.D) - Hd)[i, i] for w in om])
        assert rel(G, ref) < 1e-10


def test_moment_stats_fixed_table_matches_oracle(kpm):
    """kpm_moment_stats (error bars, reading X28) vs oracle.moment_stats on a seeded table
    spanning several 128-thread blocks and a ragged tail; R = 1 gives NaN; bad args raise."""
    pv = np.random.default_rng(5).normal(0.3, 0.02, size=(37, 301))
    mean, sem = kpm.kpm_moment_stats(pv)
    rm, rs = oracle.moment_stats(pv)
    assert rel(mean, rm) < 1e-14 and rel(sem, rs) < 1e-12
    m1, s1 = kpm.kpm_moment_stats(pv[:1])
    assert np.array_equal(m1, pv[0]) and np.isnan(s1).all()
    with pytest.raises(kpm.KPMError):
        kpm.kpm_moment_stats(np.zeros((0, 4)))


@pytest.mark.parametrize("L,R,N", [((16, 16, 10), 32, 31), ((64, 40, 1), 16, 50)])
def test_moment_stats_of_gpu_per_vector_moments(kpm, L, R, N):
    """Error bars end to end: per-vector moments from the GPU recursion (KPM_PER_VECTOR),
    then kpm_moment_stats; the mean equals kpm_moments (same vectors) and both outputs
    match the oracle's per-vector moments run through oracle.moment_stats."""
    lat = lat_of(3 if L[2] > 1 else 2, L, W=2.0)
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    _, ref_pv = oracle.moments_doubling(H, a, b, ki.rademacher(13, R, lat["D"]), N, per_vector=True)
    rm, rs = oracle.moment_stats(ref_pv)
    h = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"])
    pv = h.moments_ex(N, R, 13, flags=kpm.KPM_PER_VECTOR)
    mean, sem = kpm.kpm_moment_stats(pv)
    assert rel(mean, h.moments(N, R, 13)) < 1e-13
    assert rel(mean, rm) < 1e-10
    assert sem[0] < 1e-15 and rel(sem, rs) < 1e-7


def test_moment_stats_over_a_vector_partition(kpm):
    """Error bars under KPM_PART_VECTORS: the per-vector moments of a 3-way vector split,
    concatenated in rank order, are the global vectors' moments, so their statistics match
    the oracle's on all R vectors."""
    lat = lat_of(2, (48, 20), W=1.0)
    N, R = 40, 20
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    _, ref_pv = oracle.moments_doubling(H, a, b, ki.rademacher(9, R, lat["D"]), N, per_vector=True)
    parts = []
    for rank in range(3):
        h = kpm.kpm_create_stencil(2, lat["L"], -1.0, a, b, onsite=lat["onsite"],
                                   dist=(kpm.KPM_PART_VECTORS, rank, 3))
        parts.append(h.moments_ex(N, R, 9, flags=kpm.KPM_PER_VECTOR))
    pv = np.concatenate(parts)
    assert pv.shape == (R, N)
    mean, sem = kpm.kpm_moment_stats(pv)
    rm, rs = oracle.moment_stats(ref_pv)
    assert rel(mean, rm) < 1e-10 and rel(sem, rs) < 1e-7
