"""GPU parity of the dense-H variant (the paper's own scheme,
PAPER.md:140, 241-253): DMMA GEMM step with the fused recursion and moment sums
(kpm_dense.cuh) against the CPU oracle on the same stored H and start vectors.
Bar: reading X17, normwise 1e-10."""
import numpy as np
import pytest

import kpm_inputs as ki
import oracle

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.fixture(scope="module")
def kpm():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1105_5481_b200 import kpm as k
    return k


def normwise(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300)


def random_symmetric(D, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((D, D))
    return (A + A.T) / 2


CASES = {
    # name: (H builder, N, R) -- ragged D (padding to 64) and R (padding to 64), several tiles
    "random_D100_R10": (lambda: random_symmetric(100, 1), 33, 10),
    "random_D200_R130": (lambda: random_symmetric(200, 2), 40, 130),
    "paper_10cube_R70": (lambda: ki.lattice_dense(ki.lattice(ki.CONFIGS["c3"], L=(10, 10, 10), W=0.0)), 64, 70),
    "anderson_D512_R64": (lambda: ki.lattice_dense(ki.lattice(ki.CONFIGS["c3"], L=(8, 8, 8))), 21, 64),
    "tiny_D5_R1": (lambda: random_symmetric(5, 3), 9, 1),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_dense_moments_match_oracle(kpm, case):
    build, N, R = CASES[case]
    Hd = build()
    D = Hd.shape[0]
    a, b = kpm.kpm_gershgorin_dense(Hd)
    H = oracle.csr_from_dense(Hd)
    ao, bo = oracle.gershgorin(H)
    assert abs(a - ao) < 1e-12 * abs(ao) and abs(b - bo) < 1e-12 * max(1, abs(bo))
    b += 0.04 * a
    a *= 1.05
    r = ki.rademacher(17, R, D)
    ref, ref_pv = oracle.moments_doubling(H, a, b, r, N, per_vector=True)
    h = kpm.kpm_create_dense(Hd, a, b)
    mu = h.moments(N, R, 17)
    assert normwise(mu, ref) < TOL
    assert np.array_equal(h.moments_ex(N, R, 17, r0=r), mu), "generated vs caller-supplied start block"
    pv = h.moments_ex(N, R, 17, flags=kpm.KPM_PER_VECTOR)
    assert normwise(pv, ref_pv) < TOL
    assert np.array_equal(h.moments(N, R, 17), mu), "not deterministic"


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 8, 9])
def test_dense_small_N_and_odd_tail(kpm, N):
    Hd = random_symmetric(70, 5)
    H = oracle.csr_from_dense(Hd)
    a, b = oracle.gershgorin(H)
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(2, 9, 70), N)
    h = kpm.kpm_create_dense(Hd, a, b)
    assert normwise(h.moments(N, 9, 2), ref) < TOL


def test_dense_equals_stencil_same_lattice(kpm):
    """Q14: the same lattice H as dense matrix and as stencil gives the same moments."""
    lat = ki.lattice(ki.CONFIGS["c3"], L=(8, 6, 10))
    a, b = kpm.kpm_gershgorin_stencil(3, lat["L"], -1.0, onsite=lat["onsite"])
    hs = kpm.kpm_create_stencil(3, lat["L"], -1.0, a, b, onsite=lat["onsite"])
    hd = kpm.kpm_create_dense(ki.lattice_dense(lat), a, b)
    assert normwise(hd.moments(100, 40, 9), hs.moments(100, 40, 9)) < 1e-13


def test_dense_local_moments_and_vector_partition(kpm):
    """KPM_LOCAL through the dense path, and a 2-rank vector split (raw sums summed on the
    host + kpm_assemble) equal to the single-rank moments."""
    Hd = ki.lattice_dense(ki.lattice(ki.CONFIGS["c3"], L=(6, 5, 4)))
    H = oracle.csr_from_dense(Hd)
    a, b = oracle.gershgorin(H)
    sites = [0, 7, 59, 119]
    h = kpm.kpm_create_dense(Hd, a, b)
    assert normwise(h.moments_local(30, sites), oracle.local_moments(H, a, b, sites, 30)) < TOL
    N, R = 24, 13
    full = h.moments(N, R, 4)
    S = sum(kpm.kpm_create_dense(Hd, a, b, dist=(kpm.KPM_PART_VECTORS, g, 2)).moments_ex(N, R, 4, flags=kpm.KPM_RAW_SUMS)
            for g in range(2))
    assert normwise(kpm.kpm_assemble_host(S, N, 120, R), full) < 1e-13


def test_dense_rejects_complex_and_direct(kpm):
    Hd = random_symmetric(16, 1)
    h = kpm.kpm_create_dense(Hd, 20.0, 0.0)
    with pytest.raises(kpm.KPMError):
        h.moments_ex(8, 4, 1, flags=kpm.KPM_DIRECT)
