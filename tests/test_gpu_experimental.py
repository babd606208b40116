"""GPU parity of the EXPERIMENTAL kernels (libkpm_exp.so, kpm_plan_opts.experimental): parity-green
but measured slower than the default plan, so they are not in libkpm.so.
Same bar as tests/test_gpu_parity.py (X17)."""
import numpy as np
import pytest

import kpm_inputs as ki
import oracle
from test_gpu_parity import CASES, TMA_CASES, TOL, lat_of, make, normwise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kpm():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1105_5481_b200 import kpm as k
    k.use_experimental(True)
    yield k
    k.use_experimental(False)


THREE_D_TWO_STEP_CASES = {
    "anderson_rr": (lat_of(3, (64, 32, 6), W=2.0), 64),          # 4 lane groups x 32 pencils: round-robin
    "clean_rr": (lat_of(3, (64, 64, 5)), 48),                    # 3 lane groups, no on-site array
    "anderson_contig": (lat_of(3, (16, 16, 10), W=2.0), 32),     # 8 columns -> contiguous plane ranges
    "single_pencil_L2_2": (lat_of(3, (16, 8, 2), W=1.0), 16),    # z wraps onto itself, H = 1 segments
    "one_pencil_wide_R": (lat_of(3, (8, 8, 9), W=1.0), 128),     # 8 lane groups of one pencil
}


@pytest.mark.parametrize("shape", [0, 1, 2, 3])
@pytest.mark.parametrize("case", sorted(THREE_D_TWO_STEP_CASES))
@pytest.mark.parametrize("N", [6, 7, 8, 9, 12, 15])
def test_3d_two_step_kernel_matches_oracle(kpm, case, N, shape):
    """3D temporal blocking (kpm_tma32.cuh, experimental = 1) for every instantiated tile
    (exp_param: 8x8 sites x 8 lanes, 16x4x8, 8x4x16, 16x8x8) and every parity of the step count and of N, vs
    the oracle and vs the single-step dense-box kernel."""
    lat, R = THREE_D_TWO_STEP_CASES[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    b += 0.02 * a
    a *= 1.03
    r = ki.rademacher(8, R, lat["D"])
    ref, ref_pv = oracle.moments_doubling(H, a, b, r, N, per_vector=True)
    h = make(kpm, lat, a, b, no_small=1, experimental=kpm.EXP_3D_TWO_STEP, exp_param=shape)
    info = h.plan_info(N, R)
    tx, ty, tl = {0: (8, 8, 8), 1: (16, 4, 8), 2: (8, 4, 16), 3: (16, 8, 8)}[shape]
    fits = (lat["L"][0] % tx == 0 and lat["L"][1] % ty == 0 and ((R + 1) // 2) % tl == 0)
    assert info["two_step3d"] == int(N // 2 - 1 >= 2 and fits), info
    mu = h.moments(N, R, 8)
    assert normwise(mu, ref) < TOL
    pv = h.moments_ex(N, R, 8, flags=kpm.KPM_PER_VECTOR)
    assert normwise(pv, ref_pv) < TOL
    assert np.array_equal(h.moments(N, R, 8), mu), "not deterministic"
    assert np.array_equal(h.moments_ex(N, R, 8, r0=r), mu)
    h.set_plan_opts(no_small=1)
    assert h.plan_info(N, R)["two_step3d"] == 0
    assert normwise(h.moments(N, R, 8), ref) < TOL


KSTEP_CASES = {
    "2d_R64": (lat_of(2, (64, 200)), 64),                        # segments cross pencil columns
    "2d_anderson_R16": (lat_of(2, (128, 24), W=2.0), 16),        # 8 lanes per site: TL 8, TX 64
    "2d_peierls_R32": (lat_of(2, (64, 16), flux=1 / 8), 32),
    "2d_peierls_anderson_R16": (lat_of(2, (32, 30), flux=1 / 4, W=1.0), 16),
    "2d_one_row_per_cta": (lat_of(2, (32, 4)), 32),              # 8 output rows -> 8 CTAs, H = 1
    "2d_L1_2": (lat_of(2, (64, 2), W=1.0), 48),                  # rows wrap around several times
    "2d_R96_two_groups": (lat_of(2, (96, 40)), 96),              # 3 pencils x 3 lane groups
}


@pytest.mark.parametrize("ks", [3, 4])
@pytest.mark.parametrize("case", sorted(KSTEP_CASES))
@pytest.mark.parametrize("N", [10, 11, 12, 13, 16, 19, 26])
def test_multi_step_kernel_matches_oracle(kpm, case, N, ks):
    """2D: the KS-step (default KS = 3) deep temporal-blocking kernel (kpm_tmak.cuh) mixed with two-step and
    single-step launches for the remainder, every parity of N (odd-N tail in the last launch)."""
    lat, R = KSTEP_CASES[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    b -= 0.02 * a
    a *= 1.03
    r = ki.rademacher(13, R, lat["D"])
    ref, ref_pv = oracle.moments_doubling(H, a, b, r, N, per_vector=True)
    h = make(kpm, lat, a, b, no_small=1, experimental=kpm.EXP_KSTEP, exp_param=ks, no_three_step=1, no_four_step=1)
    info = h.plan_info(N, R)
    assert info["ks"] == ks, info
    mu = h.moments(N, R, 13)
    assert normwise(mu, ref) < TOL
    pv = h.moments_ex(N, R, 13, flags=kpm.KPM_PER_VECTOR)
    assert normwise(pv, ref_pv) < TOL
    assert np.array_equal(h.moments(N, R, 13), mu), "not deterministic"
    _, launches, _ = h.last_timing()
    M = N // 2
    rem = (M - 1) % ks
    assert launches == (M - 1) // ks + (rem // 2 + rem % 2 if info["two_step"] else rem), (launches, info)
    h.set_plan_opts(no_small=1, no_three_step=1, no_four_step=1)
    assert h.plan_info(N, R)["ks"] == 0
    assert normwise(h.moments(N, R, 13), ref) < TOL




PERSIST_CASES = dict(**{k: v for k, v in CASES.items()}, **{"tma_" + k: v for k, v in TMA_CASES.items()})


@pytest.mark.parametrize("form", ["stencil", "csr"])
@pytest.mark.parametrize("case", sorted(PERSIST_CASES))
def test_persistent_kernel_matches_oracle(kpm, case, form):
    """The whole recursion in one cooperative launch with grid-wide barriers between steps
    (kpm_persist.cuh, L2-resident blocks): same moments as the oracle, per vector too, with
    generated and caller-supplied start vectors, deterministic."""
    lat, N, R = PERSIST_CASES[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    b -= 0.02 * a
    a *= 1.04
    r = ki.rademacher(12, R, lat["D"])
    ref, ref_pv = oracle.moments_doubling(H, a, b, r, N, per_vector=True)
    h = make(kpm, lat, a, b, form, no_small=1, experimental=kpm.EXP_PERSIST)
    assert h.plan_info(N, R)["persist"] == int(N // 2 >= 2), h.plan_info(N, R)
    mu = h.moments(N, R, 12)
    assert normwise(mu, ref) < TOL
    assert normwise(h.moments_ex(N, R, 12, flags=kpm.KPM_PER_VECTOR), ref_pv) < TOL
    assert np.array_equal(h.moments_ex(N, R, 12, r0=r), mu)
    assert np.array_equal(h.moments(N, R, 12), mu), "not deterministic"


