"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same
seeded inputs.  Bar (X17): normwise max_n |mu_gpu - mu_orc| <= 1e-10 *
max_n |mu_orc|; bitwise for config c1 (every a_n is integer-valued, Q4) and for the
Rademacher generator (integer work)."""
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


def make(kpm, lat, a, b, form="stencil", **opts):
    """A handle for lattice lat (stencil descriptor or the same H as CSR) with plan options opts
    (kpm_plan_opts fields, e.g. no_small=1)."""
    if form == "stencil":
        h = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"], flux=lat["flux"])
    else:
        H = oracle.lattice_csr(lat)
        val = H.val_re + 1j * H.val_im if H.is_complex else H.val_re
        h = kpm.kpm_create_csr(H.D, H.rowptr, H.col, val, a, b)
    if opts:
        h.set_plan_opts(**opts)
    return h


def lat_of(ndim, L, t=-1.0, W=0.0, flux=0.0, dseed=5):
    L = tuple(L) + (1,) * (3 - len(L))
    D = L[0] * L[1] * L[2]
    return dict(ndim=ndim, L=L, D=D, t=t, onsite=ki.anderson_onsite(dseed, D, W) if W else None, flux=flux)


CASES = {
    # name: (lattice, N, R)  -- sizes span several CTAs/lane groups with ragged tails
    "1d_ragged": (lat_of(1, (1000,)), 37, 5),
    "2d": (lat_of(2, (37, 29)), 64, 7),
    "2d_wide": (lat_of(2, (64, 48)), 33, 70),          # R > 64: two lane groups, odd N
    "3d_clean": (lat_of(3, (13, 11, 9)), 50, 13),
    "3d_anderson": (lat_of(3, (12, 10, 16), W=2.0), 64, 16),
    "3d_L2": (lat_of(3, (2, 7, 5), W=1.0), 20, 3),    # L = 2: both neighbours coincide
    "peierls": (lat_of(2, (32, 20), flux=1 / 8), 60, 9),
    "peierls_anderson": (lat_of(2, (24, 24), flux=1 / 4, W=1.0), 41, 4),
}


@pytest.mark.parametrize("path", ["default", "no_small"])
@pytest.mark.parametrize("form", ["stencil", "csr"])
@pytest.mark.parametrize("case", sorted(CASES))
def test_moments_match_oracle(kpm, case, form, path):
    """default: these sizes run the single-launch shared-memory path (kpm_small.cuh);
    no_small: the per-step launch path (first-step + generic/ELL step kernels)."""
    lat, N, R = CASES[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    b += 0.05 * a  # exercise the shift term (still encloses the spectrum after widening a)
    a *= 1.06
    r = ki.rademacher(11, R, lat["D"])
    ref, ref_pv = oracle.moments_doubling(H, a, b, r, N, per_vector=True)
    h = make(kpm, lat, a, b, form, no_small=int(path == "no_small"))
    mu = h.moments(N, R, 11)
    assert normwise(mu, ref) < TOL
    mu_r0 = h.moments_ex(N, R, 11, r0=r)
    assert np.array_equal(mu, mu_r0), "on-the-fly generator differs from kpm_inputs.rademacher"
    pv = h.moments_ex(N, R, 11, flags=kpm.KPM_PER_VECTOR)
    assert pv.shape == (R, N) and normwise(pv, ref_pv) < TOL
    assert np.array_equal(h.moments(N, R, 11), mu), "not deterministic"


# shapes that take the TMA-pipelined march kernel (lanes per site a multiple of 8, tiles
# dividing the lattice), incl. more planes than CTAs (ranges crossing pencils), PX = PY = 1
TMA_CASES = {
    "2d_R64": (lat_of(2, (64, 200)), 40, 64),
    "2d_anderson_R16": (lat_of(2, (128, 24), W=2.0), 33, 16),
    "2d_peierls_R32": (lat_of(2, (64, 16), flux=1 / 8), 41, 32),
    "2d_peierls_anderson_R16": (lat_of(2, (32, 30), flux=1 / 4, W=1.0), 30, 16),
    "3d_R16": (lat_of(3, (32, 32, 40)), 24, 16),
    "3d_anderson_R32": (lat_of(3, (16, 16, 10), W=2.0), 31, 32),
    "3d_single_pencil": (lat_of(3, (16, 8, 6), W=1.0), 20, 16),
    "3d_anderson_R48": (lat_of(3, (32, 16, 12), W=2.0), 19, 48),
    "3d_round_robin": (lat_of(3, (256, 128, 4), W=2.0), 17, 64),  # 4 lane groups x 256 pencils
    # 4 lanes per site (small R per GPU, e.g. c2's share at 8 GPUs): 64-site two-step tiles
    "2d_R8_four_lanes": (lat_of(2, (128, 40)), 40, 8),
    "2d_anderson_R8_four_lanes": (lat_of(2, (256, 20), W=2.0), 33, 8),
    "2d_peierls_R4_four_lanes": (lat_of(2, (64, 16), flux=1 / 8), 41, 4),
}


def two_step_expected(lat, info, N=None):
    """The planner's two-step rule: 2D, a tile width TX2 (1024 lanes per row, or 64 sites with 4
    lanes per site) dividing L0, at least two recursion steps."""
    L0 = lat["L"][0]
    ok = lat["ndim"] == 2 and (L0 % (1024 // info["TL"]) == 0 or (info["TL"] == 4 and L0 % 64 == 0))
    if N is not None:
        ok = ok and N // 2 - 1 >= 2
    if info["two_step"]:
        assert L0 % info["TX2"] == 0 and info["TX2"] in (1024 // info["TL"], 64), info
    return int(ok)


@pytest.mark.parametrize("case", sorted(TMA_CASES))
def test_tma_march_matches_oracle(kpm, case):
    lat, N, R = TMA_CASES[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    b -= 0.03 * a
    a *= 1.05
    r = ki.rademacher(21, R, lat["D"])
    ref, ref_pv = oracle.moments_doubling(H, a, b, r, N, per_vector=True)
    h = make(kpm, lat, a, b, no_small=1)  # some of these fit the single-launch smem path
    info = h.plan_info(N, R)
    assert info["tma"] == 1, info
    assert info["round_robin"] == (case == "3d_round_robin"), info
    if lat["ndim"] == 2:
        assert info["two_step"] == two_step_expected(lat, info), info
    else:  # the 3D two-step kernel (kpm_tma32.cuh) is experimental (libkpm_exp.so)
        assert info["two_step"] == info["two_step3d"] == 0, info
    mu = h.moments(N, R, 21)
    assert normwise(mu, ref) < TOL
    pv = h.moments_ex(N, R, 21, flags=kpm.KPM_PER_VECTOR)
    assert normwise(pv, ref_pv) < TOL
    assert np.array_equal(h.moments(N, R, 21), mu), "not deterministic"
    assert np.array_equal(h.moments_ex(N, R, 21, r0=r), mu)
    if lat["ndim"] == 3:  # dense-box kernel (kpm_tma3.cuh) vs the generic-tile march kernel
        assert info["box3"] == ((info["TX"], info["TY"], info["TL"]) in [(16, 8, 8), (8, 8, 16), (4, 8, 32)]), info
        h.set_plan_opts(no_small=1, no_box3=1)
        assert h.plan_info(N, R)["box3"] == 0
        assert normwise(h.moments(N, R, 21), ref) < TOL


@pytest.mark.parametrize("tl", [8, 16, 32])
def test_3d_box_kernel_every_tile_width(kpm, tl):
    """The 3D dense-box kernel for each instantiated tile (TL = 8, 16, 32 lanes per site; the
    plan's TL pinned by kpm_plan_opts.tma_lanes), on-site disorder, round-robin columns, vs the oracle."""
    lat = lat_of(3, (32, 24, 10), W=2.0)
    N, R = 23, 64
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(6, R, lat["D"]), N)
    h = make(kpm, lat, a, b, no_small=1, tma_lanes=tl)
    info = h.plan_info(N, R)
    assert info["TL"] == tl and info["box3"] == 1, info
    assert normwise(h.moments(N, R, 6), ref) < TOL


@pytest.mark.parametrize("case", [c for c in sorted(TMA_CASES) if c.startswith("2d")])
@pytest.mark.parametrize("N", [5, 6, 7, 8, 9])
def test_two_step_pairs_and_single_steps(kpm, case, N):
    """2D: the two-step kernel (temporal blocking) and the single-step kernel give the oracle's
    moments for every parity of the step count and of N (odd-N tail inside a pair)."""
    lat, _, R = TMA_CASES[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(5, R, lat["D"]), N)
    h = make(kpm, lat, a, b, no_small=1)
    info = h.plan_info(N, R)
    assert info["two_step"] == two_step_expected(lat, info, N), info
    h.set_plan_opts(no_small=1, no_three_step=1, no_four_step=1)  # the two-step kernel itself
    mu2 = h.moments(N, R, 5)
    for xw in (1, 2):  # with and without the halo warp
        h.set_plan_opts(no_small=1, halo_warp=xw, no_three_step=1, no_four_step=1)
        assert normwise(h.moments(N, R, 5), ref) < TOL
    h.set_plan_opts(no_small=1, no_two_step=1)
    assert h.plan_info(N, R)["two_step"] == 0
    mu1 = h.moments(N, R, 5)
    assert normwise(mu2, ref) < TOL and normwise(mu1, ref) < TOL


@pytest.mark.parametrize("case", ["2d", "3d_anderson", "peierls"])
def test_direct_mode_matches_oracle_direct(kpm, case):
    """KPM_DIRECT: the paper's own estimator, Eq (19): mu_n = <r|a_n>, N-1 products."""
    lat, N, R = CASES[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    r = ki.rademacher(3, R, lat["D"])
    ref = oracle.moments_direct(H, a, b, r, N)
    h = make(kpm, lat, a, b)
    assert normwise(h.moments_ex(N, R, 3, flags=kpm.KPM_DIRECT), ref) < TOL
    assert normwise(h.moments_ex(N, R, 3, r0=r, flags=kpm.KPM_DIRECT), ref) < TOL


def test_c1_bitwise(kpm):
    """Q4: config c1 is exact in fp64, so the GPU equals the oracle bit for bit."""
    c = ki.CONFIGS["c1"]
    lat = ki.lattice(c)
    H = oracle.lattice_csr(lat)
    ref = oracle.moments_doubling(H, 2.0, 0.0, ki.rademacher(c["seed"], c["R"], lat["D"]), c["N"])
    mu = make(kpm, lat, 2.0, 0.0).moments(c["N"], c["R"], c["seed"])
    assert np.array_equal(mu, ref)
    assert mu[0] == 1.0


@pytest.mark.parametrize("path", ["default", "no_small"])
@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 8, 9])
@pytest.mark.parametrize("R", [1, 2, 3])
def test_small_N_and_R_edges(kpm, N, R, path):
    lat = lat_of(2, (9, 7), W=1.0)
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(9, R, lat["D"]), N)
    mu = make(kpm, lat, a, b, no_small=int(path == "no_small")).moments(N, R, 9)
    assert mu.shape == (N,) and normwise(mu, ref) < TOL


def test_unit_vectors_give_exact_trace_on_gpu(kpm):
    """Q2 through the GPU: R = D unit vectors sqrt(D) e_i (caller start block) give
    (1/D) Tr T_n(H~) of the paper's 10x10x10 lattice."""
    lat = lat_of(3, (10, 10, 10))
    H = oracle.lattice_csr(lat)
    ex = oracle.exact_moments_dense(H, 6.0, 0.0, 128)
    r = np.sqrt(1000.0) * np.eye(1000)
    mu = make(kpm, lat, 6.0, 0.0).moments_ex(128, 1000, 0, r0=r)
    assert np.abs(mu - ex).max() < 1e-12


def test_spectrum_guard(kpm):
    lat = lat_of(2, (16, 16))
    h = make(kpm, lat, 2.0, 0.0)  # a = 2 < spectral radius 4: recursion diverges
    with pytest.raises(kpm.KPMError) as e:
        h.moments(64, 4, 1)
    assert e.value.status == kpm.KPM_ERR_SPECTRUM


def test_raw_sums_and_assemble(kpm):
    lat, N, R = CASES["3d_anderson"]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    h = make(kpm, lat, a, b)
    S = h.moments_ex(N, R, 5, flags=kpm.KPM_RAW_SUMS)
    mu = h.assemble(S, N, R)
    assert np.array_equal(mu, h.moments(N, R, 5))


def test_vector_partition_ranks_sum_to_whole(kpm):
    """P1 host logic on one GPU: per-rank raw sums of a 3-way vector partition add up to the
    1-rank sums (same global vectors), and assemble to the same moments."""
    lat, N, R = CASES["2d_wide"]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    whole = make(kpm, lat, a, b).moments_ex(N, R, 2, flags=kpm.KPM_RAW_SUMS)
    parts = []
    for rank in range(3):
        h = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, dist=(kpm.KPM_PART_VECTORS, rank, 3))
        parts.append(h.moments_ex(N, R, 2, flags=kpm.KPM_RAW_SUMS))
    S = parts[0] + parts[1] + parts[2]
    assert normwise(S, whole) < 1e-13
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(2, R, lat["D"]), N)
    assert normwise(h.assemble(S, N, R), ref) < TOL


def test_dos_matches_oracle(kpm):
    lat = lat_of(2, (32, 32), flux=1 / 8)
    H = oracle.lattice_csr(lat)
    mu = oracle.moments_doubling(H, 4.0, 0.0, ki.rademacher(1, 4, 1024), 256)
    om = np.linspace(-4.5, 4.5, 1001)
    for kern, name in [(kpm.KPM_KERNEL_JACKSON, "jackson"), (kpm.KPM_KERNEL_NONE, "none")]:
        rho = kpm.kpm_dos(mu, 4.0, 0.0, om, kernel=kern)
        ref = oracle.dos(mu, 4.0, 0.0, om, kernel=name)
        assert np.abs(rho - ref).max() < 1e-10 * np.abs(ref).max()


# ---------------------------------------------------------------- row partition (P2)
ROW_CASES = {
    "1d": (lat_of(1, (600,)), 30, 5),
    "2d_simple": (lat_of(2, (37, 29)), 26, 7),
    "2d_tma": (lat_of(2, (64, 40)), 24, 64),
    "2d_peierls_tma": (lat_of(2, (64, 16), flux=1 / 8, W=1.0), 21, 32),
    "3d_simple": (lat_of(3, (13, 11, 9), W=2.0), 22, 6),
    "3d_tma": (lat_of(3, (32, 16, 12), W=2.0), 25, 16),
}


@pytest.mark.parametrize("comm", ["self", "nccl"])
@pytest.mark.parametrize("case", sorted(ROW_CASES))
def test_row_partition_world1_matches_oracle(kpm, case, comm):
    """KPM_PART_ROWS with one rank: slab + ghost planes refreshed after every step (a local
    copy, or NCCL send/recv to itself), moment sums through the NCCL all-reduce."""
    lat, N, R = ROW_CASES[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    r = ki.rademacher(8, R, lat["D"])
    ref, ref_pv = oracle.moments_doubling(H, a, b, r, N, per_vector=True)
    if comm == "self":
        dist = (kpm.KPM_PART_ROWS, 0, 1, kpm.KPM_COMM_SELF)
    else:
        dist = (kpm.KPM_PART_ROWS, 0, 1, kpm.KPM_COMM_NCCL, kpm.kpm_nccl_unique_id())
    h = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"], flux=lat["flux"], dist=dist)
    info = h.plan_info(N, R)
    assert info["two_step"] == 0
    assert info["overlap"] == (info["tma"] == 1 and lat["L"][lat["ndim"] - 1] >= 3)
    mu = h.moments(N, R, 8)
    assert normwise(mu, ref) < TOL
    assert normwise(h.moments_ex(N, R, 8, flags=kpm.KPM_PER_VECTOR), ref_pv) < TOL
    assert np.array_equal(h.moments_ex(N, R, 8, r0=r), mu)  # a_0 ghosts exchanged before the first step
    whole = make(kpm, lat, a, b).moments(N, R, 8)
    assert normwise(mu, whole) < 1e-13
    if info["overlap"]:  # boundary planes + exchange on the comm stream + interior, vs serialised
        h.set_plan_opts(no_overlap=1)
        assert h.plan_info(N, R)["overlap"] == 0
        assert normwise(h.moments(N, R, 8), mu) < 1e-13


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("case", ["1d", "2d_tma", "2d_peierls_tma", "3d_simple", "3d_tma"])
def test_row_partition_local_group_matches_oracle(kpm, case, world, fused):
    """KPM_COMM_LOCAL: `world` slab handles in one process (one GPU) exchange halo planes
    after every step; uneven slabs included.  Same global vectors as one whole lattice.
    fused = 1: the TMA march kernels store their boundary planes straight into the neighbours'
    ghost planes (peer memory, no copy step); fused = 0: plane copies between launches."""
    lat, N, R = ROW_CASES[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(8, R, lat["D"]), N)
    hs = [kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"], flux=lat["flux"],
                                 dist=(kpm.KPM_PART_ROWS, rk, world, kpm.KPM_COMM_LOCAL)) for rk in range(world)]
    hs[0].set_plan_opts(no_fused_halo=int(fused == "0"))
    mu = kpm.kpm_moments_group(hs, N, R, 8)
    assert normwise(mu, ref) < TOL
    st = hs[0].last_stats()
    tma = hs[0].plan_info(N, R)["tma"] == 1
    on = fused == "1" and tma  # the fused halo needs the TMA march kernels
    assert st["fused_halo"] == (st["step_launches"] if on else 0), st
    assert st["halo_copies"] == (2 if on else 2 * (st["step_launches"] + 1)), st  # + the first step's copies


def random_sparse_hermitian(D, deg, seed, cplx):
    """Irregular sparse Hermitian H (random graph, long-range bonds, ragged row lengths)."""
    rng = np.random.default_rng(seed)
    A = np.zeros((D, D), dtype=np.complex128 if cplx else np.float64)
    for i in range(D):
        for j in rng.choice(D, size=int(rng.integers(1, deg + 1)), replace=False):
            v = rng.normal() + (1j * rng.normal() if cplx else 0.0)
            A[i, j] += v
    A = A + A.conj().T
    A[np.diag_indices(D)] = rng.normal(size=D)
    return oracle.csr_from_dense(A)


SPARSE_ROW_CASES = {
    "3d_anderson_csr": lambda: oracle.lattice_csr(lat_of(3, (6, 5, 8), W=2.0)),
    "2d_peierls_csr": lambda: oracle.lattice_csr(lat_of(2, (16, 12), flux=1 / 4)),
    "random_real": lambda: random_sparse_hermitian(150, 5, 3, False),
    "random_complex_wide_rows": lambda: random_sparse_hermitian(97, 12, 4, True),
}


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("case", sorted(SPARSE_ROW_CASES))
def test_csr_row_partition_matches_oracle(kpm, case, world):
    """General-sparse row partition: `world` CSR handles, each with its
    row block + ghost sites gathered from the owners after every step (KPM_COMM_LOCAL, one GPU;
    world 1: KPM_COMM_SELF through kpm_moments), vs the oracle on the same global vectors."""
    H = SPARSE_ROW_CASES[case]()
    a, b = oracle.gershgorin(H)
    b += 0.01 * a
    a *= 1.02
    N, R = 29, 6
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(4, R, H.D), N)
    val = H.val_re + 1j * H.val_im if H.is_complex else H.val_re
    if world == 1:
        h = kpm.kpm_create_csr(H.D, H.rowptr, H.col, val, a, b, dist=(kpm.KPM_PART_ROWS, 0, 1, kpm.KPM_COMM_SELF))
        mu = h.moments(N, R, 4)
        direct = h.moments_ex(N, R, 4, flags=kpm.KPM_DIRECT)
        assert normwise(direct, oracle.moments_direct(H, a, b, ki.rademacher(4, R, H.D), N)) < TOL
    else:
        hs = [kpm.kpm_create_csr(H.D, H.rowptr, H.col, val, a, b,
                                 dist=(kpm.KPM_PART_ROWS, rk, world, kpm.KPM_COMM_LOCAL)) for rk in range(world)]
        assert sum(h.D_local for h in hs) == H.D
        mu = kpm.kpm_moments_group(hs, N, R, 4)
    assert normwise(mu, ref) < TOL


def test_csr_row_partition_nccl_world1(kpm):
    """The NCCL path of the CSR row partition at world 1 (no ghosts; all-reduce of the sums),
    with caller start vectors and per-vector output."""
    H = SPARSE_ROW_CASES["random_real"]()
    a, b = oracle.gershgorin(H)
    N, R = 24, 5
    r = ki.rademacher(2, R, H.D)
    ref, ref_pv = oracle.moments_doubling(H, a, b, r, N, per_vector=True)
    h = kpm.kpm_create_csr(H.D, H.rowptr, H.col, H.val_re, a, b,
                           dist=(kpm.KPM_PART_ROWS, 0, 1, kpm.KPM_COMM_NCCL, kpm.kpm_nccl_unique_id()))
    assert normwise(h.moments(N, R, 2), ref) < TOL
    assert normwise(h.moments_ex(N, R, 2, r0=r), ref) < TOL
    assert normwise(h.moments_ex(N, R, 2, flags=kpm.KPM_PER_VECTOR), ref_pv) < TOL


@pytest.mark.parametrize("vworld", [2, 3])
@pytest.mark.parametrize("case", ["2d_tma", "3d_tma", "3d_simple"])
def test_hybrid_rows_x_vectors_matches_oracle(kpm, case, vworld):
    """Hybrid decomposition: vworld vector groups, each a 2-slab row
    partition (in-process group) over its share of the global vectors; the groups' moments
    combine with weights R_g / R (the doubling transform is linear in the raw sums)."""
    lat, N, R = ROW_CASES[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(8, R, lat["D"]), N)
    mu = np.zeros(N)
    for vg in range(vworld):
        hs = [kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"], flux=lat["flux"],
                                     dist=(kpm.KPM_PART_ROWS, rk, 2, kpm.KPM_COMM_LOCAL, None, vg, vworld))
              for rk in range(2)]
        _, Rg = hs[0].r_local(R)
        assert Rg == kpm.kpm_vector_range(R, vg, vworld)[1]
        mu += Rg / R * kpm.kpm_moments_group(hs, N, R, 8)
    assert normwise(mu, ref) < TOL


def test_hybrid_raw_sums_over_nccl_row_groups(kpm):
    """Row partition over NCCL (world 1 per group) with KPM_RAW_SUMS: the vector groups' raw
    sums add up to the whole estimate through kpm_assemble with the global R."""
    lat, N, R = ROW_CASES["3d_tma"]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(8, R, lat["D"]), N)
    S = np.zeros(N)
    for vg in range(2):
        h = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"], flux=lat["flux"],
                                   dist=(kpm.KPM_PART_ROWS, 0, 1, kpm.KPM_COMM_NCCL, kpm.kpm_nccl_unique_id(), vg, 2))
        S += h.moments_ex(N, R, 8, flags=kpm.KPM_RAW_SUMS)
    assert normwise(h.assemble(S, N, R), ref) < TOL


def test_randomized_shapes_sweep(kpm):
    """Random small lattices (1D/2D/3D, with/without disorder or flux), R, N and (a, b): all
    kernel paths (generic, TMA march, two-step) against the oracle."""
    rng = np.random.default_rng(1234)
    for trial in range(24):
        ndim = int(rng.integers(1, 4))
        if ndim == 1:
            L = (int(rng.integers(3, 400)),)
        elif ndim == 2:
            L = tuple(int(v) for v in rng.choice([4, 6, 16, 32, 64], 2)) if trial % 2 else \
                tuple(int(v) for v in rng.integers(3, 40, 2))
        else:
            L = tuple(int(v) for v in rng.choice([4, 8, 16, 32], 3)) if trial % 2 else \
                tuple(int(v) for v in rng.integers(3, 14, 3))
        flux = 0.0
        if ndim == 2 and rng.random() < 0.4:
            q = int(rng.choice([2, 4, 8]))
            if L[0] % q == 0:
                flux = 1.0 / q
        W = float(rng.choice([0.0, 1.5]))
        R = int(rng.choice([1, 3, 8, 16, 32, 64]))
        N = int(rng.integers(1, 40))
        lat = lat_of(ndim, L, W=W, flux=flux, dseed=trial)
        H = oracle.lattice_csr(lat)
        a, b = oracle.gershgorin(H)
        a *= 1.0 + 0.1 * rng.random()
        ref = oracle.moments_doubling(H, a, b, ki.rademacher(trial, R, lat["D"]), N)
        mu = make(kpm, lat, a, b, no_small=trial % 2).moments(N, R, trial)  # both launch paths
        assert normwise(mu, ref) < TOL, (trial, ndim, L, flux, W, R, N)


FIRST_CASES = {
    "2d_ragged_tile": (lat_of(2, (70, 9), W=1.0), 12, 6),          # L0 not a multiple of the 64-site tile
    "2d_peierls_lanes_masked": (lat_of(2, (48, 12), flux=1 / 4), 9, 20),  # 20 lanes: 16-lane groups, masked
    "3d_ragged": (lat_of(3, (20, 18, 7), W=2.0), 10, 5),            # 16 x 16 tiles, ragged in x and y
    "3d_L2": (lat_of(3, (2, 3, 2)), 7, 3),                          # one tile, halos wrap onto the tile
    "3d_lane_groups": (lat_of(3, (16, 16, 6)), 8, 40),              # 20 lanes: 8-lane groups, masked
}


@pytest.mark.parametrize("case", sorted(FIRST_CASES))
@pytest.mark.parametrize("first_tile", [0, 1])
def test_first_step_tile_kernel(kpm, case, first_tile):
    """a_0 hashed once per element into a plane ring (kpm_first.cuh) vs the generic first step:
    both equal the oracle; N = 3 puts the odd-N tail <a_1|a_1> into the first launch."""
    lat, N, R = FIRST_CASES[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    b += 0.03 * a
    a *= 1.04
    r = ki.rademacher(17, R, lat["D"])
    for n in (N, 3, 2):
        ref, ref_pv = oracle.moments_doubling(H, a, b, r, n, per_vector=True)
        h = make(kpm, lat, a, b, no_small=1, no_first_tile=int(not first_tile))
        assert normwise(h.moments(n, R, 17), ref) < TOL
        assert normwise(h.moments_ex(n, R, 17, flags=kpm.KPM_PER_VECTOR), ref_pv) < TOL
    # local moments (unit start vectors) and a one-slab row partition through the same kernel
    sites = [0, lat["D"] - 1, lat["D"] // 3]
    h = make(kpm, lat, a, b, no_small=1, no_first_tile=int(not first_tile))
    assert normwise(h.moments_local(N, sites), oracle.local_moments(H, a, b, sites, N)) < TOL
    hr = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"], flux=lat["flux"],
                                dist=(kpm.KPM_PART_ROWS, 0, 1, kpm.KPM_COMM_SELF))
    hr.set_plan_opts(no_first_tile=int(not first_tile))
    assert normwise(hr.moments(N, R, 17), oracle.moments_doubling(H, a, b, r, N)) < TOL


QUAD_CASES = {
    "2d_R64": TMA_CASES["2d_R64"],
    "2d_anderson_R16": TMA_CASES["2d_anderson_R16"],
    "2d_peierls_R32": TMA_CASES["2d_peierls_R32"],
    # 2 lane groups x 3 pencils, 20 rows over the grid: ragged segments, on-site + Peierls
    "2d_peierls_anderson_R16": (lat_of(2, (192, 20), flux=1 / 8, W=1.0), 30, 16),
    # 4 lanes per site (8 real / 4 complex vectors: one GPU's share of c2 at 8 GPUs): 128-site tiles,
    # the a_{n-1} halo padded to 4 sites; no three-step kernel, so a remainder of 3 = single + pair
    "2d_R8_four_lanes": TMA_CASES["2d_R8_four_lanes"],
    "2d_anderson_R8_four_lanes": TMA_CASES["2d_anderson_R8_four_lanes"],
    "2d_peierls_R4_four_lanes": (lat_of(2, (128, 16), flux=1 / 8, W=1.0), 41, 4),
}


@pytest.mark.parametrize("case", list(QUAD_CASES))
@pytest.mark.parametrize("N", [9, 10, 11, 12, 13, 14, 15, 16, 17, 40, 41])
def test_four_step_kernel(kpm, case, N):
    """2D: four recursion steps per launch (kpm_quad.cuh, the default for 2D tiles of >= 8 lanes), the step-count
    remainder first (a three-step launch, a pair or a single step), odd-N tail inside the last
    launch: the oracle's moments, per vector too, bitwise equal to the run from the same a_0."""
    lat, _, R = QUAD_CASES[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    b += 0.01 * a
    a *= 1.02
    r = ki.rademacher(23, R, lat["D"])
    ref, ref_pv = oracle.moments_doubling(H, a, b, r, N, per_vector=True)
    h = make(kpm, lat, a, b, no_small=1)
    info = h.plan_info(N, R)
    nsteps = N // 2 - 1
    tri_ok = info["TL"] >= 8  # the three-step kernel needs tiles of >= 8 lanes
    assert info["four_step"] == (1 if nsteps >= 4 else 0), info
    assert info["ks"] == (4 if nsteps >= 4 else (3 if tri_ok else 0)), info
    mu = h.moments(N, R, 23)
    assert normwise(mu, ref) < TOL
    assert normwise(h.moments_ex(N, R, 23, flags=kpm.KPM_PER_VECTOR), ref_pv) < TOL
    assert np.array_equal(h.moments_ex(N, R, 23, r0=r), mu)
    assert np.array_equal(h.moments(N, R, 23), mu), "not deterministic"
    _, launches, _ = h.last_timing()
    rem = nsteps % 4
    assert launches == nsteps // 4 + (0 if rem == 0 else (2 if rem == 3 and not tri_ok else 1)), (launches, nsteps)


@pytest.mark.parametrize("case", ["2d_R64", "2d_anderson_R16", "2d_peierls_R32", "2d_R8_four_lanes"])
@pytest.mark.parametrize("N", [7, 8, 9, 10, 11, 12, 13, 15, 16, 40])
def test_three_step_kernel(kpm, case, N):
    """2D: three recursion steps per launch (kpm_tri.cuh), the step-count remainder as a leading
    pair or single step, odd-N tail inside the last launch: the oracle's moments, per vector too,
    and the same launch count the schedule implies.  (4-lane tiles keep the two-step kernel.)"""
    lat, _, R = TMA_CASES[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    b += 0.01 * a
    a *= 1.02
    r = ki.rademacher(19, R, lat["D"])
    ref, ref_pv = oracle.moments_doubling(H, a, b, r, N, per_vector=True)
    h = make(kpm, lat, a, b, no_small=1, no_four_step=1)  # (the plan for 2D tiles of >= 8 lanes without kpm_quad.cuh)
    info = h.plan_info(N, R)
    nsteps = N // 2 - 1
    tri = info["two_step"] == 1 and info["TL"] >= 8 and nsteps >= 3
    assert info["ks"] == (3 if tri else 0), info
    mu = h.moments(N, R, 19)
    assert normwise(mu, ref) < TOL
    assert normwise(h.moments_ex(N, R, 19, flags=kpm.KPM_PER_VECTOR), ref_pv) < TOL
    assert np.array_equal(h.moments_ex(N, R, 19, r0=r), mu)
    assert np.array_equal(h.moments(N, R, 19), mu), "not deterministic"
    if tri:
        _, launches, _ = h.last_timing()
        rem = nsteps % 3
        assert launches == nsteps // 3 + (1 if rem else 0), (launches, nsteps)


def random_sparse_k(D, K, seed, cplx):
    """Random Hermitian H with at most K stored entries per row (ELL width K): a random symmetric
    bond pattern of degree <= K - 1 plus the diagonal."""
    rng = np.random.default_rng(seed)
    A = np.zeros((D, D), dtype=np.complex128 if cplx else np.float64)
    deg = np.zeros(D, dtype=int)
    for i in rng.permutation(D):
        for j in rng.choice(D, size=K, replace=False):
            if i != j and deg[i] < K - 1 and deg[j] < K - 1 and A[i, j] == 0:
                v = rng.normal() + (1j * rng.normal() if cplx else 0.0)
                A[i, j], A[j, i] = v, np.conj(v)
                deg[i] += 1
                deg[j] += 1
    A[np.diag_indices(D)] = rng.normal(size=D)
    return oracle.csr_from_dense(A)


@pytest.mark.parametrize("K", [3, 5, 9, 14, 16])
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("R", [7, 64])
def test_ell_kernel_entry_widths(kpm, K, cplx, R):
    """The staged ELL kernel for every stored width KP = 4, 8 (256-row tiles), 12, 16 (K rounded up to
    a multiple of 4, padding entries (row, 0)), real and complex, ragged last tile, 1-2 lane groups."""
    H = random_sparse_k(1300, K, 11 + K, cplx)
    a, b = oracle.gershgorin(H)
    N = 22
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(6, R, H.D), N)
    val = H.val_re + 1j * H.val_im if H.is_complex else H.val_re
    h = kpm.kpm_create_csr(H.D, H.rowptr, H.col, val, a, b)
    h.set_plan_opts(no_small=1)
    assert normwise(h.moments(N, R, 6), ref) < TOL
    assert np.array_equal(h.moments(N, R, 6), h.moments(N, R, 6)), "not deterministic"
