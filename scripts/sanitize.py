"""Small parity cases for compute-sanitizer (memcheck / racecheck / synccheck): the three-step
rings (2D, on-site, Peierls), the two-step rings (4- and 16-lane tiles, the halo warp), the 3D
dense-box march, the in-place a_{n+1}-over-a_{n-1} single steps, the fused peer-plane stores of an
in-process slab group, the ELL kernel with bulk-staged entries, the first-step plane ring, and the
finish/assemble kernels -- each checked against the oracle.
usage: compute-sanitizer --tool memcheck python scripts/sanitize.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kpm_inputs as ki  # noqa: E402
import oracle  # noqa: E402
from paper_1105_5481_b200 import kpm  # noqa: E402


def lat_of(ndim, L, W=0.0, flux=0.0):
    L = tuple(L) + (1,) * (3 - len(L))
    D = L[0] * L[1] * L[2]
    return dict(ndim=ndim, L=L, D=D, t=-1.0, onsite=ki.anderson_onsite(5, D, W) if W else None, flux=flux)


def check(name, mu, ref):
    err = np.abs(mu - ref).max() / np.abs(ref).max()
    print(f"{name}: {err:.2e}", flush=True)
    assert err < 1e-10, name


cases = [
    ("three_step_16_lanes_onsite", lat_of(2, (128, 12), W=1.0), 16, 32, {}),
    ("three_step_peierls", lat_of(2, (128, 9), flux=1 / 8), 17, 32, {}),
    ("two_step_16_lanes", lat_of(2, (128, 12), W=1.0), 14, 32, {"no_three_step": 1}),
    ("two_step_4_lanes", lat_of(2, (128, 10)), 14, 8, {}),
    ("two_step_peierls_halo_warp", lat_of(2, (64, 8), flux=1 / 8), 13, 32, {"no_three_step": 1}),
    ("single_steps_in_place", lat_of(2, (64, 8), W=1.0), 12, 16, {"no_two_step": 1}),
    ("box3_march", lat_of(3, (16, 8, 6), W=2.0), 12, 32, {}),
    ("generic_first_and_steps", lat_of(3, (9, 7, 5), W=1.0), 11, 3, {"no_tma": 1, "no_first_tile": 1}),
]
for name, lat, N, R, opts in cases:
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(3, R, lat["D"]), N)
    h = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"], flux=lat["flux"])
    h.set_plan_opts(no_small=1, **opts)
    check(name, h.moments(N, R, 3), ref)
    h.close()
# ELL kernel
lat = lat_of(3, (12, 10, 8), W=2.0)
H = oracle.lattice_csr(lat)
a, b = oracle.gershgorin(H)
h = kpm.kpm_create_csr(H.D, H.rowptr, H.col, H.val_re, a, b)
h.set_plan_opts(no_small=1)
check("ell", h.moments(12, 16, 3), oracle.moments_doubling(H, a, b, ki.rademacher(3, 16, H.D), 12))
# fused peer-plane stores: 3 slabs in one process, one device
lat = lat_of(3, (16, 8, 9), W=2.0)
H = oracle.lattice_csr(lat)
a, b = oracle.gershgorin(H)
hs = [kpm.kpm_create_stencil(3, lat["L"], -1.0, a, b, onsite=lat["onsite"],
                             dist=(kpm.KPM_PART_ROWS, rk, 3, kpm.KPM_COMM_LOCAL)) for rk in range(3)]
mu = kpm.kpm_moments_group(hs, 12, 16, 3)
assert hs[0].last_stats()["fused_halo"] > 0
check("fused_halo_group", mu, oracle.moments_doubling(H, a, b, ki.rademacher(3, 16, H.D), 12))
print("sanitize cases done")
