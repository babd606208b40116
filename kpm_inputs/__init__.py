"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the Kernel Polynomial Method (no rescaling,
no recursion, no moments, no kernels, no DoS).  It only produces the raw
inputs of the paper's workloads, deterministically from integer seeds:

* the random start vectors |r> = sum_i xi_{r,i} |i> of Eq (15)
  (Sec II-A.3) with iid real xi of mean 0 and variance 1
  (Eq 14).  Reading X1 of DESIGN.md: Rademacher +-1 drawn
  from a counter-based hash so that the GPU can regenerate the same numbers
  on the fly (the paper draws them inside its kernel);
* the Anderson on-site energies eps_i (reading X14);
* the lattice descriptors of BASELINE.json's five configs (the paper's model
  is the periodic nearest-neighbour lattice with t = -1).

The counter-based generator (splitmix64 finaliser) is specified here in
numpy; the CUDA library implements the same specification independently
(paper_1105_5481_b200/csrc/kpm_rng.cuh), and a GPU test checks the two
agree bit for bit.
"""
from __future__ import annotations

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def mix64(z):
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64).copy()
    z ^= z >> np.uint64(30)
    z *= np.uint64(0xBF58476D1CE4E5B9)
    z ^= z >> np.uint64(27)
    z *= np.uint64(0x94D049BB133111EB)
    z ^= z >> np.uint64(31)
    return z


def mix64_int(z: int) -> int:
    """The same finaliser on a Python int (used for key derivation)."""
    z &= M64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & M64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & M64
    z ^= z >> 31
    return z


def vector_key(seed: int) -> int:
    return mix64_int((seed + GOLDEN) & M64)


def rademacher(seed: int, R: int, D: int, r_offset: int = 0, D_total: int | None = None,
               i_offset: int = 0) -> np.ndarray:
    """Start vectors xi[r, i] in {-1, +1}, shape (R, D), vector-major (reading X19).

    xi = 1 - 2 * (mix64(key ^ ctr) >> 63), key = mix64(seed + GOLDEN),
    ctr = (r_offset + r) * D_total + (i_offset + i)  (global indices, so the
    vector set does not depend on how vectors or rows are partitioned).
    """
    if D_total is None:
        D_total = D
    key = np.uint64(vector_key(seed))
    out = np.empty((R, D), dtype=np.float64)
    i = np.arange(i_offset, i_offset + D, dtype=np.uint64)
    for r in range(R):
        ctr = np.uint64((r_offset + r) * D_total) + i
        bit = mix64(key ^ ctr) >> np.uint64(63)
        out[r] = 1.0 - 2.0 * bit.astype(np.float64)
    return out


def anderson_onsite(disorder_seed: int, D: int, W: float) -> np.ndarray:
    """On-site energies eps_i = W (u_i - 1/2), u_i uniform in [0, 1) (reading X14)."""
    key = np.uint64(vector_key(disorder_seed))
    i = np.arange(D, dtype=np.uint64)
    u = (mix64(key ^ i) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return W * (u - 0.5)


# BASELINE.json configs, made concrete (readings X12-X15 in DESIGN.md).
CONFIGS = {
    "c1": dict(name="1D chain L=1024", ndim=1, L=(1024, 1, 1), t=-1.0, W=0.0, disorder_seed=0,
               flux=0.0, N=128, R=8, seed=1),
    "c2": dict(name="2D square 512x512", ndim=2, L=(512, 512, 1), t=-1.0, W=0.0, disorder_seed=0,
               flux=0.0, N=1024, R=64, seed=2),
    "c3": dict(name="3D Anderson 128^3 W=2", ndim=3, L=(128, 128, 128), t=-1.0, W=2.0,
               disorder_seed=103, flux=0.0, N=2048, R=128, seed=3),
    "c4": dict(name="2D Peierls 1024x1024 phi=1/8", ndim=2, L=(1024, 1024, 1), t=-1.0, W=0.0,
               disorder_seed=0, flux=0.125, N=4096, R=256, seed=4),
    "c5": dict(name="3D Anderson 512^3 W=2", ndim=3, L=(512, 512, 512), t=-1.0, W=2.0,
               disorder_seed=105, flux=0.0, N=1024, R=32, seed=5),
    # the paper's own dense-H experiment (Exp IV.C largest point: H_SIZE = 4096,
    # R*S = 14*128 = 1792, N = 128) on its model lattice (3D cubic, t = -1, periodic; 16^3 = 4096)
    "pd": dict(name="paper Exp IV.C: dense H_SIZE=4096 (3D 16^3), RS=1792, N=128", ndim=3, L=(16, 16, 16),
               t=-1.0, W=0.0, disorder_seed=0, flux=0.0, N=128, R=1792, seed=6, format="dense"),
}


def lattice_dense(lat: dict) -> np.ndarray:
    """The lattice Hamiltonian as a dense row-major D x D array (input construction for
    kpm_create_dense; real lattices only)."""
    rowptr, col, val = lattice_csr(lat)
    assert not np.iscomplexobj(val), "dense input: real H only"
    D = len(rowptr) - 1
    H = np.zeros((D, D))
    rows = np.repeat(np.arange(D), np.diff(rowptr))
    np.add.at(H, (rows, col), val)
    return H


def num_sites(L) -> int:
    return int(L[0]) * int(L[1]) * int(L[2])


def lattice(cfg: dict, **overrides) -> dict:
    """Concrete lattice descriptor for a config: dims, hopping, on-site array, flux."""
    c = dict(cfg)
    c.update(overrides)
    L = tuple(int(v) for v in c["L"])
    D = num_sites(L)
    onsite = anderson_onsite(c["disorder_seed"], D, c["W"]) if c.get("W", 0.0) != 0.0 else None
    return dict(ndim=int(c["ndim"]), L=L, D=D, t=float(c["t"]), onsite=onsite,
                flux=float(c.get("flux", 0.0)))


def lattice_csr(lat: dict):
    """The lattice Hamiltonian of a descriptor as CSR arrays (rowptr int64, col int32, val
    float64 or complex128), built with numpy for feeding kpm_create_csr.  Input
    construction only (the same H the stencil descriptor defines: periodic nearest-neighbour
    bonds t, Peierls phase e^{+i 2 pi phi x} on the y-bond (x,y)->(x,y+1), on-site eps)."""
    ndim, L = lat["ndim"], tuple(int(v) for v in lat["L"])
    D = L[0] * L[1] * L[2]
    idx = np.arange(D, dtype=np.int64)
    c = [idx % L[0], (idx // L[0]) % L[1], idx // (L[0] * L[1])]
    cols, vals = [], []
    flux, t = float(lat.get("flux", 0.0)), float(lat["t"])
    if lat.get("onsite") is not None:
        cols.append(idx)
        vals.append(np.asarray(lat["onsite"], dtype=np.float64).astype(np.complex128))
    for d in range(ndim):
        stride = [1, L[0], L[0] * L[1]][d]
        for s in (+1, -1):
            nd = (c[d] + s) % L[d]
            j = idx + (nd - c[d]) * stride
            # bond (u -> u + e_d) carries H[u+e_d][u] = t e^{i theta(u)}, theta = 2 pi phi x_u on y-bonds
            theta = 2.0 * np.pi * flux * c[0] if d == 1 else np.zeros(D)
            h = t * np.exp(-1j * theta) if s == +1 else t * np.exp(1j * theta)
            cols.append(j)
            vals.append(h)
    col = np.stack(cols, axis=1).astype(np.int32)
    val = np.stack(vals, axis=1)
    rowptr = np.arange(D + 1, dtype=np.int64) * col.shape[1]
    if flux == 0.0:
        val = val.real.copy()
    return rowptr, col.ravel(), val.ravel()
