"""CPU oracle for the KPM hot path (arxiv 1105.5481).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  It shares no
code with the CUDA path (paper_1105_5481_b200/) and neither imports the other;
the only shared module is kpm_inputs (seeded inputs, no method arithmetic).

Layout
  kpm_oracle.c   O1-O3 in plain C (CSR build, Gerschgorin, direct Eq 17-19,
                 doubling); loaded through ctypes below.
  exact.py       O4-O7 in numpy/scipy (exact traces Eq 13, analytic spectra,
                 Jackson kernel, DoS Eq 6, closed-form DoS).

Pins: every function here is checked in tests/test_oracle_*.py against what the
paper and the mathematics fix.  Functions
with no independent pin are listed there as "parity unpinned"; at present
there are none in this package.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kpm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile kpm_oracle.c into liboracle.so (plain gcc + OpenMP, portable flags)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=gnu11", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32, f64 = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        lib.oracle_num_threads.restype = ctypes.c_int
        lib.oracle_lattice_nnz.restype = i64
        lib.oracle_lattice_nnz.argtypes = [ctypes.c_int, P, ctypes.c_int]
        lib.oracle_build_lattice_csr.restype = ctypes.c_int
        lib.oracle_build_lattice_csr.argtypes = [ctypes.c_int, P, f64, P, f64, P, P, P, P]
        lib.oracle_gershgorin.restype = None
        lib.oracle_gershgorin.argtypes = [i64, P, P, P, P, f64, P, P]
        for fn in (lib.oracle_moments_direct, lib.oracle_moments_doubling):
            fn.restype = ctypes.c_int
            fn.argtypes = [i64, P, P, P, P, ctypes.c_int, f64, f64, i64, P, ctypes.c_int, P, P]
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return int(_load().oracle_num_threads())


class CSR:
    """H in CSR form: rowptr int64[D+1], col int32[nnz], val complex or real."""

    def __init__(self, D, rowptr, col, val_re, val_im, is_complex):
        self.D = int(D)
        self.rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
        self.col = np.ascontiguousarray(col, dtype=np.int32)
        self.val_re = np.ascontiguousarray(val_re, dtype=np.float64)
        self.val_im = np.ascontiguousarray(val_im, dtype=np.float64)
        self.is_complex = bool(is_complex)

    @property
    def nnz(self):
        return int(self.rowptr[-1])

    def dense(self) -> np.ndarray:
        """Dense H (test-only, tiny D)."""
        H = np.zeros((self.D, self.D), dtype=np.complex128 if self.is_complex else np.float64)
        for i in range(self.D):
            for k in range(self.rowptr[i], self.rowptr[i + 1]):
                v = self.val_re[k] + (1j * self.val_im[k] if self.is_complex else 0.0)
                H[i, self.col[k]] += v
        return H


def lattice_csr(lat: dict) -> CSR:
    """O1: the lattice Hamiltonian as CSR, built by kpm_oracle.c."""
    lib = _load()
    L = np.asarray(lat["L"], dtype=np.int64)
    onsite = lat.get("onsite")
    if onsite is not None:
        onsite = np.ascontiguousarray(onsite, dtype=np.float64)
    nnz = int(lib.oracle_lattice_nnz(int(lat["ndim"]), _ptr(L), int(onsite is not None)))
    D = int(L.prod())
    rowptr = np.zeros(D + 1, dtype=np.int64)
    col = np.zeros(nnz, dtype=np.int32)
    vre = np.zeros(nnz, dtype=np.float64)
    vim = np.zeros(nnz, dtype=np.float64)
    rc = lib.oracle_build_lattice_csr(int(lat["ndim"]), _ptr(L), float(lat["t"]), _ptr(onsite),
                                      float(lat.get("flux", 0.0)), _ptr(rowptr), _ptr(col),
                                      _ptr(vre), _ptr(vim))
    if rc != 0:
        raise ValueError("oracle_build_lattice_csr failed")
    return CSR(D, rowptr, col, vre, vim, lat.get("flux", 0.0) != 0.0)


def csr_from_dense(H: np.ndarray, keep_zeros: bool = False) -> CSR:
    """CSR of an arbitrary dense Hermitian H (test-only helper); keep_zeros stores all D^2
    entries (the dense variant's arithmetic, for the CPU baseline of the dense config)."""
    D = H.shape[0]
    rows, cols = np.nonzero(np.ones_like(H, dtype=bool) if keep_zeros else H)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    rowptr = np.zeros(D + 1, dtype=np.int64)
    np.add.at(rowptr, rows + 1, 1)
    rowptr = np.cumsum(rowptr)
    vals = H[rows, cols]
    return CSR(D, rowptr, cols, np.real(vals), np.imag(vals) if np.iscomplexobj(H) else
               np.zeros(len(vals)), np.iscomplexobj(H))


def gershgorin(H: CSR, eps: float = 0.0):
    """Eq (8)-(9): (a, b) = (alpha_-, alpha_+) from Gerschgorin bounds."""
    a = ctypes.c_double()
    b = ctypes.c_double()
    _load().oracle_gershgorin(H.D, _ptr(H.rowptr), _ptr(H.col), _ptr(H.val_re), _ptr(H.val_im),
                              float(eps), ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def _moments(fn, H: CSR, a, b, r, N, per_vector):
    r = np.ascontiguousarray(r, dtype=np.float64)
    R, D = r.shape
    assert D == H.D
    mu = np.zeros(N, dtype=np.float64)
    pv = np.zeros((R, N), dtype=np.float64) if per_vector else None
    rc = fn(H.D, _ptr(H.rowptr), _ptr(H.col), _ptr(H.val_re), _ptr(H.val_im), int(H.is_complex),
            float(a), float(b), R, _ptr(r), int(N), _ptr(mu), _ptr(pv))
    if rc != 0:
        raise ValueError(f"oracle moments failed rc={rc}")
    return (mu, pv) if per_vector else mu


def moments_direct(H: CSR, a, b, r, N, per_vector=False):
    """O2: Eq (17)-(19) for start vectors r (R, D); mu[N] (and (R, N) per vector)."""
    return _moments(_load().oracle_moments_direct, H, a, b, r, N, per_vector)


def moments_doubling(H: CSR, a, b, r, N, per_vector=False):
    """O3: doubling identities, floor(N/2) applications of H~; the GPU parity target."""
    return _moments(_load().oracle_moments_doubling, H, a, b, r, N, per_vector)


def local_moments(H: CSR, a, b, sites, N):
    """Local moments mu_n^(i) = <i|T_n(H~)|i> (the local DoS of site i; SURVEY.md 8(f)
    NEXT-1): O3 with the unit start vectors e_i, whose per-vector moments are
    (1/D) <i|T_n(H~)|i>, times D.  Returns (len(sites), N)."""
    sites = np.asarray(sites, dtype=np.int64)
    r = np.zeros((len(sites), H.D))
    r[np.arange(len(sites)), sites] = 1.0
    _, pv = moments_doubling(H, a, b, r, N, per_vector=True)
    return pv * H.D


from .exact import (chebyshev_nodes, dos, dos_closed_1d, dos_closed_2d,  # noqa: E402,F401
                    exact_moments_dense, exact_moments_from_eigs, green, green_closed_1d,
                    harper_spectrum, jackson, kernel_coeffs, lattice_spectrum, moment_stats)
