"""Thin ctypes binding of libkpm.so (include/kpm.h): argument marshalling only.

Every step of the method runs in the CUDA kernels behind the C ABI; nothing
here computes moments.  If libkpm.so is missing this module raises on import
(there is no CPU fallback).  Names follow the C ABI: kpm_create_stencil,
kpm_create_csr, kpm_create_ell, kpm_gershgorin_stencil, kpm_gershgorin_csr,
kpm_moments, kpm_moments_ex, kpm_moments_local, kpm_assemble, kpm_dos, kpm_dos_ex,
kpm_green, kpm_damping, kpm_moment_stats, kpm_workspace_size,
kpm_set_workspace, kpm_set_stream, kpm_last_timing, kpm_step_bytes,
kpm_destroy, kpm_last_error, kpm_version.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkpm.so")
LIB_EXP_PATH = os.path.join(_HERE, "libkpm_exp.so")  # + the experimental (slower) kernels
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                      "g.build()'` (nvcc, sm_100a).  There is no CPU fallback.")

(KPM_OK, KPM_ERR_INVALID_ARG, KPM_ERR_OOM, KPM_ERR_CUDA, KPM_ERR_UNSUPPORTED, KPM_ERR_SPECTRUM, KPM_ERR_NCCL,
 KPM_ERR_COMM) = range(8)
KPM_REAL64, KPM_COMPLEX128 = 0, 1
KPM_KERNEL_JACKSON, KPM_KERNEL_NONE, KPM_KERNEL_LORENTZ, KPM_KERNEL_FEJER = 0, 1, 2, 3
KPM_LORENTZ_DEFAULT_LAMBDA = 4.0
KPM_PER_VECTOR, KPM_DIRECT, KPM_DEVICE_OUT, KPM_RAW_SUMS, KPM_DEVICE_IN, KPM_LOCAL = 1, 2, 4, 8, 16, 32
KPM_PART_NONE, KPM_PART_VECTORS, KPM_PART_ROWS = 0, 1, 2
KPM_COMM_SELF, KPM_COMM_NCCL, KPM_COMM_LOCAL, KPM_COMM_IPC = 0, 1, 2, 3

EXPORTS = ["kpm_create_stencil", "kpm_create_csr", "kpm_create_ell", "kpm_gershgorin_stencil",
           "kpm_gershgorin_csr", "kpm_set_stream", "kpm_workspace_size", "kpm_set_workspace",
           "kpm_moments", "kpm_moments_ex", "kpm_assemble", "kpm_dos", "kpm_last_timing",
           "kpm_step_bytes", "kpm_plan_info", "kpm_vector_range", "kpm_slab_range", "kpm_nccl_unique_id",
           "kpm_moments_group", "kpm_ipc_unique_name", "kpm_dos_ex", "kpm_green", "kpm_damping", "kpm_moment_stats", "kpm_moments_local", "kpm_create_dense",
           "kpm_gershgorin_dense", "kpm_csr_partition", "kpm_last_stats", "kpm_set_plan_opts",
           "kpm_step_traffic", "kpm_destroy", "kpm_last_error", "kpm_version"]


class kpm_stencil_desc(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int32), ("L", ctypes.c_int64 * 3), ("t", ctypes.c_double),
                ("onsite", ctypes.c_void_p), ("flux", ctypes.c_double)]


class kpm_plan_opts(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "no_small", "no_tma", "no_two_step", "no_box3", "tma_lanes", "halo_warp", "ell_generic", "no_overlap",
        "no_fused_halo", "contiguous", "experimental", "exp_param", "two_step_ctas",
        "no_pdl", "no_first_tile", "no_three_step", "no_zorder", "no_four_step")] + [("reserved", ctypes.c_int32 * 2)]


PLAN_OPTS = [f[0] for f in kpm_plan_opts._fields_ if f[0] != "reserved"]
EXP_3D_TWO_STEP, EXP_KSTEP, EXP_PERSIST = 1, 2, 3  # kpm_plan_opts.experimental


class kpm_dist(ctypes.Structure):
    _fields_ = [("partition", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("comm", ctypes.c_int32), ("nccl_id", ctypes.c_void_p), ("vrank", ctypes.c_int32),
                ("vworld", ctypes.c_int32), ("ipc_name", ctypes.c_char_p)]


_P, _i32, _i64, _u32, _u64, _f64, _sz = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32,
                                         ctypes.c_uint64, ctypes.c_double, ctypes.c_size_t)
_SIG = {
    "kpm_create_stencil": [ctypes.POINTER(kpm_stencil_desc), _f64, _f64, _i32, ctypes.POINTER(kpm_dist), _P],
    "kpm_create_csr": [_i64, _P, _P, _P, _i32, _f64, _f64, _i32, ctypes.POINTER(kpm_dist), _P],
    "kpm_create_ell": [_i64, _i32, _P, _P, _i32, _f64, _f64, _i32, ctypes.POINTER(kpm_dist), _P],
    "kpm_csr_partition": [_i64, _P, _P, _i32, _i32, _P, _P, _P, _P],
    "kpm_last_stats": [_P, _P],
    "kpm_gershgorin_stencil": [ctypes.POINTER(kpm_stencil_desc), _f64, _P, _P],
    "kpm_gershgorin_csr": [_i64, _P, _P, _P, _i32, _f64, _P, _P],
    "kpm_set_stream": [_P, _P],
    "kpm_workspace_size": [_P, _i32, _i64, _u32, _P],
    "kpm_set_workspace": [_P, _P, _sz],
    "kpm_moments": [_P, _i32, _i64, _u64, _P],
    "kpm_moments_ex": [_P, _i32, _i64, _u64, _P, _u32, _P],
    "kpm_assemble": [_P, _P, _i32, _i64, _i64, _u32, _P],
    "kpm_vector_range": [_i64, _i32, _i32, _P, _P],
    "kpm_dos": [_P, _i32, _i32, _f64, _f64, _P, _i64, _P, _i32],
    "kpm_dos_ex": [_P, _i32, _i32, _f64, _f64, _f64, _P, _i64, _P, _i32],
    "kpm_green": [_P, _i32, _i32, _f64, _f64, _f64, _P, _i64, _P, _i32],
    "kpm_damping": [_i32, _i32, _f64, _P, _i32],
    "kpm_moment_stats": [_P, _i64, _i32, _P, _P, _i32],
    "kpm_create_dense": [_i64, _P, _i32, _f64, _f64, _i32, ctypes.POINTER(kpm_dist), _P],
    "kpm_gershgorin_dense": [_i64, _P, _i32, _f64, _P, _P],
    "kpm_moments_local": [_P, _i32, _P, _i64, _P],
    "kpm_last_timing": [_P, _P, _P, _P],
    "kpm_step_bytes": [_P, _P],
    "kpm_plan_info": [_P, _i32, _i64, _u32, _P],
    "kpm_slab_range": [_i64, _i32, _i32, _P, _P],
    "kpm_nccl_unique_id": [_P],
    "kpm_ipc_unique_name": [_P],
    "kpm_moments_group": [_P, _i32, _i32, _i64, _u64, _P],
    "kpm_set_plan_opts": [_P, ctypes.POINTER(kpm_plan_opts)],
    "kpm_step_traffic": [_P, _P],
}


def _load(path):
    lib = ctypes.CDLL(path)
    for name, args in _SIG.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int32
    lib.kpm_destroy.argtypes = [_P]
    lib.kpm_destroy.restype = None
    lib.kpm_last_error.restype = ctypes.c_char_p
    lib.kpm_version.restype = ctypes.c_char_p
    return lib


_lib = _load(LIB_PATH)
_lib_default = _lib
_lib_exp = None


def use_experimental(on: bool = True):
    """Route the handles created from now on to libkpm_exp.so (the same library plus the
    experimental kernels of kpm_plan_opts.experimental), or back to libkpm.so.  A handle keeps
    the library it was created with."""
    global _lib, _lib_exp
    if on:
        if _lib_exp is None:
            if not os.path.exists(LIB_EXP_PATH):
                raise ImportError(f"{LIB_EXP_PATH} is missing (built by __graft_entry__.build())")
            _lib_exp = _load(LIB_EXP_PATH)
        _lib = _lib_exp
    else:
        _lib = _lib_default


class KPMError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"kpm status {status}: {msg}")
        self.status = status


def _check(st, lib=None):
    if st != KPM_OK:
        raise KPMError(st, (lib or _lib).kpm_last_error().decode())


def _ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def kpm_last_error() -> str:
    return _lib.kpm_last_error().decode()


def kpm_version() -> str:
    return _lib.kpm_version().decode()


def _desc(ndim, L, t, onsite, flux):
    L = tuple(int(v) for v in L) + (1,) * (3 - len(L))
    on = None if onsite is None else np.ascontiguousarray(onsite, dtype=np.float64)
    d = kpm_stencil_desc(int(ndim), (ctypes.c_int64 * 3)(*L), float(t),
                         None if on is None else on.ctypes.data, float(flux))
    return d, on


def _dist(dist):
    """dist: None, (partition, rank, world) or (partition, rank, world, comm[, nccl_id bytes[, vrank,
    vworld]]) -- the last two: hybrid rows x vectors (row partitions only)."""
    if dist is None:
        return None, None
    part, rank, world = dist[:3]
    comm = dist[3] if len(dist) > 3 else KPM_COMM_SELF
    nid = dist[4] if len(dist) > 4 else None
    vrank, vworld = (int(dist[5]), int(dist[6])) if len(dist) > 6 else (0, 0)
    if comm == KPM_COMM_IPC:  # dist[4]: the shared-segment name (kpm_ipc_unique_name)
        name = nid.encode() if isinstance(nid, str) else bytes(nid)
        st = kpm_dist(int(part), int(rank), int(world), int(comm), None, vrank, vworld, name)
        return ctypes.byref(st), (st, name)
    keep = ctypes.create_string_buffer(bytes(nid), 128) if nid is not None else None
    st = kpm_dist(int(part), int(rank), int(world), int(comm), ctypes.cast(keep, ctypes.c_void_p) if keep else None,
                  vrank, vworld, None)
    return ctypes.byref(st), (st, keep)


def kpm_gershgorin_stencil(ndim, L, t, onsite=None, flux=0.0, eps=0.0):
    d, _keep = _desc(ndim, L, t, onsite, flux)
    a, b = ctypes.c_double(), ctypes.c_double()
    _check(_lib.kpm_gershgorin_stencil(ctypes.byref(d), float(eps), ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def _csr_arrays(rowptr, col, val):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    val = np.asarray(val)
    if np.iscomplexobj(val):
        v = np.ascontiguousarray(val, dtype=np.complex128).view(np.float64)
        return rowptr, col, v, KPM_COMPLEX128
    return rowptr, col, np.ascontiguousarray(val, dtype=np.float64), KPM_REAL64


def kpm_gershgorin_csr(D, rowptr, col, val, eps=0.0):
    rowptr, col, v, dt = _csr_arrays(rowptr, col, val)
    a, b = ctypes.c_double(), ctypes.c_double()
    _check(_lib.kpm_gershgorin_csr(int(D), _ptr(rowptr), _ptr(col), _ptr(v), dt, float(eps),
                                   ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


class Handle:
    """Owns one kpm_handle (one GPU, one process)."""

    def __init__(self, raw, D, R_of=None, dist=None):
        self._lib = _lib         # the library that created it (libkpm.so or libkpm_exp.so)
        self._h = raw
        self.D = int(D)          # global number of sites
        self.D_local = int(D)    # sites on this rank (row partition: its slab)
        self.dist = dist

    def __del__(self):
        self.close()

    def _ck(self, st):
        _check(st, self._lib)

    def set_plan_opts(self, **opts):
        """kpm_set_plan_opts: keyword fields of kpm_plan_opts (no_small=1, tma_lanes=8, ...);
        no keywords = the default plan."""
        unknown = set(opts) - set(PLAN_OPTS)
        if unknown:
            raise ValueError(f"unknown plan options {sorted(unknown)}")
        if not opts:
            self._ck(self._lib.kpm_set_plan_opts(self._h, None))
            return
        o = kpm_plan_opts(**{k: int(v) for k, v in opts.items()})
        self._ck(self._lib.kpm_set_plan_opts(self._h, ctypes.byref(o)))

    def step_traffic(self):
        """(SURVEY 8(d) algorithmic bytes, compulsory DRAM bytes of the kernels that ran) of the
        recursion steps of the last call."""
        b = (ctypes.c_double * 2)()
        self._ck(self._lib.kpm_step_traffic(self._h, b))
        return b[0], b[1]

    def close(self):
        if getattr(self, "_h", None):
            self._lib.kpm_destroy(self._h)
            self._h = None

    @property
    def raw(self):
        return self._h

    def set_stream(self, stream_ptr: int):
        self._ck(self._lib.kpm_set_stream(self._h, ctypes.c_void_p(int(stream_ptr))))

    def workspace_size(self, N, R, flags=0):
        n = ctypes.c_size_t()
        self._ck(self._lib.kpm_workspace_size(self._h, int(N), int(R), int(flags), ctypes.byref(n)))
        return n.value

    def set_workspace(self, dev_ptr: int, nbytes: int):
        self._ck(self._lib.kpm_set_workspace(self._h, ctypes.c_void_p(int(dev_ptr)) if dev_ptr else None, int(nbytes)))

    def r_local(self, R):
        if self.dist is not None and self.dist[0] == KPM_PART_ROWS and len(self.dist) > 6 and self.dist[6] > 1:
            return kpm_vector_range(R, self.dist[5], self.dist[6])  # hybrid rows x vectors
        if self.dist is None or self.dist[0] != KPM_PART_VECTORS:
            return 0, int(R)
        _, rank, world = self.dist[:3]
        return kpm_vector_range(R, rank, world)

    def moments(self, N, R, seed):
        mu = np.zeros(int(N), dtype=np.float64)
        self._ck(self._lib.kpm_moments(self._h, int(N), int(R), int(seed), _ptr(mu)))
        return mu

    def moments_ex(self, N, R, seed, r0=None, flags=0, out=None):
        """out: None -> a new host array of the right shape; an int -> device pointer
        (pass KPM_DEVICE_OUT).  r0: host array (R_local, D) or an int device pointer
        (pass KPM_DEVICE_IN)."""
        _, R_loc = self.r_local(R)
        keep = None
        if r0 is None:
            r0p = None
        elif isinstance(r0, (int, np.integer)):
            r0p = ctypes.c_void_p(int(r0))
        elif flags & KPM_LOCAL:  # host list of R global sites
            keep = np.ascontiguousarray(r0, dtype=np.int64)
            assert keep.shape == (int(R),), keep.shape
            r0p = _ptr(keep)
            R_loc = self.r_local(R)[1]
        else:
            keep = np.ascontiguousarray(r0, dtype=np.float64)
            assert keep.shape == (R_loc, self.D_local), (keep.shape, (R_loc, self.D_local))
            r0p = _ptr(keep)
        if isinstance(out, (int, np.integer)):
            self._ck(self._lib.kpm_moments_ex(self._h, int(N), int(R), int(seed), r0p, int(flags),
                                       ctypes.c_void_p(int(out))))
            return None
        shape = (R_loc, int(N)) if flags & (KPM_PER_VECTOR | KPM_LOCAL) else (int(N),)
        res = np.zeros(shape, dtype=np.float64)
        self._ck(self._lib.kpm_moments_ex(self._h, int(N), int(R), int(seed), r0p, int(flags), _ptr(res)))
        return res

    def moments_local(self, N, sites):
        sites = np.ascontiguousarray(sites, dtype=np.int64)
        _, n_loc = self.r_local(len(sites))
        res = np.zeros((n_loc, int(N)), dtype=np.float64)
        self._ck(self._lib.kpm_moments_local(self._h, int(N), _ptr(sites), len(sites), _ptr(res)))
        return res

    def assemble(self, S, N, R, flags=0, out=None):
        """Raw sums -> moments (kpm_assemble); S: host array, or int device pointer with out."""
        if isinstance(S, (int, np.integer)):
            self._ck(self._lib.kpm_assemble(self._h, ctypes.c_void_p(int(S)), int(N), self.D, int(R),
                                     int(flags) | KPM_DEVICE_OUT, ctypes.c_void_p(int(out))))
            return None
        return kpm_assemble_host(S, N, self.D, R, flags)

    def last_timing(self):
        ms, sl, tl = ctypes.c_double(), ctypes.c_int32(), ctypes.c_int32()
        self._ck(self._lib.kpm_last_timing(self._h, ctypes.byref(ms), ctypes.byref(sl), ctypes.byref(tl)))
        return ms.value, sl.value, tl.value

    def plan_info(self, N, R, flags=0):
        info = np.zeros(12, dtype=np.int64)
        self._ck(self._lib.kpm_plan_info(self._h, int(N), int(R), int(flags), _ptr(info)))
        keys = ["tma", "TL", "TX", "TY", "ctas", "smem", "lanes", "_", "TX2", "ctas_per_sm2", "grid2"]
        d = {k: int(v) for k, v in zip(keys, info) if k != "_"}
        d["round_robin"] = int(info[7] & 1)
        d["two_step"] = int((info[7] >> 1) & 1)
        d["overlap"] = int((info[7] >> 2) & 1)
        d["box3"] = int((info[7] >> 3) & 1)  # 3D dense-box march kernel (kpm_tma3.cuh)
        d["two_step3d"] = int((info[7] >> 4) & 1)  # 3D two-step kernel (kpm_tma32.cuh)
        d["persist"] = int((info[7] >> 5) & 1)  # whole recursion in one cooperative launch (kpm_persist.cuh)
        d["ks"] = int(info[11])  # steps per launch of the deep temporal-blocking kernel (0 = not used)
        d["three_step"] = int((info[7] >> 6) & 1)  # three steps per launch (kpm_tri.cuh)
        d["four_step"] = int((info[7] >> 7) & 1)  # four steps per launch (kpm_quad.cuh)
        return d

    def last_stats(self):
        """step launches, all launches, halo plane copies, fused-halo launches of the last call"""
        st = np.zeros(4, dtype=np.int64)
        self._ck(self._lib.kpm_last_stats(self._h, _ptr(st)))
        return dict(step_launches=int(st[0]), launches=int(st[1]), halo_copies=int(st[2]), fused_halo=int(st[3]))

    def step_bytes(self):
        """Algorithmic HBM bytes of the recursion-step launches of the last call."""
        b = ctypes.c_double()
        self._ck(self._lib.kpm_step_bytes(self._h, ctypes.byref(b)))
        return b.value


def kpm_create_stencil(ndim, L, t, a, b, onsite=None, flux=0.0, device=0, dist=None) -> Handle:
    d, _keep = _desc(ndim, L, t, onsite, flux)
    h = ctypes.c_void_p()
    dp, _keep2 = _dist(dist)
    _check(_lib.kpm_create_stencil(ctypes.byref(d), float(a), float(b), int(device), dp, ctypes.byref(h)))
    Ls = tuple(L) + (1,) * (3 - len(L))
    hd = Handle(h.value, Ls[0] * Ls[1] * Ls[2], dist=dist)
    if dist is not None and dist[0] == KPM_PART_ROWS:
        slow = int(ndim) - 1
        _, cnt = kpm_slab_range(Ls[slow], dist[1], dist[2])
        hd.D_local = hd.D // Ls[slow] * cnt
    return hd


def kpm_create_csr(D, rowptr, col, val, a, b, device=0, dist=None) -> Handle:
    rowptr, col, v, dt = _csr_arrays(rowptr, col, val)
    h = ctypes.c_void_p()
    dp, _keep = _dist(dist)
    _check(_lib.kpm_create_csr(int(D), _ptr(rowptr), _ptr(col), _ptr(v), dt, float(a), float(b), int(device),
                               dp, ctypes.byref(h)))
    return _sparse_handle(h.value, D, dist)


def _sparse_handle(raw, D, dist):
    """Row partition of a general sparse H: this rank owns rows kpm_slab_range(D, rank, world)."""
    hd = Handle(raw, D, dist=dist)
    if dist is not None and dist[0] == KPM_PART_ROWS:
        hd.D_local = kpm_slab_range(D, dist[1], dist[2])[1]
    return hd


def kpm_create_dense(H, a, b, device=0, dist=None) -> Handle:
    """Dense real H (row-major D x D): the paper's own variant (DMMA GEMM per step)."""
    Hd = np.ascontiguousarray(H, dtype=np.float64)
    D = Hd.shape[0]
    assert Hd.shape == (D, D)
    dp, keep = _dist(dist)
    h = ctypes.c_void_p()
    _check(_lib.kpm_create_dense(D, _ptr(Hd), KPM_REAL64, float(a), float(b), int(device), dp, ctypes.byref(h)))
    return Handle(h.value, D, dist=dist)


def kpm_gershgorin_dense(H, eps=0.0):
    Hd = np.ascontiguousarray(H, dtype=np.float64)
    a, b = ctypes.c_double(), ctypes.c_double()
    _check(_lib.kpm_gershgorin_dense(Hd.shape[0], _ptr(Hd), KPM_REAL64, float(eps), ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def kpm_create_ell(D, K, col, val, a, b, device=0, dist=None) -> Handle:
    col = np.ascontiguousarray(col, dtype=np.int32)
    val = np.asarray(val)
    if np.iscomplexobj(val):
        v, dt = np.ascontiguousarray(val, dtype=np.complex128).view(np.float64), KPM_COMPLEX128
    else:
        v, dt = np.ascontiguousarray(val, dtype=np.float64), KPM_REAL64
    h = ctypes.c_void_p()
    dp, _keep = _dist(dist)
    _check(_lib.kpm_create_ell(int(D), int(K), _ptr(col), _ptr(v), dt, float(a), float(b), int(device),
                               dp, ctypes.byref(h)))
    return _sparse_handle(h.value, D, dist)


def kpm_moments(h: Handle, N, R, seed):
    return h.moments(N, R, seed)


def kpm_moments_ex(h: Handle, N, R, seed, r0=None, flags=0, out=None):
    return h.moments_ex(N, R, seed, r0=r0, flags=flags, out=out)


def kpm_assemble(h: Handle, S, N, R, flags=0, out=None):
    return h.assemble(S, N, R, flags=flags, out=out)


def kpm_assemble_host(S, N, D, R, flags=0):
    """kpm_assemble on host arrays (no GPU needed)."""
    S = np.ascontiguousarray(S, dtype=np.float64)
    mu = np.zeros(int(N), dtype=np.float64)
    _check(_lib.kpm_assemble(None, _ptr(S), int(N), int(D), int(R), int(flags) & ~KPM_DEVICE_OUT, _ptr(mu)))
    return mu


def kpm_csr_partition(D, rowptr, col, rank, world):
    """Host-side row-partition plan of a CSR matrix (include/kpm.h): dict with n_local, ghosts
    (global indices, ascending), send_rows (local rows per peer) and peers [world][4] =
    (ghost offset, ghost count, send offset, send count)."""
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    counts = np.zeros(3, dtype=np.int64)
    _check(_lib.kpm_csr_partition(int(D), _ptr(rowptr), _ptr(col), int(rank), int(world), _ptr(counts),
                                  None, None, None))
    ghosts = np.zeros(int(counts[1]), dtype=np.int64)
    send = np.zeros(int(counts[2]), dtype=np.int64)
    peers = np.zeros((int(world), 4), dtype=np.int64)
    _check(_lib.kpm_csr_partition(int(D), _ptr(rowptr), _ptr(col), int(rank), int(world), _ptr(counts),
                                  _ptr(ghosts), _ptr(send), _ptr(peers)))
    return dict(n_local=int(counts[0]), ghosts=ghosts, send_rows=send, peers=peers)


def kpm_slab_range(Lm, rank, world):
    """(begin, count) of the planes of the slowest lattice dimension rank owns under KPM_PART_ROWS."""
    b, c = ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.kpm_slab_range(int(Lm), int(rank), int(world), ctypes.byref(b), ctypes.byref(c)))
    return b.value, c.value


def kpm_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.kpm_nccl_unique_id(buf))
    return buf.raw


def kpm_ipc_unique_name() -> str:
    """A fresh shared-segment name for KPM_COMM_IPC (make it on one rank, pass it to all)."""
    buf = ctypes.create_string_buffer(64)
    _check(_lib.kpm_ipc_unique_name(buf))
    return buf.value.decode()


def kpm_moments_group(handles, N, R, seed):
    """KPM_COMM_LOCAL partitions: all rank handles of this process (row partition: slabs in lock
    step with halo exchange; vector partition: every rank's share, sums combined in rank order)."""
    arr = (ctypes.c_void_p * len(handles))(*[h.raw for h in handles])
    mu = np.zeros(int(N), dtype=np.float64)
    lib = handles[0]._lib
    _check(lib.kpm_moments_group(arr, len(handles), int(N), int(R), int(seed), _ptr(mu)), lib)
    return mu


def nccl_id_for_group(group=None) -> bytes:
    """ncclUniqueId made on rank 0 and broadcast to every rank with torch.distributed
    (the plumbing for KPM_COMM_NCCL; the library then creates its own communicator)."""
    import torch
    import torch.distributed as dist
    t = torch.zeros(128, dtype=torch.uint8)
    if dist.get_rank(group) == 0:
        t = torch.frombuffer(bytearray(kpm_nccl_unique_id()), dtype=torch.uint8).clone()
    backend = dist.get_backend(group)
    if backend == "nccl":
        t = t.cuda()
    dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return bytes(t.cpu().numpy().tobytes())


def kpm_vector_range(R, rank, world):
    """(begin, count) of the global vectors rank owns under KPM_PART_VECTORS."""
    b, c = ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.kpm_vector_range(int(R), int(rank), int(world), ctypes.byref(b), ctypes.byref(c)))
    return b.value, c.value


def kpm_dos(mu, a, b, omega, kernel=KPM_KERNEL_JACKSON, device=0):
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    om = np.ascontiguousarray(omega, dtype=np.float64)
    rho = np.zeros(len(om), dtype=np.float64)
    _check(_lib.kpm_dos(_ptr(mu), len(mu), int(kernel), float(a), float(b), _ptr(om), len(om), _ptr(rho),
                        int(device)))
    return rho


def kpm_dos_ex(mu, a, b, omega, kernel=KPM_KERNEL_JACKSON, lam=KPM_LORENTZ_DEFAULT_LAMBDA, device=0):
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    om = np.ascontiguousarray(omega, dtype=np.float64)
    rho = np.zeros(len(om), dtype=np.float64)
    _check(_lib.kpm_dos_ex(_ptr(mu), len(mu), int(kernel), float(lam), float(a), float(b), _ptr(om), len(om),
                           _ptr(rho), int(device)))
    return rho


def kpm_green(mu, a, b, omega, kernel=KPM_KERNEL_JACKSON, lam=KPM_LORENTZ_DEFAULT_LAMBDA, device=0):
    """Retarded Green's function G(omega) (complex128[K]) from the damped moments."""
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    om = np.ascontiguousarray(omega, dtype=np.float64)
    G = np.zeros(2 * len(om), dtype=np.float64)
    _check(_lib.kpm_green(_ptr(mu), len(mu), int(kernel), float(lam), float(a), float(b), _ptr(om), len(om),
                          _ptr(G), int(device)))
    return G[0::2] + 1j * G[1::2]


def kpm_damping(N, kernel=KPM_KERNEL_JACKSON, lam=KPM_LORENTZ_DEFAULT_LAMBDA, device=0):
    g = np.zeros(int(N), dtype=np.float64)
    _check(_lib.kpm_damping(int(N), int(kernel), float(lam), _ptr(g), int(device)))
    return g


def kpm_moment_stats(mu_pv, device=0):
    """(mean[N], sem[N]) of per-vector moments [R][N] (KPM_PER_VECTOR): the stochastic
    estimate and its standard error."""
    pv = np.ascontiguousarray(mu_pv, dtype=np.float64)
    if pv.ndim != 2:
        raise ValueError("mu_pv must be [R][N]")
    R, N = pv.shape
    mean, sem = np.zeros(N), np.zeros(N)
    _check(_lib.kpm_moment_stats(_ptr(pv), R, N, _ptr(mean), _ptr(sem), int(device)))
    return mean, sem


def kpm_moments_local(h: Handle, N, sites):
    """<i|T_n(H~)|i> for the global sites i (this rank's share under KPM_PART_VECTORS)."""
    return h.moments_local(N, sites)


def kpm_destroy(h: Handle):
    h.close()


def moments_distributed(h, N, R, seed, group=None, flags=0, device=None):
    """Random-vector partition across ranks (one process per GPU).

    A handle created with dist = (KPM_PART_VECTORS, rank, world, KPM_COMM_NCCL, nccl_id) owns
    the collective: kpm_moments runs this rank's share of the R vectors and the library's one
    ncclAllReduce of the sums, and returns mu on every rank -- this function only marshals.
    A handle without a library communicator (KPM_COMM_SELF, e.g. ranks that share one GPU,
    where NCCL refuses duplicate devices) gets the caller-owned form of the same collective:
    raw sums (KPM_RAW_SUMS), one torch.distributed all-reduce (gloo or NCCL), kpm_assemble.
    device: torch device for the sums in that form (default: the current CUDA device)."""
    d = getattr(h, "dist", None)
    if d is not None and len(d) > 3 and d[3] == KPM_COMM_NCCL and not flags:
        return h.moments(N, R, seed)
    import torch
    import torch.distributed as dist
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type == "cuda":
        S = torch.empty(int(N), dtype=torch.float64, device=device)
        h.moments_ex(N, R, seed, flags=flags | KPM_RAW_SUMS | KPM_DEVICE_OUT, out=S.data_ptr())
        torch.cuda.synchronize(device)
        dist.all_reduce(S, op=dist.ReduceOp.SUM, group=group)
        mu = torch.empty_like(S)
        h.assemble(S.data_ptr(), N, R, flags=flags & KPM_DIRECT, out=mu.data_ptr())
        torch.cuda.synchronize(device)
        return mu.cpu().numpy()
    S = torch.from_numpy(np.ascontiguousarray(h.moments_ex(N, R, seed, flags=flags | KPM_RAW_SUMS)))
    dist.all_reduce(S, op=dist.ReduceOp.SUM, group=group)
    return h.assemble(S.numpy(), N, R, flags=flags & KPM_DIRECT)
