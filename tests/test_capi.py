"""C-ABI library checks that need no GPU: it loads, exports every symbol include/kpm.h
declares, and its host-side helpers (Gerschgorin, argument validation) behave."""
import os
import re

import numpy as np
import pytest

import kpm_inputs as ki
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "kpm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kpm_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_1105_5481_b200 import kpm
    syms = declared_symbols()
    assert len(syms) >= 15
    lib = ctypes.CDLL(kpm.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), f"libkpm.so does not export {s}"
    assert set(syms) == set(kpm.EXPORTS)
    assert "sm_100a" in kpm.kpm_version()


def test_library_has_sm100a_code_only():
    import subprocess
    from paper_1105_5481_b200 import kpm
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", kpm.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_gershgorin_stencil_matches_oracle():
    from paper_1105_5481_b200 import kpm
    for ndim, L, W in [(1, (64, 1, 1), 0.0), (2, (16, 8, 1), 1.0), (3, (6, 5, 4), 2.0)]:
        D = int(np.prod(L))
        eps = ki.anderson_onsite(7, D, W) if W else None
        a, b = kpm.kpm_gershgorin_stencil(ndim, L, -1.0, onsite=eps)
        ao, bo = oracle.gershgorin(oracle.lattice_csr(dict(ndim=ndim, L=L, t=-1.0, onsite=eps, flux=0.0)))
        assert abs(a - ao) < 1e-14 and abs(b - bo) < 1e-14


def test_gershgorin_csr_matches_oracle_complex():
    from paper_1105_5481_b200 import kpm
    rng = np.random.default_rng(1)
    A = rng.normal(size=(20, 20)) + 1j * rng.normal(size=(20, 20))
    A = A + A.conj().T
    H = oracle.csr_from_dense(A)
    a, b = kpm.kpm_gershgorin_csr(H.D, H.rowptr, H.col, H.val_re + 1j * H.val_im)
    ao, bo = oracle.gershgorin(H)
    assert abs(a - ao) < 1e-12 and abs(b - bo) < 1e-12


def test_invalid_arguments_are_rejected():
    from paper_1105_5481_b200 import kpm
    with pytest.raises(kpm.KPMError) as e:
        kpm.kpm_gershgorin_stencil(4, (4, 4, 4), -1.0)
    assert e.value.status == kpm.KPM_ERR_INVALID_ARG
    with pytest.raises(kpm.KPMError):
        kpm.kpm_gershgorin_stencil(2, (10, 10, 1), -1.0, flux=0.125)  # flux * L0 not integer
    with pytest.raises(kpm.KPMError):
        kpm.kpm_gershgorin_stencil(3, (1, 4, 4), -1.0)
    with pytest.raises(kpm.KPMError):
        kpm.kpm_gershgorin_stencil(2, (4, 4, 2), -1.0)                # unused dim must be 1
    with pytest.raises(kpm.KPMError) as e:
        kpm.kpm_create_stencil(2, (8, 8), -1.0, a=-1.0, b=0.0)       # a <= 0
    assert e.value.status == kpm.KPM_ERR_INVALID_ARG


def test_ipc_unique_name_and_dist_layout():
    """KPM_COMM_IPC plumbing that needs no GPU: fresh shared-segment names ("/kpm-<pid>-<hex>",
    < 64 bytes, distinct per call) and the ctypes kpm_dist carrying the name at the end."""
    import ctypes
    from paper_1105_5481_b200 import kpm
    names = {kpm.kpm_ipc_unique_name() for _ in range(8)}
    assert len(names) == 8
    for n in names:
        assert re.fullmatch(r"/kpm-%d-[0-9a-f]{16}" % os.getpid(), n) and len(n) < 64
    ref, keep = kpm._dist((kpm.KPM_PART_ROWS, 1, 3, kpm.KPM_COMM_IPC, "/kpm-x"))
    st = keep[0]
    assert (st.partition, st.rank, st.world, st.comm) == (kpm.KPM_PART_ROWS, 1, 3, kpm.KPM_COMM_IPC)
    assert st.ipc_name == b"/kpm-x" and st.nccl_id is None
    assert kpm_dist_fields_match_header()


def kpm_dist_fields_match_header():
    """the binding's kpm_dist field order equals the header's struct members"""
    from paper_1105_5481_b200 import kpm
    src = re.sub(r"/\*.*?\*/", "", open(os.path.join(ROOT, "include", "kpm.h")).read(), flags=re.S)
    body = re.search(r"typedef struct \{([^}]*)\} kpm_dist;", src).group(1)
    names = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        head, *rest = decl.split(",")
        names.append(re.findall(r"(\w+)\s*$", head)[0])
        names += [r.strip().lstrip("*") for r in rest]
    return names == [f[0] for f in kpm.kpm_dist._fields_]
