"""KPM_COMM_IPC: partitions whose ranks are separate PROCESSES exchanging halos and sums through
CUDA IPC (the multi-process NVLink halo).

Each case starts `world` processes on cuda:0 (this pool has one GPU; NCCL refuses two ranks on
one device, CUDA IPC does not).  Row partition: every recursion launch of a rank stores its
boundary planes straight into the neighbours' ghost planes (fused halo, counted by
kpm_last_stats[3]); only the first step's ghosts are copied.  Ordering between launches is by
interprocess CUDA events, so no kernel spins on a peer.  Every rank must return the oracle's
moments (X17, 1e-10) and all ranks identical bits."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import kpm_inputs as ki
import oracle
from test_gpu_parity import lat_of, normwise

pytestmark = pytest.mark.gpu
TOL = 1e-10
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_WORKER = r'''
import sys, json
sys.path.insert(0, sys.argv[1])
import numpy as np
import kpm_inputs as ki
from paper_1105_5481_b200 import kpm
rank, world, name = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
spec = json.loads(sys.argv[5])
L = tuple(spec["L"]); D = int(np.prod(L))
ndim = spec["ndim"]
onsite = ki.anderson_onsite(5, D, spec["W"]) if spec["W"] else None
a, b = kpm.kpm_gershgorin_stencil(ndim, L, -1.0, onsite=onsite, flux=spec["flux"])
part = kpm.KPM_PART_ROWS if spec["part"] == "rows" else kpm.KPM_PART_VECTORS
h = kpm.kpm_create_stencil(ndim, L, -1.0, a, b, onsite=onsite, flux=spec["flux"],
                           dist=(part, rank, world, kpm.KPM_COMM_IPC, name))
if spec.get("no_fused"):
    h.set_plan_opts(no_fused_halo=1)
N = spec["N"] + (1 if (rank == 1 and spec.get("bad_N")) else 0)
out = {"rank": rank, "a": a, "b": b}
try:
    mus = [h.moments(N, spec["R"], spec["seed"]).tolist() for _ in range(spec.get("calls", 1))]
    out["mu"] = mus[0]
    out["repeat_same"] = all(m == mus[0] for m in mus)
    out["stats"] = h.last_stats()
    if spec.get("per_vector"):
        out["pv"] = h.moments_ex(N, spec["R"], spec["seed"], flags=kpm.KPM_PER_VECTOR).tolist()
except kpm.KPMError as e:
    out["error"] = e.status
print(json.dumps(out))
h.close()
'''


def run_world(tmp_path, world, spec, timeout=240):
    from paper_1105_5481_b200 import kpm
    w = tmp_path / "ipc_worker.py"
    w.write_text(_WORKER)
    name = kpm.kpm_ipc_unique_name()
    procs = [subprocess.Popen([sys.executable, str(w), ROOT, str(r), str(world), name, json.dumps(spec)],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True) for r in range(world)]
    outs = []
    try:
        for p in procs:
            o, e = p.communicate(timeout=timeout)
            assert p.returncode == 0, e[-3000:]
            outs.append(json.loads(o.strip().splitlines()[-1]))
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert not os.path.exists("/dev/shm" + name), "rank 0 removes the segment name"
    return outs


def reference(spec, a, b):
    lat = lat_of(spec["ndim"], spec["L"], W=spec["W"], flux=spec["flux"])
    H = oracle.lattice_csr(lat)
    ao, bo = oracle.gershgorin(H)
    assert abs(ao - a) < 1e-14 * a and abs(bo - b) < 1e-14 * a
    r0 = ki.rademacher(spec["seed"], spec["R"], lat["D"])
    return oracle.moments_doubling(H, a, b, r0, spec["N"]), H, r0


ROWS = {
    # 3D Anderson slabs along z: TMA box march (in-place single steps), fused peer-plane stores
    "3d_anderson": dict(ndim=3, L=[32, 16, 12], W=2.0, flux=0.0, N=25, R=48, seed=9),
    # 2D clean lattice, slabs along y, odd N (the tail reduction)
    "2d_odd_N": dict(ndim=2, L=[64, 40], W=0.0, flux=0.0, N=31, R=32, seed=3),
    # complex128 Peierls lattice (flux 1/8), slabs along y
    "2d_peierls": dict(ndim=2, L=[64, 24], W=1.0, flux=0.125, N=28, R=16, seed=4),
    # uneven slabs (10 planes over 3 ranks: 3, 3, 4), 16-lane box tiles
    "3d_uneven_slabs": dict(ndim=3, L=[16, 8, 10], W=2.0, flux=0.0, N=19, R=32, seed=8),
}


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", sorted(ROWS))
def test_ipc_row_partition_fused_halo(tmp_path, case, world):
    spec = dict(ROWS[case], part="rows", calls=2)
    outs = run_world(tmp_path, world, spec)
    ref, _, _ = reference(spec, outs[0]["a"], outs[0]["b"])
    for o in outs:
        assert "error" not in o, o
        assert o["mu"] == outs[0]["mu"], "ranks disagree"
        assert o["repeat_same"], "a second call (mapped workspaces reused) changed the result"
        assert normwise(np.array(o["mu"]), ref) < TOL
        copies, fused = o["stats"]["halo_copies"], o["stats"]["fused_halo"]
        assert fused == spec["N"] // 2 - 1 and copies == 2, o["stats"]  # only the first step's ghosts copied


def test_ipc_row_partition_copy_mode_and_per_vector(tmp_path):
    """opts.no_fused_halo: ghost planes pulled from the neighbours' mapped blocks after every launch;
    per-vector moments summed over the slabs."""
    spec = dict(ROWS["3d_anderson"], part="rows", no_fused=True, per_vector=True)
    outs = run_world(tmp_path, 2, spec)
    ref, H, r0 = reference(spec, outs[0]["a"], outs[0]["b"])
    _, ref_pv = oracle.moments_doubling(H, outs[0]["a"], outs[0]["b"], r0, spec["N"], per_vector=True)
    for o in outs:
        assert normwise(np.array(o["mu"]), ref) < TOL
        assert o["stats"]["fused_halo"] == 0 and o["stats"]["halo_copies"] == 2 * (spec["N"] // 2), o["stats"]
        assert normwise(np.array(o["pv"]), ref_pv) < TOL
    assert outs[0]["pv"] == outs[1]["pv"]


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_vector_partition(tmp_path, world):
    """Random-vector partition over processes: each rank runs kpm_vector_range(R, rank, world); the
    library sums S over the ranks (rank order) and returns mu on every rank."""
    spec = dict(ndim=2, L=[64, 40], W=1.0, flux=0.0, N=40, R=64, seed=6, part="vectors")
    outs = run_world(tmp_path, world, spec)
    ref, _, _ = reference(spec, outs[0]["a"], outs[0]["b"])
    for o in outs:
        assert o["mu"] == outs[0]["mu"]
        assert normwise(np.array(o["mu"]), ref) < TOL


def test_ipc_mismatched_calls_fail_on_every_rank(tmp_path):
    """Ranks that call with different N: every rank returns KPM_ERR_COMM (no hang)."""
    from paper_1105_5481_b200 import kpm
    spec = dict(ROWS["2d_odd_N"], part="rows", bad_N=True)
    outs = run_world(tmp_path, 2, spec)
    assert all(o.get("error") == kpm.KPM_ERR_COMM for o in outs), outs
