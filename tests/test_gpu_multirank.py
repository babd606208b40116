"""Multi-rank random-vector partition through the REAL kernels, and the
boundary's error paths that came with it (KPM_ERR_NCCL, kpm_plan_opts, per-device state).

On one GPU NCCL refuses two ranks on the same device, so the multi-rank cases here are:
(i) the library's NCCL communicator at world 1 (KPM_COMM_NCCL: the all-reduce inside
kpm_moments); (ii) in-process rank handles (KPM_COMM_LOCAL, kpm_moments_group: every rank's
share of the vectors on its own stream, sums combined in rank order); (iii) two processes on
cuda:0 with a gloo all-reduce of the library's raw sums (the caller-owned form of the same
collective, kpm.moments_distributed); (iv) bench.py --gpus 2 on one GPU.  Bar: DESIGN.md X17."""
import json
import os
import socket
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


@pytest.fixture(scope="module")
def kpm():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1105_5481_b200 import kpm as k
    return k


CASES = {
    "2d_two_step_R64": (lat_of(2, (64, 40)), 40, 64),
    "3d_anderson_R48": (lat_of(3, (32, 16, 12), W=2.0), 25, 48),
    "peierls_R32": (lat_of(2, (64, 16), flux=1 / 8, W=1.0), 31, 32),
    "2d_small_R5": (lat_of(2, (37, 29)), 26, 5),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_library_nccl_vector_partition_world1(kpm, case):
    """KPM_COMM_NCCL on the vector partition: the handle owns the communicator and kpm_moments
    returns mu (the one ncclAllReduce of S runs inside the library)."""
    lat, N, R = CASES[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(4, R, lat["D"]), N)
    nid = kpm.kpm_nccl_unique_id()
    h = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"], flux=lat["flux"],
                               dist=(kpm.KPM_PART_VECTORS, 0, 1, kpm.KPM_COMM_NCCL, nid))
    mu = h.moments(N, R, 4)
    assert normwise(mu, ref) < TOL
    assert np.array_equal(kpm.moments_distributed(h, N, R, 4), mu)  # marshalling only
    # a second handle from the same id shares the communicator; both keep working
    h2 = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"], flux=lat["flux"],
                                dist=(kpm.KPM_PART_VECTORS, 0, 1, kpm.KPM_COMM_NCCL, nid))
    assert np.array_equal(h2.moments(N, R, 4), mu)
    h2.close()
    assert np.array_equal(h.moments(N, R, 4), mu)


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("case", sorted(CASES))
def test_local_vector_group_matches_oracle(kpm, case, world):
    """KPM_COMM_LOCAL vector partition: `world` rank handles in this process, each running its
    share kpm_vector_range(R, rank, world) of the global vectors through the real kernels."""
    lat, N, R = CASES[case]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(4, R, lat["D"]), N)
    hs = [kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"], flux=lat["flux"],
                                 dist=(kpm.KPM_PART_VECTORS, rk, world, kpm.KPM_COMM_LOCAL)) for rk in range(world)]
    mu = kpm.kpm_moments_group(hs, N, R, 4)
    assert normwise(mu, ref) < TOL
    whole = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b, onsite=lat["onsite"],
                                   flux=lat["flux"]).moments(N, R, 4)
    assert normwise(mu, whole) < 1e-13


def test_vector_partition_without_comm_refuses_plain_moments(kpm):
    lat, N, R = CASES["2d_small_R5"]
    h = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], 4.0, 0.0, dist=(kpm.KPM_PART_VECTORS, 0, 2))
    with pytest.raises(kpm.KPMError) as e:
        h.moments(N, R, 1)
    assert e.value.status == kpm.KPM_ERR_INVALID_ARG


_WORKER = r'''
import os, sys, json
sys.path.insert(0, sys.argv[1])
import numpy as np, torch, torch.distributed as dist
rank, world = int(sys.argv[2]), int(sys.argv[3])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + sys.argv[4], rank=rank, world_size=world)
torch.cuda.set_device(0)
import kpm_inputs as ki
from paper_1105_5481_b200 import kpm
lat = dict(ndim=3, L=(32, 16, 12), D=6144, t=-1.0, onsite=ki.anderson_onsite(5, 6144, 2.0), flux=0.0)
a, b = kpm.kpm_gershgorin_stencil(3, lat["L"], -1.0, onsite=lat["onsite"])
h = kpm.kpm_create_stencil(3, lat["L"], -1.0, a, b, onsite=lat["onsite"], dist=(kpm.KPM_PART_VECTORS, rank, world))
mu = kpm.moments_distributed(h, 33, 48, 9, device=torch.device("cpu"))
print(json.dumps({"rank": rank, "a": a, "b": b, "mu": mu.tolist(), "r_local": h.r_local(48)}))
dist.destroy_process_group()
'''


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_processes_gloo_real_kernels(kpm, tmp_path):
    """Two processes on cuda:0, each running its share of the 48 global vectors through the CUDA
    kernels; one gloo all-reduce of the raw sums; both ranks return the oracle's moments."""
    w = tmp_path / "worker.py"
    w.write_text(_WORKER)
    port = str(_port())
    procs = [subprocess.Popen([sys.executable, str(w), ROOT, str(r), "2", port], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for r in range(2)]
    outs = []
    for p in procs:
        o, e = p.communicate(timeout=300)
        assert p.returncode == 0, e[-3000:]
        outs.append(json.loads(o.strip().splitlines()[-1]))
    lat = dict(ndim=3, L=(32, 16, 12), D=6144, t=-1.0, onsite=ki.anderson_onsite(5, 6144, 2.0), flux=0.0)
    H = oracle.lattice_csr(lat)
    a, b = outs[0]["a"], outs[0]["b"]
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(9, 48, 6144), 33)
    assert outs[0]["r_local"] == [0, 24] and outs[1]["r_local"] == [24, 24]
    assert outs[0]["mu"] == outs[1]["mu"], "ranks disagree"
    assert normwise(np.array(outs[0]["mu"]), ref) < TOL


def test_bench_two_ranks_on_one_gpu():
    """bench.py --gpus 2 starts two ranks itself (torch.distributed.run); on one GPU they share
    it through gloo and the line says n_gpus = 2 with the strong-scaling split of R."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "c2", "--steps", "2",
                        "--warmup", "1", "--no-cpu-baseline", "--no-e2e"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong", line
    assert line["config"]["R_total"] == 64 and line["config"]["R_per_gpu"] == 32, line["config"]
    assert line["mu_check"]["mu0"] == 1.0
    assert line["gpu_launches"] > 0 and line["roofline"]["achieved"] > 0


def test_bench_rows_two_ranks_ipc_halo():
    """bench.py --gpus 2 --partition rows: two processes (sharing the one GPU here), slabs of c3 with
    the KPM_COMM_IPC fused halo -- every recursion launch stores into the peer's ghost planes."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "c3", "--partition",
                        "rows", "--steps", "1", "--warmup", "1", "--no-cpu-baseline"], capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "rows2", line
    assert line["halo_stats"]["fused_halo"] == 2048 // 2 - 1 and line["halo_stats"]["halo_copies"] == 2
    assert line["mu_check"]["mu0"] == 1.0 and line["mu_check"]["max_abs_mu"] <= 1.0


def test_plan_opts_validation(kpm):
    lat, N, R = CASES["2d_small_R5"]
    h = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], 4.0, 0.0)
    with pytest.raises(kpm.KPMError) as e:
        h.set_plan_opts(no_small=-1)
    assert e.value.status == kpm.KPM_ERR_INVALID_ARG
    with pytest.raises(kpm.KPMError) as e:
        h.set_plan_opts(experimental=kpm.EXP_PERSIST)  # not in the default libkpm.so
    assert e.value.status == kpm.KPM_ERR_UNSUPPORTED
    with pytest.raises(ValueError):
        h.set_plan_opts(bogus=1)
    h.set_plan_opts()  # default plan


def test_ell_kernel_smem_fallback_small_R(kpm):
    """a 3D CSR lattice past the small-kernel limit with R = 1 and one local site (the
    staged ELL kernel's tile would exceed shared memory) falls back to the generic kernel."""
    lat = lat_of(3, (32, 28, 24), W=2.0)
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    h = kpm.kpm_create_csr(H.D, H.rowptr, H.col, H.val_re, a, b)
    h.set_plan_opts(no_small=1)
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(3, 1, H.D), 20)
    assert normwise(h.moments(20, 1, 3), ref) < TOL
    sites = [7]
    lm = h.moments_local(20, sites)
    assert normwise(lm, oracle.local_moments(H, a, b, sites, 20)) < TOL


def test_set_stream_switch_keeps_results(kpm):
    """switching from one caller stream to another with work queued on the first."""
    import torch
    lat, N, R = CASES["2d_two_step_R64"]
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    h = kpm.kpm_create_stencil(lat["ndim"], lat["L"], lat["t"], a, b)
    ref = h.moments(N, R, 2)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    S = torch.empty(N, dtype=torch.float64, device="cuda")
    h.set_stream(s1.cuda_stream)
    h.moments_ex(N, R, 2, flags=kpm.KPM_DEVICE_OUT, out=S.data_ptr())  # queued on s1
    h.set_stream(s2.cuda_stream)  # must wait for s1's work before the workspace is reused
    mu = h.moments(N, R, 2)
    s1.synchronize()
    assert np.array_equal(mu, ref) and np.array_equal(S.cpu().numpy(), ref)


@pytest.mark.skipif("int(__import__('torch').cuda.device_count()) < 2")
def test_slab_group_on_two_devices(kpm):
    """shared-memory attributes are per device -- a slab group spanning two GPUs."""
    lat = lat_of(3, (32, 16, 12), W=2.0)
    H = oracle.lattice_csr(lat)
    a, b = oracle.gershgorin(H)
    N, R = 25, 16
    ref = oracle.moments_doubling(H, a, b, ki.rademacher(8, R, lat["D"]), N)
    hs = [kpm.kpm_create_stencil(3, lat["L"], -1.0, a, b, onsite=lat["onsite"], device=rk,
                                 dist=(kpm.KPM_PART_ROWS, rk, 2, kpm.KPM_COMM_LOCAL)) for rk in range(2)]
    assert normwise(kpm.kpm_moments_group(hs, N, R, 8), ref) < TOL
